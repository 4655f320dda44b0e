"""Command line for the B200 query path: search, bench (with an index), inspect.

Mirror of the query-side commands of /root/reference/pkg/src/icq/cli.py
(SURVEY §8(f)4): the same flags, the same resolved-configuration echo on
stderr, the same payload files byte for byte, the same exit codes (usage 2,
runtime failure 1, success 0).  Every query of a command runs in one batched
device call per engine instead of one Python call per query.

    python -m paper_1912_08756_b200.cli search --index I.icqi --queries Q.icqd --k 10 --out R.csv
    python -m paper_1912_08756_b200.cli search --mode brute --data D.icqd --queries Q.icqd --out R.csv
    python -m paper_1912_08756_b200.cli bench --in D.icqd --queries Q.icqd --index I.icqi --out B.csv
    python -m paper_1912_08756_b200.cli inspect FILE

Training, data generation and the unseen-class protocol (``gen``, ``train``,
``bench`` without ``--index``) are outside the query path and stay with the
reference package.
"""

from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import numpy as np

from .data import FormatError, ValidationError
from .evaluate import run_benchmark
from .io import load_dataset, load_index
from .search import search_bruteforce_batch, search_exact_batch, search_two_step_batch


def _echo(command: str, args: argparse.Namespace) -> None:
    pairs = sorted((k, v) for k, v in vars(args).items() if k != "func" and not k.startswith("_"))
    print(f"# {command}: " + " ".join(f"{k}={v}" for k, v in pairs), file=sys.stderr)


def _search_sigma(args: argparse.Namespace, index):
    """cli.py:128-132: --sigma-scale times the summed variance outside the mask."""
    if args.sigma_scale is None:
        return None
    lam = index.lambdas.astype(np.float64)
    return args.sigma_scale * float(lam[index.xi == 0].sum())


def cmd_search(args: argparse.Namespace) -> int:
    """cli.py:135-162: one CSV row per (query, rank)."""
    _echo("search", args)
    queries = load_dataset(args.queries)
    if args.mode == "brute":
        if args.data is None:
            raise ValidationError("brute mode needs --data with the raw dataset")
        res = search_bruteforce_batch(load_dataset(args.data), queries.vectors, args.k)
        fallback = [0] * queries.n
    else:
        if args.index is None:
            raise ValidationError(f"{args.mode} mode needs --index")
        index = load_index(args.index)
        if args.mode == "exact":
            res = search_exact_batch(index, queries.vectors, args.k)
        else:
            res = search_two_step_batch(index, queries.vectors, args.k, sigma=_search_sigma(args, index))
        fallback = [int(res.fallback)] * queries.n
    lines = ["query,rank,id,score,fast_adds,exact_adds,lut_ops,fallback"]
    for qi in range(queries.n):
        ops = res.ops[qi]
        for rank, (i, s) in enumerate(zip(res.ids[qi], res.scores[qi])):
            lines.append(f"{qi},{rank},{i},{float(s)!r},{ops.fast_adds},{ops.exact_adds},"
                         f"{ops.lut_ops},{fallback[qi]}")
    Path(args.out).write_text("\n".join(lines) + "\n")
    return 0


def cmd_bench(args: argparse.Namespace) -> int:
    """cli.py:165-196 with a given index (training is not on the query path)."""
    _echo("bench", args)
    if args.unseen_fraction is not None or not args.index:
        raise ValidationError("training is outside the B200 query path: pass --index "
                              "(and --queries); use the reference CLI to train")
    ds = load_dataset(args.in_path)
    if args.queries is None:
        raise ValidationError("bench needs --queries unless --unseen-fraction is set")
    queries = load_dataset(args.queries)
    index = load_index(args.index)
    labeled = ds.labels is not None and queries.labels is not None
    threads = int(os.environ.get("ICQ_THREADS", "1") or 1)
    report = run_benchmark(index, ds, queries, truth="labels" if labeled else "brute", k=args.k,
                           threads=threads)
    Path(args.out).write_text(report.to_csv())
    print(f"# bench: map={report.map!r} map_exact={report.map_exact!r} "
          f"avg_ops={report.avg_ops!r} avg_ops_exact={report.avg_ops_exact!r} "
          f"ecl={report.effective_code_length!r} fallbacks={report.fallbacks}", file=sys.stderr)
    return 0


def cmd_inspect(args: argparse.Namespace) -> int:
    """cli.py:199-222."""
    _echo("inspect", args)
    with open(args.path, "rb") as f:
        magic = f.read(4)
    if magic == b"ICQD":
        ds = load_dataset(args.path)
        print(f"dataset: n={ds.n} d={ds.d} labeled={ds.labels is not None}")
        if ds.labels is not None and ds.n:
            print(f"classes: {np.unique(ds.labels).size}")
    elif magic == b"ICQI":
        index = load_index(args.path)
        cfg = index.cfg
        print(f"index: n={index.n} d={index.d} K={cfg.K} m={cfg.m}")
        print(f"psi: {int(index.xi.sum())} of {index.d} dims")
        print(f"fast: {index.fast.tolist()}")
        print(f"sigma: {index.sigma!r}")
        print(f"config: gamma1={cfg.gamma1} gamma2={cfg.gamma2} sigma_scale={cfg.sigma_scale} "
              f"epochs={cfg.epochs} batch_size={cfg.batch_size} "
              f"learning_rate={cfg.learning_rate} seed={cfg.seed}")
    else:
        raise FormatError(f"unrecognized magic {magic!r} in {args.path}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="icq-b200", description=__doc__)
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("search", help="query an index (or brute-force a dataset)")
    p.add_argument("--index", default=None)
    p.add_argument("--queries", required=True)
    p.add_argument("--k", type=int, default=10)
    p.add_argument("--mode", choices=["two-step", "exact", "brute"], default="two-step")
    p.add_argument("--sigma-scale", type=float, default=None,
                   help="override sigma as scale * sum of lambdas outside the mask")
    p.add_argument("--data", default=None, help="raw dataset for brute mode")
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_search)
    p = sub.add_parser("bench", help="benchmark an index against exact / ground truth")
    p.add_argument("--in", dest="in_path", required=True)
    p.add_argument("--queries", default=None)
    p.add_argument("--index", default=None, help="the index to benchmark (required here)")
    p.add_argument("--unseen-fraction", type=float, default=None)
    p.add_argument("--k", type=int, default=10)
    p.add_argument("--out", required=True)
    p.set_defaults(func=cmd_bench)
    p = sub.add_parser("inspect", help="summarize a dataset or index file")
    p.add_argument("path")
    p.set_defaults(func=cmd_inspect)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ValidationError, FormatError, OSError, ValueError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
