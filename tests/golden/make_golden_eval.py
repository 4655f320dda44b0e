"""Golden outputs of the reference's benchmark driver and CLI (query side).

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden_eval.py

Builds a small reference-encoded index over a labeled Gaussian-mixture
dataset, writes the index / dataset / query files with the reference's own
writers (save_index, save_dataset: data.py:266-322), and records:
* run_benchmark (evaluate.py:106-187) reports as CSV, truth "brute" and
  "labels", sigma None and 0.0, k 10 and 25;
* `icq search` (cli.py:135-162) CSV outputs for --mode two-step / exact /
  brute and --sigma-scale;
* `icq inspect` stdout for the index and the dataset.
The GPU tests replay the same files through paper_1912_08756_b200 and require
byte-identical outputs.
"""

import contextlib
import io
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

from icq import (CodebookSet, CodeMatrix, Config, EmbeddedDataset, SearchIndex,  # noqa: E402
                 save_dataset, save_index)
from icq.cli import main as icq_main  # noqa: E402
from icq.evaluate import run_benchmark  # noqa: E402
from icq.train import _init_books, assign_codes  # noqa: E402


def main():
    rng = np.random.default_rng(77)
    n, d, K, m, F, nq = 3000, 16, 4, 16, 2, 24
    means = rng.standard_normal((6, d)) * 2.0
    lab = rng.integers(0, 6, size=n + nq)
    x = (means[lab] + 0.5 * rng.standard_normal((n + nq, d))).astype(np.float32)
    data = EmbeddedDataset(x[:n], lab[:n])
    queries = EmbeddedDataset(x[n:], lab[n:])
    books = _init_books(x[:1000].astype(np.float64), K, m, rng).astype(np.float32)
    codes = assign_codes(x[:n], books).codes
    xi = np.zeros(d, dtype=np.uint8)
    xi[: d // 2] = 1
    lam = x[:n].var(axis=0).astype(np.float32)
    index = SearchIndex(books=CodebookSet(books), codes=CodeMatrix(codes), xi=xi,
                        fast=np.arange(F, dtype=np.uint32), sigma=0.75, lambdas=lam,
                        cfg=Config(K=K, m=m, epochs=3, seed=11))
    out = {}
    for truth in ("brute", "labels"):
        for sigma in (None, 0.0):
            for k in (10, 25):
                rep = run_benchmark(index, data, queries, truth=truth, k=k, sigma=sigma)
                out[f"bench_{truth}_{'none' if sigma is None else 'zero'}_k{k}"] = rep.to_csv()
    with tempfile.TemporaryDirectory() as td:
        t = Path(td)
        save_index(index, t / "i.icqi")
        save_dataset(data, t / "d.icqd")
        save_dataset(queries, t / "q.icqd")
        files = {nm: np.frombuffer((t / nm).read_bytes(), dtype=np.uint8)
                 for nm in ("i.icqi", "d.icqd", "q.icqd")}
        runs = {
            "search_two": ["--index", str(t / "i.icqi"), "--k", "7"],
            "search_two_scale": ["--index", str(t / "i.icqi"), "--k", "7", "--sigma-scale", "0.25"],
            "search_exact": ["--index", str(t / "i.icqi"), "--k", "7", "--mode", "exact"],
            "search_brute": ["--data", str(t / "d.icqd"), "--k", "7", "--mode", "brute"],
        }
        for name, extra in runs.items():
            dst = t / f"{name}.csv"
            with contextlib.redirect_stderr(io.StringIO()):
                rc = icq_main(["search", "--queries", str(t / "q.icqd"), "--out", str(dst), *extra])
            assert rc == 0, name
            out[name] = dst.read_text()
        for name, path in (("inspect_index", t / "i.icqi"), ("inspect_data", t / "d.icqd")):
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(io.StringIO()):
                assert icq_main(["inspect", str(path)]) == 0
            out[name] = buf.getvalue()
    np.savez_compressed(HERE / "eval_cli.npz", **{f"file_{k}": v for k, v in files.items()},
                        **{k: np.array(v) for k, v in out.items()})
    print("eval_cli:", sorted(out))


if __name__ == "__main__":
    sys.exit(main())
