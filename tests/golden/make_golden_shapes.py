"""Golden vectors at the BASELINE shapes, from the REAL reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden_shapes.py

For every BASELINE config (c1..c5: d in {96, 128, 960}, (K, |F|) in
{(8, 2), (16, 4)}) this takes the reference-trained books committed under
bench_data/, draws a seeded database sample of the config's distribution
(tools/workloads.py), encodes it with the reference encoder
(icq.train.assign_codes, train.py:196-243), and stores the reference's
build_lut / search_two_step / search_exact outputs for a few queries at
k in {10, 100} and sigma in {0, mean lambda, 4 mean lambda, learned}.  The
database is a sample (n = 20k) of the config's size so that the reference
finishes here; the GPU tests cover the full sizes through oracle
comparisons (tests/test_gpu_shapes.py).

One extra case passes sigma as np.float32 (numpy 2 promotion of
``bound + sigma``, search.py:149).
"""

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from icq import CodebookSet, CodeMatrix, Config, SearchIndex  # noqa: E402  (reference)
from icq.search import build_lut, search_exact, search_two_step  # noqa: E402
from icq.train import assign_codes  # noqa: E402

from tools.workloads import CONFIGS, load_books, sample_numpy  # noqa: E402

N_SAMPLE = 20_000
SEED = 2024


def save_case(name, index, queries, ks, sigmas, f32=False):
    rows, out = [], {}
    for qi, q in enumerate(queries):
        for k in ks:
            for s in sigmas:
                sig = np.float32(s) if f32 else s
                two = search_two_step(index, q, k, sigma=sig)
                rows.append((qi, k, float(sig), 0, int(f32)))
                i = len(rows) - 1
                out[f"r{i}_ids"], out[f"r{i}_scores"] = two.ids, two.scores
                out[f"r{i}_ops"] = np.array(
                    [two.ops.fast_adds, two.ops.exact_adds, two.ops.lut_ops,
                     two.ops.evaluations, two.ops.refinements, int(two.fallback)], dtype=np.int64)
            ex = search_exact(index, q, k)
            rows.append((qi, k, 0.0, 1, 0))
            i = len(rows) - 1
            out[f"r{i}_ids"], out[f"r{i}_scores"] = ex.ids, ex.scores
            out[f"r{i}_ops"] = np.array(
                [ex.ops.fast_adds, ex.ops.exact_adds, ex.ops.lut_ops,
                 ex.ops.evaluations, ex.ops.refinements, int(ex.fallback)], dtype=np.int64)
    luts = np.stack([build_lut(index, q) for q in queries])
    np.savez_compressed(
        HERE / f"{name}.npz",
        books=index.books.codewords.astype(np.float32),
        codes=index.codes.codes.astype(np.uint8),
        fast=index.fast.astype(np.uint32),
        sigma=np.float64(index.sigma),
        queries=np.asarray(queries, dtype=np.float64),
        rows=np.array(rows, dtype=np.float64),  # (query, k, sigma|-1, is_exact, sigma_f32)
        luts=luts,
        **out,
    )
    print(f"{name}: n={index.n} d={index.d} K={index.cfg.K} F={index.fast.size} "
          f"rows={len(rows)}", flush=True)


def main(names):
    for name in names:
        w = CONFIGS[name]
        books, meta = load_books(w)
        rng = np.random.default_rng(SEED + int(name[1:]))
        x = sample_numpy(w, N_SAMPLE, rng)
        t0 = time.time()
        codes = assign_codes(x, books).codes  # reference ICM, default sweeps
        te = time.time() - t0
        lam = np.asarray(meta["lambdas"], dtype=np.float64)
        learned = float(meta["learned_sigma"])
        index = SearchIndex(books=CodebookSet(books), codes=CodeMatrix(codes),
                            xi=np.ones(w.d, dtype=np.uint8),
                            fast=np.arange(w.F, dtype=np.uint32), sigma=learned,
                            lambdas=np.asarray(meta["lambdas"], dtype=np.float32),
                            cfg=Config(K=w.K, m=256))
        q = sample_numpy(w, 3, rng).astype(np.float64)
        sigmas = sorted({0.0, float(lam.mean()), 4.0 * float(lam.mean()), learned})
        ks = [10, 100]
        save_case(f"shape_{name}", index, q, ks, sigmas)
        print(f"  encode {te:.0f}s, sigmas {sigmas}", flush=True)
        if name == "c1":
            save_case("shape_c1_sigma_f32", index, q[:2], [10, 100],
                      [0.0, float(lam.mean()), 0.37, 4.0 * float(lam.mean())], f32=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c4", "c5", "c3"])
