"""Generate golden vectors from the REAL reference implementation.

Run in the build container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Every case builds a reference ``icq.SearchIndex`` (the index shapes and
fixture builder follow the reference's own tests: ``pkg/tests/conftest.py``
``build_index`` and ``pkg/tests/test_search.py``), calls the reference's
``build_lut`` / ``search_two_step`` / ``search_exact`` and stores inputs and
outputs in ``tests/golden/<case>.npz``.  The oracle and the GPU path are then
checked against these files bit for bit.
"""

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

import icq  # noqa: E402  (reference, from /root/reference/pkg/src)
from icq import CodebookSet, CodeMatrix, Config, SearchIndex  # noqa: E402
from icq.search import build_lut, search_exact, search_two_step  # noqa: E402
from icq.train import assign_codes, fast_set, _init_books  # noqa: E402
from conftest import build_index  # noqa: E402  (reference pkg/tests/conftest.py)

SIGMA_DEFAULT = -1.0  # marker: use the index margin (sigma=None)


def _with(index, **kw):
    f = dict(books=index.books, codes=index.codes, xi=index.xi, fast=index.fast,
             sigma=index.sigma, lambdas=index.lambdas, cfg=index.cfg)
    f.update(kw)
    return SearchIndex(**f)


def save_case(name, index, queries, ks, sigmas):
    books = index.books.codewords.astype(np.float32)
    codes = index.codes.codes
    rows = []
    out = {}
    for qi, q in enumerate(queries):
        for k in ks:
            for s in sigmas:
                sig = None if s == SIGMA_DEFAULT else s
                two = search_two_step(index, q, k, sigma=sig)
                rows.append((qi, k, s, 0))
                out[f"r{len(rows)-1}_ids"] = two.ids
                out[f"r{len(rows)-1}_scores"] = two.scores
                out[f"r{len(rows)-1}_ops"] = np.array(
                    [two.ops.fast_adds, two.ops.exact_adds, two.ops.lut_ops,
                     two.ops.evaluations, two.ops.refinements, int(two.fallback)], dtype=np.int64)
            ex = search_exact(index, q, k)
            rows.append((qi, k, 0.0, 1))
            out[f"r{len(rows)-1}_ids"] = ex.ids
            out[f"r{len(rows)-1}_scores"] = ex.scores
            out[f"r{len(rows)-1}_ops"] = np.array(
                [ex.ops.fast_adds, ex.ops.exact_adds, ex.ops.lut_ops,
                 ex.ops.evaluations, ex.ops.refinements, int(ex.fallback)], dtype=np.int64)
    luts = np.stack([build_lut(index, q) for q in queries[:2]])
    np.savez_compressed(
        HERE / f"{name}.npz",
        books=books,
        codes=codes.astype(np.uint8 if index.cfg.m <= 256 else np.uint32),
        fast=index.fast.astype(np.uint32),
        sigma=np.float64(index.sigma),
        queries=np.asarray(queries, dtype=np.float64),
        rows=np.array(rows, dtype=np.float64),  # (query, k, sigma|-1, is_exact)
        luts=luts,
        **out,
    )
    print(f"{name}: n={index.n} d={index.d} K={index.cfg.K} m={index.cfg.m} "
          f"F={index.fast.size} rows={len(rows)}")


def tiny_index():
    """test_search.py:23-41 worked example."""
    books = np.array([[[0.0, 0.0], [1.0, 0.0]], [[0.0, 0.0], [0.0, 1.0]]], dtype=np.float32)
    codes = np.array([[1, 1], [0, 0], [1, 0]], dtype=np.uint32)
    return SearchIndex(books=CodebookSet(books), codes=CodeMatrix(codes),
                       xi=np.array([1, 0], dtype=np.uint8), fast=np.array([0], dtype=np.uint32),
                       sigma=0.5, lambdas=np.array([1.0, 1.0], dtype=np.float32),
                       cfg=Config(K=2, m=2))


def gmm(rng, n, means, std):
    lab = rng.integers(0, means.shape[0], size=n)
    return (means[lab] + std * rng.standard_normal((n, means.shape[1]))).astype(np.float32)


def trained_index(rng, n, d, K, F, m=256, ntrain=4000, sweeps=3):
    """Residual k-means books (reference _init_books, train.py:130-140) and
    reference ICM codes (assign_codes, train.py:196-243); fast = first F books."""
    means = rng.standard_normal((16, d))
    x = gmm(rng, n, means, 0.3)
    books = _init_books(x[:ntrain].astype(np.float64), K, m, rng).astype(np.float32)
    codes = assign_codes(x, books, max_sweeps=sweeps).codes
    lam = x.var(axis=0).astype(np.float32)
    return SearchIndex(books=CodebookSet(books), codes=CodeMatrix(codes),
                       xi=np.ones(d, dtype=np.uint8), fast=np.arange(F, dtype=np.uint32),
                       sigma=0.0, lambdas=lam, cfg=Config(K=K, m=m)), means


def main():
    rng = np.random.default_rng(42)
    save_case("tiny", tiny_index(), np.array([[1.0, 1.0], [0.2, -0.3]]), [1, 2, 3],
              [SIGMA_DEFAULT, 0.0, 1e18])

    idx = build_index(rng, n=120, d=8, K=4, m=5)
    save_case("small_k4m5", idx, rng.normal(size=(6, 8)), [1, 7],
              [SIGMA_DEFAULT, 0.0, 1e18])

    idx = build_index(rng, n=300, d=8, K=4, m=6, sigma=0.1)
    save_case("small_k4m6_prune", idx, rng.normal(size=(6, 8)), [5, 9],
              [SIGMA_DEFAULT, 0.0, 0.3])

    idx = build_index(rng, n=100, d=6, K=3, m=4)
    codes = idx.codes.codes.copy()
    codes[1::2] = codes[0::2]
    idx = _with(idx, codes=CodeMatrix(codes))
    save_case("dups_k3m4", idx, rng.normal(size=(6, 6)), [11, 20],
              [SIGMA_DEFAULT, 0.0, 1e18])

    idx = build_index(rng, n=80, d=8, K=3, m=4, xi=np.zeros(8, dtype=np.uint8))
    assert idx.fast.size == 0
    save_case("empty_fast", idx, rng.normal(size=(3, 8)), [6], [SIGMA_DEFAULT])

    idx = build_index(rng, n=40, d=8, K=3, m=4)
    save_case("k_eq_n", idx, rng.normal(size=(3, 8)), [40], [1e18, 0.0])

    idx = build_index(rng, n=257, d=5, K=5, m=7, sigma=0.2)
    save_case("odd_k5m7", idx, rng.normal(size=(4, 5)), [1, 13], [SIGMA_DEFAULT, 0.0])

    # reference-trained books + reference ICM codes (the bench's code distribution)
    idx, means = trained_index(rng, n=12000, d=32, K=8, F=2)
    q = gmm(rng, 6, means, 0.3)
    save_case("trained_k8f2", idx, q, [10, 100], [0.0, 1.0, 4.0])
    all_fast = _with(idx, fast=np.arange(8, dtype=np.uint32), sigma=0.0)
    save_case("trained_k8_allfast", all_fast, q[:3], [10], [0.0])

    idx, means = trained_index(rng, n=6000, d=24, K=16, F=4, ntrain=3000, sweeps=2)
    q = gmm(rng, 4, means, 0.3)
    save_case("trained_k16f4", idx, q, [10, 100], [0.0, 2.0])

    # n == 1: numpy's gathered (1, K) array is C-contiguous, so the row sums
    # run numpy's pairwise kernel instead of the column-sequential order
    for K, F in ((9, 8), (16, 12)):
        books = (rng.standard_normal((K, 5, 3)) * 7).astype(np.float32)
        idx = SearchIndex(books=CodebookSet(books),
                          codes=CodeMatrix(rng.integers(0, 5, size=(1, K))),
                          xi=np.ones(3, dtype=np.uint8), fast=np.arange(F, dtype=np.uint32),
                          sigma=0.0, lambdas=np.ones(3, dtype=np.float32), cfg=Config(K=K, m=5))
        save_case(f"single_k{K}", idx, rng.normal(size=(3, 3)) * 5, [1], [0.0, 1e18])


if __name__ == "__main__":
    sys.exit(main())
