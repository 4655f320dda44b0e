"""Pin the CPU oracle (oracle/icq_oracle.py) to the reference's own outputs.

The golden files were produced by calling the real reference
(/root/reference/pkg/src/icq/search.py) — see tests/golden/make_golden.py.
Everything here is bitwise: ids, float64 scores, op counters.
"""

import numpy as np
import pytest

from _golden import CASES, load
from oracle import icq_oracle as O


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(name):
    c = load(name)
    for qi in range(len(c.luts)):
        assert np.array_equal(O.lut(c.books, c.queries[qi]), c.luts[qi])
    for r in c.rows:
        q = c.queries[r.query]
        if r.is_exact:
            got = O.exact(c.books, c.codes, q, r.k)
        else:
            sigma = c.sigma if r.sigma is None else r.sigma
            got = O.two_step(c.books, c.codes, c.fast, sigma, q, r.k)
            if not got.fallback:
                assert got.survivors.size == r.refinements
                assert np.all(np.diff(got.survivors) > 0)
        assert np.array_equal(got.ids, r.ids), (name, r.query, r.k, r.sigma)
        assert np.array_equal(got.scores, r.scores), (name, r.query, r.k, r.sigma)
        assert got.ops.fast_adds == r.fast_adds
        assert got.ops.exact_adds == r.exact_adds
        assert got.ops.lut_ops == r.lut_ops
        assert got.ops.evaluations == r.evaluations
        assert got.ops.refinements == r.refinements
        assert got.fallback == r.fallback


@pytest.mark.parametrize("name", ["small_k4m6_prune", "dups_k3m4", "trained_k8f2", "odd_k5m7"])
def test_chunked_replay_equals_literal_loop(name):
    c = load(name)
    for sigma in (0.0, c.sigma, 0.7, 3.0, 1e18):
        for qi in range(min(3, len(c.queries))):
            for k in (1, 5, 37):
                if k > c.n:
                    continue
                a = O.two_step(c.books, c.codes, c.fast, sigma, c.queries[qi], k, chunk=97)
                b = O.two_step_loop(c.books, c.codes, c.fast, sigma, c.queries[qi], k)
                assert np.array_equal(a.ids, b.ids)
                assert np.array_equal(a.scores, b.scores)
                assert np.array_equal(a.survivors, b.survivors)


def test_pairwise_sum_is_numpy_order():
    rng = np.random.default_rng(7)
    for n in [1, 2, 3, 7, 8, 9, 15, 16, 17, 24, 96, 127, 128, 129, 200, 255, 256, 300, 960]:
        a = rng.standard_normal((8, n)) ** 2 * rng.uniform(0.1, 100.0, size=(8, 1))
        s = a.sum(axis=1)
        for i in range(8):
            assert O.pairwise_sum(a[i]) == s[i], n


def test_pairwise_leaves_cover():
    for n in [1, 8, 128, 129, 256, 960, 1000, 4096]:
        prog = O.pairwise_leaves(n)
        leaves = [p for p in prog if p[0] == "leaf"]
        assert sum(p[2] for p in leaves) == n
        assert all(p[2] <= 128 for p in leaves)
        assert len(prog) == 2 * len(leaves) - 1


def test_gathered_row_sum_order_rule():
    """The order the CUDA kernels mirror (icq_device.cuh ref_row_sum): numpy's
    gathered (n, t) score array (search.py:94) is F-contiguous for n >= 2, so
    rows accumulate sequentially in book order; for n == 1 it is pairwise."""
    rng = np.random.default_rng(1)
    for K in (8, 9, 12, 16):
        table = rng.standard_normal((K, 256)) ** 2 * 100
        for n in (1, 2, 3, 17, 1000):
            codes = rng.integers(0, 256, size=(n, K)).astype(np.uint32)
            for books in (np.arange(K), np.arange(K)[::2].copy()):
                g = table[books[None, :], codes[:, books]]
                got = O.gather(table, codes, books)
                for i in range(n):
                    if n == 1:
                        want = O.pairwise_sum(g[i])
                    else:
                        want = 0.0
                        for x in g[i]:
                            want += float(x)
                    assert got[i] == want, (K, n, len(books))
