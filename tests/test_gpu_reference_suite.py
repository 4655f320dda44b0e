"""The reference's own query-path tests, restated against the B200 package.

The reference package does not travel to the GPU box (it is Python, read
from /root/reference only in the build container), so its test cases are
restated here, one function per reference test, with the reference's
fixture builder (pkg/tests/conftest.py:9-36, ``build_index``) restated as
``_build_index``.  Sources:
  pkg/tests/test_search.py:23-236   (scoring, exact, two-step, brute force)
  pkg/tests/test_acceptance.py:78-106 (test_01: all books fast + sigma 0 ==
                                       exact, 1000 queries, bitwise)
  pkg/tests/test_data.py:121-132    (save/load round trip answers identically)
  pkg/tests/test_evaluate.py:102-106 (thread-pool report == serial report)
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1912_08756_b200 as icq  # noqa: E402  (the drop-in, under the reference's name)


def _fast_set(books, xi):
    """train.py:246-253 fast_set: books whose every codeword has strictly more
    mass inside the mask than outside (an all-zero codeword keeps it out)."""
    b = np.asarray(books, dtype=np.float64)
    x = np.asarray(xi).astype(bool)
    sq = b ** 2
    inside = np.sqrt(sq[:, :, x].sum(axis=2)) if x.any() else np.zeros(b.shape[:2])
    outside = np.sqrt(sq[:, :, ~x].sum(axis=2)) if (~x).any() else np.zeros(b.shape[:2])
    return np.flatnonzero(np.all(outside < inside, axis=1)).astype(np.uint32)


def _build_index(rng, n=60, d=8, K=3, m=4, xi=None, sigma=0.5):
    books = rng.standard_normal((K, m, d)).astype(np.float32)
    codes = rng.integers(0, m, size=(n, K))
    if xi is None:
        xi = (rng.random(d) < 0.5).astype(np.uint8)
    if xi.any():
        boost = np.where(xi.astype(bool), 10.0, 1.0).astype(np.float32)
        books[: max(1, K // 2)] *= boost
    return icq.SearchIndex(books=icq.CodebookSet(books), codes=icq.CodeMatrix(codes), xi=xi,
                           fast=_fast_set(books, xi), sigma=sigma,
                           lambdas=np.abs(rng.standard_normal(d)).astype(np.float32),
                           cfg=icq.Config(K=K, m=m))


def _with_codes(index, codes):
    return icq.SearchIndex(books=index.books, codes=icq.CodeMatrix(codes), xi=index.xi,
                           fast=index.fast, sigma=index.sigma, lambdas=index.lambdas,
                           cfg=index.cfg)


@pytest.fixture
def rng():
    return np.random.default_rng(42)


def _tiny():
    books = np.array([[[0.0, 0.0], [1.0, 0.0]], [[0.0, 0.0], [0.0, 1.0]]], dtype=np.float32)
    return icq.SearchIndex(books=icq.CodebookSet(books),
                           codes=icq.CodeMatrix(np.array([[1, 1], [0, 0], [1, 0]], dtype=np.uint32)),
                           xi=np.array([1, 0], dtype=np.uint8), fast=np.array([0], dtype=np.uint32),
                           sigma=0.5, lambdas=np.array([1.0, 1.0], dtype=np.float32),
                           cfg=icq.Config(K=2, m=2))


# -- test_search.py TestScoring ------------------------------------------------
def test_lut_worked_example():
    ops = icq.OpCounter()
    lut = icq.build_lut(_tiny(), np.array([1.0, 1.0]), ops)
    assert np.array_equal(lut, [[2.0, 1.0], [2.0, 1.0]])
    assert ops.lut_ops == 8


def test_exact_and_fast_scores():
    idx = _tiny()
    lut = icq.build_lut(idx, np.array([1.0, 1.0]))
    ops = icq.OpCounter()
    assert icq.exact_score(lut, np.array([1, 1]), ops) == 2.0
    assert icq.exact_score(lut, np.array([0, 0]), ops) == 4.0
    assert ops.exact_adds == 2
    assert icq.fast_score(lut, np.array([1, 1]), idx.fast, ops) == 1.0
    assert ops.fast_adds == 0


def test_score_is_reconstruction_distance_plus_query_norms(rng):
    books = np.zeros((2, 3, 4), dtype=np.float32)
    books[0, :, :2] = rng.normal(size=(3, 2))
    books[1, :, 2:] = rng.normal(size=(3, 2))
    idx = icq.SearchIndex(books=books, codes=np.zeros((1, 2), dtype=np.uint32),
                          xi=np.ones(4, dtype=np.uint8), fast=np.array([0], dtype=np.uint32),
                          sigma=0.0, lambdas=np.ones(4, dtype=np.float32), cfg=icq.Config(K=2, m=3))
    q = rng.normal(size=4)
    lut = icq.build_lut(idx, q)
    for c0 in range(3):
        for c1 in range(3):
            recon = books[0, c0].astype(np.float64) + books[1, c1].astype(np.float64)
            want = float(((q - recon) ** 2).sum()) + float((q ** 2).sum())
            assert icq.exact_score(lut, np.array([c0, c1])) == pytest.approx(want, rel=1e-9)


# -- TestExactEngine -------------------------------------------------------------
def test_exact_matches_naive_ranking(rng):
    idx = _build_index(rng, n=80, d=6, K=3, m=4)
    q = rng.normal(size=6)
    lut = icq.build_lut(idx, q)
    naive = np.array([icq.exact_score(lut, row) for row in idx.codes.codes])
    res = icq.search_exact(idx, q, k=10)
    order = np.lexsort((np.arange(idx.n), naive))[:10]
    assert np.array_equal(res.ids, order)
    assert np.array_equal(res.scores, naive[order])


def test_exact_op_accounting(rng):
    idx = _build_index(rng, n=50, d=6, K=3, m=4)
    res = icq.search_exact(idx, rng.normal(size=6), k=5)
    assert (res.ops.exact_adds, res.ops.fast_adds, res.ops.lut_ops, res.ops.evaluations) == (
        100, 0, 72, 50)
    assert res.ops.total_adds == res.ops.exact_adds


def test_exact_ties_are_id_ordered(rng):
    idx = _build_index(rng, n=60, d=6, K=3, m=4)
    codes = idx.codes.codes.copy()
    codes[1::2] = codes[0::2]
    res = icq.search_exact(_with_codes(idx, codes), rng.normal(size=6), k=20)
    assert np.all(np.diff(res.scores) >= 0)
    for i in range(19):
        if res.scores[i] == res.scores[i + 1]:
            assert res.ids[i] < res.ids[i + 1]


def test_exact_k_bounds_and_query_validation(rng):
    idx = _build_index(rng, n=20)
    q = rng.normal(size=8)
    for bad in (0, 21):
        with pytest.raises(icq.ValidationError):
            icq.search_exact(idx, q, k=bad)
    assert icq.search_exact(idx, q, k=20).ids.size == 20
    with pytest.raises(icq.ValidationError):
        icq.search_exact(idx, np.zeros(7), k=1)
    with pytest.raises(icq.ValidationError):
        icq.search_exact(idx, np.full(8, np.nan), k=1)


# -- TestTwoStepEngine -----------------------------------------------------------
def test_huge_sigma_reproduces_exact(rng):
    idx = _build_index(rng, n=120, d=8, K=4, m=5)
    for _ in range(20):
        q = rng.normal(size=8)
        want = icq.search_exact(idx, q, k=7)
        got = icq.search_two_step(idx, q, k=7, sigma=1e18)
        assert np.array_equal(got.ids, want.ids) and np.array_equal(got.scores, want.scores)
        assert got.ops.refinements == idx.n - 7


def test_tie_ordering_matches_exact_under_duplicates(rng):
    idx = _build_index(rng, n=100, d=6, K=3, m=4)
    codes = idx.codes.codes.copy()
    codes[1::2] = codes[0::2]
    idx = _with_codes(idx, codes)
    for _ in range(20):
        q = rng.normal(size=6)
        assert np.array_equal(icq.search_two_step(idx, q, k=11, sigma=1e18).ids,
                              icq.search_exact(idx, q, k=11).ids)


def test_small_sigma_result_is_well_formed(rng):
    idx = _build_index(rng, n=150, d=8, K=4, m=5)
    res = icq.search_two_step(idx, rng.normal(size=8), k=10, sigma=0.0)
    assert res.ids.size == 10 and np.unique(res.ids).size == 10
    assert np.all(np.diff(res.scores) >= 0) and not res.fallback


def test_pruning_reduces_exact_evaluations(rng):
    idx = _build_index(rng, n=300, d=8, K=4, m=6, sigma=0.1)
    q = rng.normal(size=8)
    res = icq.search_two_step(idx, q, k=5)
    assert res.ops.refinements < idx.n - 5
    assert res.ops.exact_adds < icq.search_exact(idx, q, k=5).ops.exact_adds


def test_refinements_bounded_and_saturate(rng):
    idx = _build_index(rng, n=200, d=8, K=4, m=5)
    q = rng.normal(size=8)
    lo = icq.search_two_step(idx, q, 9, sigma=0.0).ops.refinements
    hi = icq.search_two_step(idx, q, 9, sigma=1e18).ops.refinements
    assert 0 <= lo <= hi == idx.n - 9


def test_two_step_op_accounting(rng):
    idx = _build_index(rng, n=150, d=8, K=4, m=5, sigma=0.3)
    res = icq.search_two_step(idx, rng.normal(size=8), 6)
    f = idx.fast.size
    assert res.ops.lut_ops == 4 * 5 * 8
    assert res.ops.fast_adds == (f - 1) * idx.n
    assert res.ops.exact_adds == 3 * (res.ops.refinements + 6)
    assert res.ops.evaluations == idx.n
    assert res.ops.total_adds == res.ops.fast_adds + res.ops.exact_adds


def test_default_sigma_and_negative_sigma(rng):
    idx = _build_index(rng, n=100, d=8, K=3, m=4, sigma=0.25)
    q = rng.normal(size=8)
    assert np.array_equal(icq.search_two_step(idx, q, k=5).ids,
                          icq.search_two_step(idx, q, k=5, sigma=0.25).ids)
    with pytest.raises(icq.ValidationError):
        icq.search_two_step(idx, q, k=3, sigma=-1.0)


def test_empty_fast_set_falls_back_to_exact(rng):
    idx = _build_index(rng, n=80, d=8, K=3, m=4, xi=np.zeros(8, dtype=np.uint8))
    assert idx.fast.size == 0
    q = rng.normal(size=8)
    res = icq.search_two_step(idx, q, k=6)
    assert res.fallback and np.array_equal(res.ids, icq.search_exact(idx, q, k=6).ids)


def test_k_equals_n(rng):
    idx = _build_index(rng, n=40, d=8, K=3, m=4)
    res = icq.search_two_step(idx, rng.normal(size=8), k=40, sigma=1e18)
    assert np.array_equal(np.sort(res.ids), np.arange(40))


# -- TestBruteforce ----------------------------------------------------------------
def test_bruteforce_matches_direct_distances(rng):
    x = rng.normal(size=(50, 5)).astype(np.float32)
    q = rng.normal(size=5)
    res = icq.search_bruteforce(icq.EmbeddedDataset(x), q, k=7)
    d2 = ((x.astype(np.float64) - q) ** 2).sum(axis=1)
    order = np.lexsort((np.arange(50), d2))[:7]
    assert np.array_equal(res.ids, order) and np.array_equal(res.scores, d2[order])
    assert res.ops.exact_adds == 4 * 50


# -- test_acceptance.py test_01 ----------------------------------------------------
def test_01_all_books_fast_zero_margin_equals_exact():
    """n=10k, d=64, K=8, m=256: 1000 queries, identical ids, bitwise scores."""
    rng = np.random.default_rng(0)
    books = rng.standard_normal((8, 256, 64)).astype(np.float32)
    codes = rng.integers(0, 256, size=(10_000, 8))
    idx = icq.SearchIndex(books=books, codes=codes, xi=np.ones(64, dtype=np.uint8),
                          fast=np.arange(8, dtype=np.uint32), sigma=0.0,
                          lambdas=np.ones(64, dtype=np.float32), cfg=icq.Config(K=8, m=256))
    Q = rng.standard_normal((1000, 64))
    two = icq.search_two_step_batch(idx, Q, 10, sigma=0.0)
    ex = icq.search_exact_batch(idx, Q, 10)
    assert np.array_equal(two.ids, ex.ids) and np.array_equal(two.scores, ex.scores)
    for qi in (0, 499, 999):  # the per-query reference-shaped calls agree too
        a, b = icq.search_two_step(idx, Q[qi], 10), icq.search_exact(idx, Q[qi], 10)
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.scores, b.scores)


# -- test_data.py:121-132 ----------------------------------------------------------
def test_roundtrip_search_identical(tmp_path, rng):
    idx = _build_index(rng, n=80, d=7, K=3, m=6)
    path = tmp_path / "i.icqi"
    icq.save_index(idx, path)
    loaded = icq.load_index(path)
    for _ in range(100):
        q = rng.standard_normal(7)
        a, b = icq.search_exact(idx, q, 5), icq.search_exact(loaded, q, 5)
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.scores, b.scores)
        a, b = icq.search_two_step(idx, q, 5), icq.search_two_step(loaded, q, 5)
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.scores, b.scores)


# -- test_evaluate.py:102-106 -------------------------------------------------------
def test_thread_pool_matches_serial(rng):
    idx = _build_index(rng, n=200, d=6, K=3, m=4)
    x = rng.normal(size=(200, 6)).astype(np.float32)
    queries = rng.normal(size=(6, 6))
    ds = icq.EmbeddedDataset(x)
    assert icq.run_benchmark(idx, ds, queries, k=5) == icq.run_benchmark(idx, ds, queries, k=5,
                                                                         threads=3)
