"""GPU parity: the CUDA path (through the C ABI) vs the reference golden vectors
and vs the oracle.  Everything is bitwise: ids, float64 scores, refinement
counts, op counters, and the survivor (refined-id) sets the reference only
counts (search.py:150)."""

import numpy as np
import pytest

from _golden import CASES, load
from oracle import icq_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1912_08756_b200 as icqb  # noqa: E402


def _surv_ids(bitmap_row, n):
    words = bitmap_row.astype(np.uint32)
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:n]
    return np.flatnonzero(bits)


def _index(c):
    return icqb.SearchIndex(books=c.books, codes=c.codes, xi=np.ones(c.d, dtype=np.uint8),
                            fast=c.fast, sigma=c.sigma,
                            lambdas=np.ones(c.d, dtype=np.float32),
                            cfg=icqb.Config(K=c.K, m=c.m))


@pytest.mark.parametrize("name", CASES)
def test_golden_reference_api(name):
    """Reference-shaped API (one query per call) == real reference outputs."""
    c = load(name)
    idx = _index(c)
    for qi in range(len(c.luts)):
        assert np.array_equal(icqb.build_lut(idx, c.queries[qi]), c.luts[qi])
    for r in c.rows:
        q = c.queries[r.query]
        if r.is_exact:
            got = icqb.search_exact(idx, q, r.k)
        else:
            got = icqb.search_two_step(idx, q, r.k, sigma=r.sigma)
        assert np.array_equal(got.ids, r.ids), (name, r.query, r.k, r.sigma, r.is_exact)
        assert np.array_equal(got.scores, r.scores), (name, r.query, r.k, r.sigma)
        assert got.ops.fast_adds == r.fast_adds
        assert got.ops.exact_adds == r.exact_adds
        assert got.ops.lut_ops == r.lut_ops
        assert got.ops.evaluations == r.evaluations
        assert got.ops.refinements == r.refinements
        assert got.fallback == r.fallback


def _random_case(rng, n, d, K, m, F, dup=False, scale_fast=4.0):
    books = rng.standard_normal((K, m, d)).astype(np.float32)
    books[:F] *= scale_fast
    codes = rng.integers(0, m, size=(n, K)).astype(np.uint8)
    if dup:
        codes[1::2] = codes[0::2]
    fast = np.arange(F, dtype=np.uint32)
    return books, codes, fast


CONFIGS = [
    # n,     d,  K,  m,  F, dup
    (5000, 16, 8, 256, 2, False),
    (5000, 16, 8, 256, 2, True),
    (9000, 12, 16, 256, 4, False),
    (3000, 8, 4, 16, 1, False),
    (2500, 8, 5, 7, 3, True),
    (7000, 20, 8, 256, 8, False),
    (4100, 6, 16, 64, 16, False),
    (20000, 32, 8, 256, 2, False),
    (100000, 16, 16, 256, 4, False),
]

# Pipeline shapes (icq_capi.cu planning knobs, read on every call):
#   default   - the prologue decides small databases alone
#   filter    - 2048-item prologue: the filter kernel lists every item under
#               theta = the live threshold at the prologue end; the replay
#               decides the lists and walks the database in order whenever
#               the live threshold rises above theta
#               (theta = A_J + sigma, A_J the max fast score over the J+1
#               largest heap entries; J the loosest on a ladder whose share
#               of the last prologue items is <= 1/128)
#   listj     - as filter, J = 5 fixed
#   listj0    - as filter, J = 0: theta = the live threshold (most walks)
#   listdiv   - as filter, J chosen for a 1/4 share, 16-page pool: long
#               lists that overflow their slices
#   prolive   - as filter with a 16k-item cap, the prologue stop rule counts
#               items under theta instead of the stale M
#   overflow  - as filter, with a 2-page candidate pool: slices overflow and
#               the replay walks them from the codes
#   subbatch  - as filter, queries in sub-batches of 4
#   rangemajor- as filter, range-major unit order over 32k-item ranges
#   noprep    - as filter, the replay's preparing warps score nothing exactly:
#               warp 0 reads every refined row itself (ICQ_DEBUG bit 1)
#   allexact  - as filter, the preparing warps score every entry (bit 3)
#   noties    - as filter, no tuple-tie rejection in the filter (bit 0)
#   overflow_walk - as overflow, walks flag every item (bit 4)
#   rounds    - as filter, every walk past 1 item stops the query; the next
#               filter/replay round lists its rest (4 rounds, the last unbounded)
#   oneround  - as filter, a single round (walks run to completion)
#   countmode - as filter, every query in count mode (the lists hold only
#               possible insertions; the count kernel tallies refinements
#               and survivor bits from the replay's threshold trajectory)
_F = {"ICQ_PRO_MAX": "2048", "ICQ_PRO_MIN": "0"}
MODES = {
    "default": {},
    "filter": dict(_F),
    "listj": dict(_F, ICQ_LIST_J="5"),
    "listj0": dict(_F, ICQ_LIST_J="0"),
    "listdiv": dict(_F, ICQ_LIST_DIV="4", ICQ_POOL_PAGES="16"),
    "prolive": {"ICQ_PRO_MAX": "16384", "ICQ_PRO_MIN": "0", "ICQ_PRO_LIVE": "1"},
    "overflow": dict(_F, ICQ_POOL_PAGES="2"),
    "subbatch": {"ICQ_PRO_MAX": "4096", "ICQ_PRO_MIN": "0", "ICQ_QBATCH": "4"},
    "rangemajor": dict(_F, ICQ_RANGE_MAJOR="1", ICQ_RANGE_ITEMS="32768"),
    "noprep": dict(_F, ICQ_DEBUG="2"),
    "allexact": dict(_F, ICQ_DEBUG="8"),
    "noties": dict(_F, ICQ_DEBUG="1"),
    "overflow_walk": dict(_F, ICQ_POOL_PAGES="2", ICQ_DEBUG="16"),
    # walks longer than 1 item hand the query to the next filter/replay round
    "rounds": dict(_F, ICQ_WALK_CAP="1", ICQ_ROUNDS="4"),
    "oneround": dict(_F, ICQ_ROUNDS="1"),
    # refinement-heavy path forced on every query: lists of possible
    # insertions only, refinements / survivors from the count kernel
    "countmode": dict(_F, ICQ_COUNT_MODE="1"),
    "countmode_overflow": dict(_F, ICQ_COUNT_MODE="1", ICQ_POOL_PAGES="2"),
    # count mode entered in the prologue: count-style blocks (float32 exact
    # pre-filter, trajectory recorded) up to item 6000 / over the whole database
    "countmode_phase2": dict(_F, ICQ_COUNT_MODE="1", ICQ_PRO_MAX_CM="6000"),
    "countmode_phase2_all": dict(_F, ICQ_COUNT_MODE="1", ICQ_PRO_MAX_CM="1073741824"),
    # count mode in two rounds: the first lists items below 4096 only, its
    # replay hands the rest to the second round (contiguous lists / slices)
    "countmode_prefix": dict(_F, ICQ_COUNT_MODE="1", ICQ_CM_PREFIX="4096"),
    "countmode_prefix_slices": dict(_F, ICQ_COUNT_MODE="1", ICQ_CM_PREFIX="4096", ICQ_CL_CAP="1"),
    # count mode for the prefix, then list mode (the hand-over finds T - Smin
    # unselective; forced here): the count kernel covers [P0, 4096) only
    "countmode_switch": dict(_F, ICQ_COUNT_MODE="1", ICQ_CM_PREFIX="4096", ICQ_DEBUG="64"),
    "countmode_switch_j0": dict(_F, ICQ_COUNT_MODE="1", ICQ_CM_PREFIX="4096", ICQ_DEBUG="64",
                                ICQ_LIST_J="0"),
    # the slice path of the replay (no contiguous lists): list threshold
    # variants, the preparing warps' debug modes, rounds, count mode
    "slices_filter": dict(_F, ICQ_CL="0"),
    "slices_listj0": dict(_F, ICQ_LIST_J="0", ICQ_CL="0"),
    "slices_noprep": dict(_F, ICQ_DEBUG="2", ICQ_CL="0"),
    "slices_allexact": dict(_F, ICQ_DEBUG="8", ICQ_CL="0"),
    "slices_rounds": dict(_F, ICQ_WALK_CAP="1", ICQ_ROUNDS="4", ICQ_CL="0"),
    "slices_countmode": dict(_F, ICQ_COUNT_MODE="1", ICQ_CL="0"),
    # refine / gather CTAs over groups of 3 ranges
    "rangegroup": dict(_F, ICQ_RANGE_ITEMS="32768", ICQ_RANGE_GROUP="3"),
    "countmode_rangegroup": dict(_F, ICQ_COUNT_MODE="1", ICQ_RANGE_ITEMS="32768", ICQ_RANGE_GROUP="3"),
    # count mode with one page per slice: overflowed slices are walked
    "countmode_pages": dict(_F, ICQ_COUNT_MODE="1", ICQ_MAX_PAGES_CM="1"),
    # list mode with one page per slice
    "listpages": dict(_F, ICQ_MAX_PAGES="1", ICQ_LIST_DIV="4"),
    # count mode + overflowed slices whose walks hand the query to new rounds
    # (the later rounds list under T - Smin at the hand-over)
    "countmode_rounds": dict(_F, ICQ_COUNT_MODE="1", ICQ_POOL_PAGES="2", ICQ_WALK_CAP="1",
                             ICQ_ROUNDS="4"),
}


@pytest.mark.parametrize("mode", sorted(MODES))
@pytest.mark.parametrize("cfg", CONFIGS)
def test_random_vs_oracle_with_survivors(cfg, mode, monkeypatch):
    for key, val in MODES[mode].items():
        monkeypatch.setenv(key, val)
    n, d, K, m, F, dup = cfg
    rng = np.random.default_rng(n + d + K + m + F)
    books, codes, fast = _random_case(rng, n, d, K, m, F, dup)
    dev = icqb.DeviceIndex(books, codes, fast)
    Q = rng.standard_normal((6, d))
    qd = torch.from_numpy(Q).cuda()
    for k in (1, 10, 100):
        for sigma in (0.0, 1.0, 25.0, 1e18, np.float32(2.5)):
            out = dev.search_device(qd, k, sigma, survivors=True, stats=True)
            torch.cuda.synchronize()
            ids = out["ids"].cpu().numpy()
            scores = out["scores"].cpu().numpy()
            refine = out["refinements"].cpu().numpy()
            surv = out["survivors"].cpu().numpy()
            for i in range(Q.shape[0]):
                ref = O.two_step(books, codes, fast, sigma, Q[i], k)
                assert np.array_equal(ids[i], ref.ids), (cfg, k, sigma, i)
                assert np.array_equal(scores[i], ref.scores), (cfg, k, sigma, i)
                assert int(refine[i]) == ref.ops.refinements, (cfg, k, sigma, i)
                assert np.array_equal(_surv_ids(surv[i], n), ref.survivors), (cfg, k, sigma, i)
        out = dev.search_device(qd, k, exact=True)
        torch.cuda.synchronize()
        for i in range(Q.shape[0]):
            ref = O.exact(books, codes, Q[i], k)
            assert np.array_equal(out["ids"][i].cpu().numpy(), ref.ids)
            assert np.array_equal(out["scores"][i].cpu().numpy(), ref.scores)


@pytest.mark.parametrize("mode", ["default", "filter"])
def test_large_k_shared_memory_heap(mode, monkeypatch):
    """k > 128: the replay's heap lives in shared memory (WarpHeap smem path)."""
    for key, val in MODES[mode].items():
        monkeypatch.setenv(key, val)
    rng = np.random.default_rng(21)
    books, codes, fast = _random_case(rng, 30000, 12, 8, 256, 2)
    dev = icqb.DeviceIndex(books, codes, fast)
    Q = rng.standard_normal((3, 12))
    for k in (129, 500, 2048):
        for sigma in (0.0, 3.0):
            ids, scores, refine, _ = dev.search_host(Q, k, sigma, exact=False)
            for i in range(Q.shape[0]):
                ref = O.two_step(books, codes, fast, sigma, Q[i], k)
                assert np.array_equal(ids[i], ref.ids), (mode, k, sigma, i)
                assert np.array_equal(scores[i], ref.scores), (mode, k, sigma, i)
                assert int(refine[i]) == ref.ops.refinements, (mode, k, sigma, i)
    with pytest.raises(icqb.UnsupportedError):
        dev.search_host(Q, 2049, 0.0, exact=False)


def test_batch_invariance():
    rng = np.random.default_rng(3)
    books, codes, fast = _random_case(rng, 12000, 16, 8, 256, 2)
    dev = icqb.DeviceIndex(books, codes, fast)
    Q = rng.standard_normal((37, 16))
    ids_all, sc_all, rf_all, _ = dev.search_host(Q, 25, 0.5, exact=False)
    for i in (0, 5, 36):
        ids1, sc1, rf1, _ = dev.search_host(Q[i:i + 1], 25, 0.5, exact=False)
        assert np.array_equal(ids1[0], ids_all[i])
        assert np.array_equal(sc1[0], sc_all[i])
        assert rf1[0] == rf_all[i]


def test_k_equals_n_and_tiny_n():
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 40):
        books, codes, fast = _random_case(rng, n, 4, 3, 4, 2)
        dev = icqb.DeviceIndex(books, codes, fast)
        q = rng.standard_normal((2, 4))
        for k in sorted({1, n}):
            ids, scores, refine, _ = dev.search_host(q, k, 0.0, exact=False)
            for i in range(2):
                ref = O.two_step(books, codes, fast, 0.0, q[i], k)
                assert np.array_equal(ids[i], ref.ids)
                assert np.array_equal(scores[i], ref.scores)


def test_validation_errors():
    rng = np.random.default_rng(9)
    books, codes, fast = _random_case(rng, 100, 4, 3, 4, 1)
    dev = icqb.DeviceIndex(books, codes, fast)
    q = rng.standard_normal((1, 4))
    with pytest.raises(icqb.ValidationError):
        dev.search_host(q, 0, 0.0, exact=False)
    with pytest.raises(icqb.ValidationError):
        dev.search_host(q, 101, 0.0, exact=False)
    with pytest.raises(icqb.ValidationError):
        dev.search_host(q, 3, -1.0, exact=False)
    with pytest.raises(icqb.ValidationError):
        dev.search_host(q, 3, float("nan"), exact=False)
    bad = codes.copy()
    bad[7, 1] = 4
    with pytest.raises(icqb.ValidationError):
        icqb.DeviceIndex(books, bad, fast)
    with pytest.raises(icqb.ValidationError):
        icqb.DeviceIndex(books, codes, np.array([1, 0], dtype=np.uint32))
    # non-finite queries: rejected on the host path, and by the LUT kernel's
    # device check on the device-pointer entry points (search.py:51-52)
    bad_q = q.copy()
    bad_q[0, 2] = np.nan
    with pytest.raises(icqb.ValidationError):
        dev.search_host(bad_q, 3, 0.0, exact=False)
    with pytest.raises(icqb.ValidationError):
        dev.search_device(torch.from_numpy(bad_q).cuda(), 3, 0.0)
    with pytest.raises(icqb.ValidationError):
        dev.build_lut_device(torch.from_numpy(np.full((2, 4), np.inf)).cuda())
    # a later clean call is unaffected (the error word is per call)
    dev.search_device(torch.from_numpy(q).cuda(), 3, 0.0)
    with pytest.raises(icqb.UnsupportedError):
        dev.search_host(q, 3, np.float16(1.0), exact=False)
    with pytest.raises(icqb.UnsupportedError):
        icqb.DeviceIndex(rng.standard_normal((2, 300, 4)).astype(np.float32),
                         rng.integers(0, 300, size=(10, 2)).astype(np.uint32),
                         np.array([0], dtype=np.uint32))


@pytest.mark.parametrize("mode", sorted(MODES))
def test_wide_mode_huge_values(mode, monkeypatch):
    """LUT entries beyond float32 headroom: float64-only path, still exact."""
    for key, val in MODES[mode].items():
        monkeypatch.setenv(key, val)
    rng = np.random.default_rng(11)
    books, codes, fast = _random_case(rng, 3000, 4, 4, 16, 2)
    books[0, 3] = 3e25
    dev = icqb.DeviceIndex(books, codes, fast)
    Q = rng.standard_normal((3, 4))
    ids, scores, refine, _ = dev.search_host(Q, 10, 0.0, exact=False)
    for i in range(3):
        ref = O.two_step(books, codes, fast, 0.0, Q[i], 10)
        assert np.array_equal(ids[i], ref.ids)
        assert np.array_equal(scores[i], ref.scores)
        assert int(refine[i]) == ref.ops.refinements
