"""GPU parity at the BASELINE shapes (VERDICT r1 "what's weak" 1).

* Reference golden vectors at every config's d / K / |F| / k / sigma
  (tests/golden/shape_*.npz, made by make_golden_shapes.py from the real
  reference on reference-encoded databases): bitwise LUT (d = 960 is the
  multi-leaf pairwise path), ids, scores, op counts, plus the survivor sets
  against the oracle, through every pipeline mode.
* n >= 2M databases built from the fixtures' reference-encoded rows (the
  code distribution the bench scans): range-major unit order, overflowing
  slices, and the in-order walks, bitwise against the oracle.
* Full BASELINE sizes (c4: 10M, c5: 100M; GPU-encoded synthetic data):
  two-step with sigma = +inf and two-step with the fast set = every book
  must equal the exact engine bitwise (search.py:97-165 degenerate
  equivalences, pkg/tests/test_acceptance.py:78-106), and one query per
  config against the oracle itself.
"""

import numpy as np
import pytest

from _golden import load
from oracle import icq_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1912_08756_b200 as icqb  # noqa: E402
from test_gpu_parity import MODES, _surv_ids  # noqa: E402

SHAPES = ["shape_c1", "shape_c2", "shape_c3", "shape_c4", "shape_c5", "shape_c1_sigma_f32"]


@pytest.mark.parametrize("name", SHAPES)
def test_shape_golden_batched(name):
    """Batched device path == the reference's outputs at the BASELINE shapes."""
    c = load(name)
    dev = icqb.DeviceIndex(c.books, c.codes.astype(np.uint8), c.fast)
    qd = torch.from_numpy(c.queries).cuda()
    lut = dev.build_lut_device(qd).cpu().numpy()
    assert np.array_equal(lut, c.luts), name  # bitwise, d = 96 / 128 / 960
    for r in c.rows:
        if r.is_exact:
            out = dev.search_device(qd[r.query:r.query + 1], r.k, exact=True)
        else:
            sigma = c.sigma if r.sigma is None else r.sigma
            out = dev.search_device(qd[r.query:r.query + 1], r.k, sigma)
        assert np.array_equal(out["ids"][0].cpu().numpy(), r.ids), (name, r.query, r.k, r.sigma)
        assert np.array_equal(out["scores"][0].cpu().numpy(), r.scores)
        assert int(out["refinements"][0]) == r.refinements, (name, r.query, r.k, r.sigma)


@pytest.mark.parametrize("mode", ["filter", "listj", "prolive", "overflow", "rangemajor",
                                  "noties", "countmode"])
@pytest.mark.parametrize("name", ["shape_c2", "shape_c3", "shape_c4", "shape_c5",
                                  "shape_c1_sigma_f32"])
def test_shape_survivors_all_modes(name, mode, monkeypatch):
    for key, val in MODES[mode].items():
        monkeypatch.setenv(key, val)
    c = load(name)
    dev = icqb.DeviceIndex(c.books, c.codes.astype(np.uint8), c.fast)
    qd = torch.from_numpy(c.queries).cuda()
    seen = set()
    for r in c.rows:
        if r.is_exact or (r.k, r.sigma) in seen:
            continue
        seen.add((r.k, r.sigma))
        out = dev.search_device(qd, r.k, r.sigma, survivors=True)
        for i in range(c.queries.shape[0]):
            ref = O.two_step(c.books, c.codes, c.fast, r.sigma, c.queries[i], r.k)
            assert np.array_equal(out["ids"][i].cpu().numpy(), ref.ids), (name, mode, r.k, r.sigma)
            assert np.array_equal(out["scores"][i].cpu().numpy(), ref.scores)
            assert int(out["refinements"][i]) == ref.ops.refinements
            assert np.array_equal(_surv_ids(out["survivors"][i].cpu().numpy(), c.n),
                                  ref.survivors), (name, mode, r.k, r.sigma, i)


def _grown(c, n, seed):
    """n rows drawn from the fixture's reference-encoded rows, 3 % of the
    codes re-drawn (keeps the code statistics, breaks exact duplication)."""
    rng = np.random.default_rng(seed)
    rows = c.codes[rng.integers(0, c.n, size=n)].astype(np.uint8)
    mut = rng.random(rows.shape) < 0.03
    rows[mut] = rng.integers(0, c.m, size=int(mut.sum()), dtype=np.uint8)
    return rows


@pytest.mark.parametrize("name,knobs", [
    ("shape_c5", {}),                                       # default plan
    ("shape_c5", {"ICQ_RANGE_MAJOR": "1", "ICQ_POOL_PAGES": "64"}),  # overflow -> walks
    ("shape_c4", {"ICQ_RANGE_MAJOR": "1"}),
    ("shape_c4", {"ICQ_LIST_J": "8", "ICQ_PRO_MAX": "8192", "ICQ_PRO_MIN": "0"}),
    ("shape_c2", {"ICQ_PRO_LIVE": "1"}),
    ("shape_c5", {"ICQ_COUNT_MODE": "1", "ICQ_RANGE_MAJOR": "1"}),
    ("shape_c4", {"ICQ_COUNT_MODE": "1"}),
    # count mode with an exhausted pool: overflowed slices, walks, new rounds
    ("shape_c4", {"ICQ_COUNT_MODE": "1", "ICQ_POOL_PAGES": "8192"}),
    ("shape_c5", {"ICQ_COUNT_MODE": "1", "ICQ_POOL_PAGES": "4096", "ICQ_WALK_CAP": "65536"}),
    # count mode, few pages per slice: overflowed slices, the slice path of the replay
    ("shape_c5", {"ICQ_COUNT_MODE": "1", "ICQ_MAX_PAGES_CM": "1"}),
    ("shape_c4", {"ICQ_COUNT_MODE": "1", "ICQ_MAX_PAGES_CM": "2", "ICQ_RANGE_MAJOR": "1"}),
    # count-style prologue blocks up to 300k items
    ("shape_c5", {"ICQ_COUNT_MODE": "1", "ICQ_PRO_MAX_CM": "300000"}),
    ("shape_c4", {"ICQ_COUNT_MODE": "1", "ICQ_PRO_MAX_CM": "300000"}),
    # count mode in two rounds (prefix, then the rest)
    ("shape_c5", {"ICQ_COUNT_MODE": "1", "ICQ_CM_PREFIX": "300000"}),
    ("shape_c4", {"ICQ_COUNT_MODE": "1", "ICQ_CM_PREFIX": "500000", "ICQ_CL_CAP": "1000"}),
    ("shape_c4", {"ICQ_COUNT_MODE": "1", "ICQ_CM_PREFIX": "500000", "ICQ_MAX_PAGES_CM": "2"}),
    # count mode for a prefix, list mode for the rest (forced switch at the hand-over)
    ("shape_c5", {"ICQ_COUNT_MODE": "1", "ICQ_CM_PREFIX": "300000", "ICQ_DEBUG": "64"}),
    ("shape_c4", {"ICQ_COUNT_MODE": "1", "ICQ_CM_PREFIX": "500000", "ICQ_DEBUG": "64"}),
    # refine / gather CTAs over groups of 7 ranges
    ("shape_c4", {"ICQ_RANGE_GROUP": "7"}),
    ("shape_c5", {"ICQ_COUNT_MODE": "1", "ICQ_RANGE_GROUP": "7"}),
    # the slice path of the replay
    ("shape_c4", {"ICQ_CL": "0"}),
    ("shape_c5", {"ICQ_CL": "0", "ICQ_RANGE_MAJOR": "1"}),
    # count mode, the contiguous list does not fit: decided from the slices
    ("shape_c4", {"ICQ_COUNT_MODE": "1", "ICQ_CL_CAP": "1000"}),
])
def test_two_million_vs_oracle(name, knobs, monkeypatch):
    for key, val in knobs.items():
        monkeypatch.setenv(key, val)
    c = load(name)
    n = 2_100_000
    codes = _grown(c, n, 7)
    dev = icqb.DeviceIndex(c.books, codes, c.fast)
    Q = c.queries[:2]
    sigmas = sorted({0.0, *(r.sigma for r in c.rows if r.sigma is not None and r.sigma < 10)})
    for k in (10, 100):
        for sigma in sigmas[:3]:
            out = dev.search_device(torch.from_numpy(Q).cuda(), k, sigma, survivors=True)
            for i in range(Q.shape[0]):
                ref = O.two_step(c.books, codes, c.fast, sigma, Q[i], k, chunk=1 << 16)
                assert np.array_equal(out["ids"][i].cpu().numpy(), ref.ids), (name, knobs, k, sigma)
                assert np.array_equal(out["scores"][i].cpu().numpy(), ref.scores)
                assert int(out["refinements"][i]) == ref.ops.refinements
                assert np.array_equal(_surv_ids(out["survivors"][i].cpu().numpy(), n),
                                      ref.survivors), (name, knobs, k, sigma, i)


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_full_size_equivalences(cfg):
    """BASELINE sizes: two-step(sigma=inf) == two-step(fast = all books,
    sigma = 0) == exact, bitwise; one query against the oracle itself."""
    from tools.workloads import CONFIGS, build_database, load_books, queries

    w = CONFIGS[cfg]
    books, _ = load_books(w)
    codes = build_database(w, books, sweeps=2)
    Qd = queries(w)[:4].contiguous()
    fast = np.arange(w.F, dtype=np.uint32)
    dev = icqb.DeviceIndex.from_device(books, codes, fast)
    ex = dev.search_device(Qd, w.k, exact=True)
    inf = dev.search_device(Qd, w.k, float("inf"))
    assert torch.equal(ex["ids"], inf["ids"]) and torch.equal(ex["scores"], inf["scores"])
    assert torch.all(inf["refinements"] == w.n - w.k)
    allf = icqb.DeviceIndex.from_device(books, codes, np.arange(w.K, dtype=np.uint32))
    a = allf.search_device(Qd, w.k, 0.0)
    assert torch.equal(ex["ids"], a["ids"]) and torch.equal(ex["scores"], a["scores"])
    two = dev.search_device(Qd[:1], w.k, 0.0, survivors=True)
    ch = codes.cpu().numpy()
    del codes
    ref = O.two_step(books, ch, fast, 0.0, Qd[0].cpu().numpy(), w.k, chunk=1 << 20)
    assert np.array_equal(two["ids"][0].cpu().numpy(), ref.ids)
    assert np.array_equal(two["scores"][0].cpu().numpy(), ref.scores)
    assert int(two["refinements"][0]) == ref.ops.refinements
    assert np.array_equal(_surv_ids(two["survivors"][0].cpu().numpy(), w.n), ref.survivors)
    ref_ex = O.exact(books, ch, Qd[0].cpu().numpy(), w.k)
    assert np.array_equal(ex["ids"][0].cpu().numpy(), ref_ex.ids)
    assert np.array_equal(ex["scores"][0].cpu().numpy(), ref_ex.scores)
