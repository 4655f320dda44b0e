"""GPU ICM encoder against the reference's assign_codes
(train.py:196-243) on golden cases made by tests/golden/make_golden_encode.py.

The reference's dgemm sums the dot products in its own blocked order, the
kernel in d order; both are float64, so codes may differ only where two
codewords tie to rounding.  Each differing row must reconstruct its vector
as well as the reference's codes do (to 1e-9 relative) and such rows must be
rare (<= 0.5 %)."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1912_08756_b200 as icqb  # noqa: E402

Z = np.load(Path(__file__).parent / "golden" / "encode_cases.npz")
CASES = sorted({k.split("_")[0] for k in Z.files})


def _loss(x, books, codes):
    b = books.astype(np.float64)
    recon = np.zeros((x.shape[0], b.shape[2]))
    for k in range(b.shape[0]):
        recon += b[k][codes[:, k].astype(np.int64)]
    return ((x.astype(np.float64) - recon) ** 2).sum(axis=1)


@pytest.mark.parametrize("case", CASES)
def test_codes_match_reference(case):
    x, books, want = Z[f"{case}_x"], Z[f"{case}_books"], Z[f"{case}_codes"]
    start = Z[f"{case}_start"] if f"{case}_start" in Z.files else None
    got = icqb.assign_codes(x, books, codes=start, max_sweeps=int(Z[f"{case}_sweeps"])).codes
    diff = np.flatnonzero(np.any(got != want, axis=1))
    assert diff.size <= max(1, x.shape[0] // 200), (case, diff.size)
    if diff.size:
        lg, lw = _loss(x[diff], books, got[diff]), _loss(x[diff], books, want[diff])
        assert np.all(np.abs(lg - lw) <= 1e-9 * np.maximum(lw, 1e-30)), case


def test_encode_dataset_mirror_and_validation():
    x, books = Z["a_x"], Z["a_books"]
    idx = icqb.SearchIndex(books=books, codes=np.zeros((1, 8), dtype=np.uint32),
                           xi=np.ones(32, dtype=np.uint8), fast=np.array([0, 1], dtype=np.uint32),
                           sigma=0.5, lambdas=np.ones(32, dtype=np.float32),
                           cfg=icqb.Config(K=8, m=256))
    enc = icqb.encode_dataset(idx, icqb.EmbeddedDataset(x))
    assert enc.n == x.shape[0] and enc.sigma == 0.5 and enc.fast.tolist() == [0, 1]
    assert np.array_equal(enc.codes.codes, icqb.assign_codes(x, books).codes)
    with pytest.raises(icqb.ValidationError):
        icqb.encode_dataset(idx, x[:, :31])
    with pytest.raises(icqb.ValidationError):
        icqb.assign_codes(x, books, codes=np.zeros((3, 8), dtype=np.uint32))


def test_max_sweeps_zero_is_greedy_and_chunk_invariant():
    x, books = Z["a_x"], Z["a_books"]
    greedy = icqb.assign_codes(x, books, max_sweeps=0).codes
    # a greedy pass restated in numpy float64 (train.py:213-219)
    b = books.astype(np.float64)
    c_sq = (b ** 2).sum(axis=2)
    res = x.astype(np.float64).copy()
    want = np.empty((x.shape[0], 8), dtype=np.int64)
    for k in range(8):
        dist = c_sq[k][None, :] - 2.0 * (res @ b[k].T)
        want[:, k] = np.argmin(dist, axis=1)
        res -= b[k][want[:, k]]
    assert np.mean(np.all(greedy == want, axis=1)) > 0.995
    # the device form on a tensor, rows split differently: identical codes
    xd = torch.from_numpy(x).cuda()
    full, _ = icqb.encode_device(xd, books)
    part = torch.cat([icqb.encode_device(xd[:1000], books)[0], icqb.encode_device(xd[1000:], books)[0]])
    assert torch.equal(full, part)
