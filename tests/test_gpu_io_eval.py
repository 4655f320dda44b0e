"""GPU checks of the §8(f) rows: ICQI streaming loader (f2), brute-force
ground truth (f3), batched run_benchmark / CLI (f4) -- all against outputs of
the real reference (tests/golden/eval_cli.npz, make_golden_eval.py) or the
oracle, byte for byte."""

import contextlib
import io
from pathlib import Path

import numpy as np
import pytest

from oracle import icq_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1912_08756_b200 as icqb  # noqa: E402
from paper_1912_08756_b200.cli import main as cli_main  # noqa: E402

GOLD = np.load(Path(__file__).parent / "golden" / "eval_cli.npz")


@pytest.fixture
def files(tmp_path):
    for nm in ("i.icqi", "d.icqd", "q.icqd"):
        (tmp_path / nm).write_bytes(GOLD[f"file_{nm}"].tobytes())
    return tmp_path


def test_load_index_matches_file(files):
    idx = icqb.load_index(files / "i.icqi")
    raw = (files / "i.icqi").read_bytes()
    assert idx.n == 3000 and idx.d == 16 and idx.cfg.K == 4 and idx.cfg.m == 16
    assert idx.fast.tolist() == [0, 1] and idx.sigma == 0.75
    # codes come back from the device exactly
    again = files / "again.icqi"
    icqb.save_index(idx, again)
    assert again.read_bytes() == raw
    q = icqb.load_dataset(files / "q.icqd").vectors.astype(np.float64)
    c = idx.codes.codes
    for i in range(4):
        r = icqb.search_two_step(idx, q[i], 9)
        o = O.two_step(idx.books.codewords, c, idx.fast, idx.sigma, q[i], 9)
        assert np.array_equal(r.ids, o.ids) and np.array_equal(r.scores, o.scores)
        assert r.ops.refinements == o.ops.refinements


def test_load_index_codes_beyond_m(files):
    raw = bytearray((files / "i.icqi").read_bytes())
    codes_off = 96 + 4 * 16 * 16 * 4
    raw[codes_off + 4 * 57:codes_off + 4 * 58] = (16).to_bytes(4, "little")  # code == m
    bad = files / "bad.icqi"
    bad.write_bytes(bytes(raw))
    with pytest.raises(icqb.FormatError):
        icqb.load_index(bad)


def test_load_index_streams_many_chunks(tmp_path):
    """> 1 pinned chunk (64 MiB of uint32 codes per chunk): 9M rows, K = 2."""
    rng = np.random.default_rng(5)
    n, K, m, d = 9_000_000, 2, 256, 8
    books = rng.standard_normal((K, m, d)).astype(np.float32)
    codes = rng.integers(0, m, size=(n, K), dtype=np.uint32)
    idx = icqb.SearchIndex(books=books, codes=codes, xi=np.ones(d, dtype=np.uint8),
                           fast=np.array([0], dtype=np.uint32), sigma=0.0,
                           lambdas=np.ones(d, dtype=np.float32), cfg=icqb.Config(K=K, m=m))
    p = tmp_path / "big.icqi"
    icqb.save_index(idx, p)
    loaded = icqb.load_index(p)
    back = loaded.device.read_codes()
    assert np.array_equal(back, codes.astype(np.uint8))
    q = rng.standard_normal((2, d))
    a = icqb.search_two_step_batch(loaded, q, 5)
    b = icqb.search_two_step_batch(idx, q, 5)
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.scores, b.scores)


@pytest.mark.parametrize("n,d,k,dup", [(1, 3, 1, False), (5000, 16, 10, False),
                                        (70001, 7, 100, True), (200000, 130, 37, True),
                                        (66000, 32, 1024, False)])
def test_bruteforce_vs_oracle(n, d, k, dup):
    rng = np.random.default_rng(n + d)
    x = rng.standard_normal((n, d)).astype(np.float32)
    if dup:  # exact score ties: (score, id) order decides (search.py:176)
        x[1::3] = x[0::3][: x[1::3].shape[0]]
    Q = rng.standard_normal((5, d))
    res = icqb.search_bruteforce_batch(x, Q, k)
    for i in range(5):
        o = O.bruteforce(x, Q[i], k)
        assert np.array_equal(res.ids[i], o.ids), (n, d, k, i)
        assert np.array_equal(res.scores[i], o.scores), (n, d, k, i)
    one = icqb.search_bruteforce(x, Q[0], k)
    assert np.array_equal(one.ids, res.ids[0])
    assert one.ops.exact_adds == (d - 1) * n and one.ops.refinements == n


def test_bruteforce_validation():
    x = np.zeros((10, 4), dtype=np.float32)
    with pytest.raises(icqb.ValidationError):
        icqb.search_bruteforce(x, np.zeros(4), 11)
    with pytest.raises(icqb.ValidationError):
        icqb.search_bruteforce(x, np.array([0, 0, np.nan, 0]), 1)
    with pytest.raises(icqb.UnsupportedError):
        icqb.search_bruteforce(np.zeros((2000, 4), dtype=np.float32), np.zeros(4), 1025)


@pytest.mark.parametrize("key", sorted(k for k in GOLD.files if k.startswith("bench_")))
def test_run_benchmark_report_is_reference_csv(files, key):
    _, truth, sg, kk = key.split("_")
    idx = icqb.load_index(files / "i.icqi")
    ds = icqb.load_dataset(files / "d.icqd")
    q = icqb.load_dataset(files / "q.icqd")
    rep = icqb.run_benchmark(idx, ds, q, truth=truth, k=int(kk[1:]),
                             sigma=None if sg == "none" else 0.0)
    assert rep.to_csv() == str(GOLD[key])


@pytest.mark.parametrize("name,extra", [
    ("search_two", ["--index", "i.icqi", "--k", "7"]),
    ("search_two_scale", ["--index", "i.icqi", "--k", "7", "--sigma-scale", "0.25"]),
    ("search_exact", ["--index", "i.icqi", "--k", "7", "--mode", "exact"]),
    ("search_brute", ["--data", "d.icqd", "--k", "7", "--mode", "brute"]),
])
def test_cli_search_csv_is_reference(files, name, extra):
    extra = [str(files / a) if a.endswith((".icqi", ".icqd")) else a for a in extra]
    out = files / f"{name}.csv"
    with contextlib.redirect_stderr(io.StringIO()):
        assert cli_main(["search", "--queries", str(files / "q.icqd"), "--out", str(out), *extra]) == 0
    assert out.read_text() == str(GOLD[name])


def test_cli_inspect_and_errors(files):
    for name, path in (("inspect_index", "i.icqi"), ("inspect_data", "d.icqd")):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(io.StringIO()):
            assert cli_main(["inspect", str(files / path)]) == 0
        assert buf.getvalue() == str(GOLD[name])
    with contextlib.redirect_stderr(io.StringIO()):
        assert cli_main(["search", "--queries", str(files / "q.icqd"), "--out",
                         str(files / "x.csv"), "--mode", "brute"]) == 1  # needs --data
        (files / "junk").write_bytes(b"NOPE1234")
        assert cli_main(["inspect", str(files / "junk")]) == 1
