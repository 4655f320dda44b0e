"""CPU checks of the file formats (no device work): ICQD reader/writer against
the reference's own files, and every ICQI FormatError / UnsupportedVersionError
condition of data.py:348-394, which the native loader detects before it
touches the GPU."""

import struct

import numpy as np
import pytest

import paper_1912_08756_b200 as icqb
from paper_1912_08756_b200 import io as bio

GOLD = np.load(__import__("pathlib").Path(__file__).parent / "golden" / "eval_cli.npz")


def _bytes(name):
    return GOLD[f"file_{name}"].tobytes()


def test_dataset_roundtrip_is_byte_identical(tmp_path):
    p = tmp_path / "d.icqd"
    p.write_bytes(_bytes("d.icqd"))
    ds = icqb.load_dataset(p)
    assert ds.vectors.dtype == np.float32 and ds.labels.dtype == np.uint32
    q = tmp_path / "again.icqd"
    icqb.save_dataset(ds, q)
    assert q.read_bytes() == p.read_bytes()


@pytest.mark.parametrize("mutate", ["short", "magic", "flag", "length"])
def test_dataset_format_errors(tmp_path, mutate):
    raw = bytearray(_bytes("q.icqd"))
    if mutate == "short":
        raw = raw[:12]
    elif mutate == "magic":
        raw[:4] = b"XXXX"
    elif mutate == "flag":
        raw[12] = 2
    else:
        raw = raw[:-3]
    p = tmp_path / "bad.icqd"
    p.write_bytes(bytes(raw))
    with pytest.raises(icqb.FormatError):
        icqb.load_dataset(p)


def _index_sections(raw):
    """Offsets of the ICQI sections of a valid file."""
    K, m = struct.unpack_from("<II", raw, 8)
    n, d = struct.unpack_from("<II", raw, 88)
    books = 96
    codes = books + K * m * d * 4
    xi = codes + n * K * 4
    fastm = xi + 4 + d
    lam = fastm + 4 + K
    sigma = lam + 4 + 4 * d
    return dict(K=K, m=m, n=n, d=d, books=books, codes=codes, xi=xi, fastm=fastm, lam=lam,
                sigma=sigma, end=sigma + 4)


def test_file_info_header_parse():
    import ctypes as C

    from paper_1912_08756_b200 import _native

    raw = _bytes("i.icqi")
    s = _index_sections(raw)
    assert s["end"] == len(raw)
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".icqi") as f:
        f.write(raw)
        f.flush()
        info = _native.IndexFileInfo()
        assert _native.lib().icq_index_file_info_read(f.name.encode(), C.byref(info)) == 0
    assert (info.K, info.m, info.n, info.d) == (s["K"], s["m"], s["n"], s["d"])
    assert info.epochs == 3 and info.seed == 11 and info.gamma1 == 0.1


CASES = {
    "bad_magic": (lambda r, s: r.__setitem__(slice(0, 4), b"ICQX"), icqb.FormatError),
    "version": (lambda r, s: r.__setitem__(slice(4, 8), struct.pack("<I", 2)),
                icqb.UnsupportedVersionError),
    "truncated_header": (lambda r, s: r.__delitem__(slice(50, None)), icqb.FormatError),
    "bad_config_pi": (lambda r, s: r.__setitem__(slice(32, 40), struct.pack("<d", 0.05)),
                      icqb.FormatError),
    "bad_config_alpha": (lambda r, s: r.__setitem__(slice(48, 56), struct.pack("<d", 1.0)),
                         icqb.FormatError),
    "truncated_codes": (lambda r, s: r.__delitem__(slice(s["codes"] + 100, None)), icqb.FormatError),
    "xi_length": (lambda r, s: r.__setitem__(slice(s["xi"], s["xi"] + 4),
                                             struct.pack("<I", s["d"] + 1)), icqb.FormatError),
    "fast_length": (lambda r, s: r.__setitem__(slice(s["fastm"], s["fastm"] + 4),
                                               struct.pack("<I", s["K"] - 1)), icqb.FormatError),
    "lam_length": (lambda r, s: r.__setitem__(slice(s["lam"], s["lam"] + 4),
                                              struct.pack("<I", 0)), icqb.FormatError),
    "trailing": (lambda r, s: r.extend(b"\0\0"), icqb.FormatError),
    "xi_value": (lambda r, s: r.__setitem__(s["xi"] + 4, 2), icqb.FormatError),
    "lambda_nan": (lambda r, s: r.__setitem__(slice(s["lam"] + 4, s["lam"] + 8),
                                              struct.pack("<f", float("nan"))), icqb.FormatError),
    "sigma_negative": (lambda r, s: r.__setitem__(slice(s["sigma"], s["sigma"] + 4),
                                                  struct.pack("<f", -1.0)), icqb.FormatError),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_index_format_errors_before_device(tmp_path, case):
    raw = bytearray(_bytes("i.icqi"))
    mutate, exc = CASES[case]
    mutate(raw, _index_sections(bytes(raw)))
    p = tmp_path / "bad.icqi"
    p.write_bytes(bytes(raw))
    with pytest.raises(exc):
        bio.load_index(p)


def test_reference_classes_when_importable():
    """With the reference on the path the mirror raises subclasses of its classes."""
    icq_data = pytest.importorskip("icq.data")
    assert issubclass(icqb.ValidationError, icq_data.ValidationError)
    assert issubclass(icqb.FormatError, icq_data.FormatError)
    assert issubclass(icqb.UnsupportedVersionError, icq_data.UnsupportedVersionError)


def test_metric_helpers_restate_reference():
    from paper_1912_08756_b200 import evaluate as E

    rng = np.random.default_rng(3)
    for _ in range(50):
        ranked = rng.permutation(40)[:10]
        rel = rng.choice(40, size=rng.integers(1, 12), replace=False)
        ap = E.average_precision(ranked, rel)
        hits = np.isin(ranked, rel)
        want = 0.0 if not hits.any() else float(
            (np.cumsum(hits) / (np.arange(10) + 1))[hits].mean())
        assert ap == want
        assert E.recall_at(ranked, rel, 5) == float(np.isin(ranked[:5], rel).sum()) / min(5, rel.size)
    with pytest.raises(icqb.ValidationError):
        E.recall_at(ranked, rel, 0)
    with pytest.raises(icqb.ValidationError):
        E.effective_code_length(32.0, 1.0, 0.0)
    assert E.code_length_bits(8, 256) == 64.0
