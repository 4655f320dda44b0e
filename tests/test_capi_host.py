"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/icq_b200.h declares, and the host wrapper rejects invalid
arguments with the reference's exception classes before touching a device."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared_symbols():
    text = (ROOT / "include" / "icq_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(icq_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    syms = _declared_symbols()
    for s in ("icq_index_create", "icq_build_lut", "icq_search_two_step", "icq_search_exact",
              "icq_search_host", "icq_last_error", "icq_index_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    import __graft_entry__ as g

    g.build()
    from paper_1912_08756_b200 import _native

    lib = _native.lib()
    for s in _declared_symbols():
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, f"{s} declared in the header but not bound"
    assert lib.icq_abi_version() == 3


def test_null_handle_is_validation_error():
    from paper_1912_08756_b200 import _native

    L = _native.lib()
    assert L.icq_index_destroy(None) == 0
    assert L.icq_index_info(None, None, None, None, None, None, None) == _native.ICQ_ERR_VALIDATION
    assert "null" in _native.last_error()


def _index(**kw):
    import paper_1912_08756_b200 as icqb

    rng = np.random.default_rng(0)
    f = dict(books=rng.standard_normal((3, 4, 8)).astype(np.float32),
             codes=rng.integers(0, 4, size=(20, 3)), xi=np.ones(8, dtype=np.uint8),
             fast=np.array([0], dtype=np.uint32), sigma=0.5,
             lambdas=np.ones(8, dtype=np.float32), cfg=icqb.Config(K=3, m=4))
    f.update(kw)
    return icqb.SearchIndex(**f)


def test_searchindex_validation_mirrors_reference():
    import paper_1912_08756_b200 as icqb

    with pytest.raises(icqb.ValidationError):
        _index(codes=np.full((20, 3), 4))
    with pytest.raises(icqb.ValidationError):
        _index(fast=np.array([1, 0], dtype=np.uint32))
    with pytest.raises(icqb.ValidationError):
        _index(fast=np.array([3], dtype=np.uint32))
    with pytest.raises(icqb.ValidationError):
        _index(sigma=-1.0)
    with pytest.raises(icqb.ValidationError):
        _index(xi=np.ones(7, dtype=np.uint8))
    idx = _index(sigma=0.1)
    assert idx.sigma == float(np.float32(0.1))


def test_engine_argument_validation_without_device():
    import paper_1912_08756_b200 as icqb

    idx = _index()
    q = np.zeros(8)
    with pytest.raises(icqb.ValidationError):
        icqb.search_two_step(idx, q, 0)
    with pytest.raises(icqb.ValidationError):
        icqb.search_two_step(idx, q, 21)
    with pytest.raises(icqb.ValidationError):
        icqb.search_two_step(idx, q, 3, sigma=-1.0)
    with pytest.raises(icqb.ValidationError):
        icqb.search_two_step(idx, q, 3, sigma=float("nan"))
    with pytest.raises(icqb.ValidationError):
        icqb.search_exact(idx, np.zeros(7), 1)
    with pytest.raises(icqb.ValidationError):
        icqb.search_exact(idx, np.full(8, np.nan), 1)


def test_row_helpers_match_reference_worked_example():
    """test_search.py:53-67 worked example on the host helpers."""
    import paper_1912_08756_b200 as icqb

    lut = np.array([[2.0, 1.0], [2.0, 1.0]])
    ops = icqb.OpCounter()
    assert icqb.exact_score(lut, np.array([1, 1]), ops) == 2.0
    assert icqb.exact_score(lut, np.array([0, 0]), ops) == 4.0
    assert ops.exact_adds == 2
    assert icqb.fast_score(lut, np.array([1, 1]), np.array([0]), ops) == 1.0
    assert ops.fast_adds == 0
