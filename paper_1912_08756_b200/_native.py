"""ctypes binding of libicq_b200.so (include/icq_b200.h).

No fallback: if the library is missing the import of any engine fails loudly
with instructions to build it.  This is the same binding INTEGRATION.md shows
for the reference side.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_DIR = Path(__file__).resolve().parent / "lib"
LIB_PATH = Path(os.environ.get("ICQ_B200_LIB", _LIB_DIR / "libicq_b200.so"))

ICQ_OK = 0
ICQ_ERR_VALIDATION = 1
ICQ_ERR_UNSUPPORTED = 2
ICQ_ERR_CUDA = 3
ICQ_ERR_NOMEM = 4
ICQ_ERR_FORMAT = 5
ICQ_ERR_VERSION = 6

class IndexFileInfo(C.Structure):
    """icq_index_file_info (include/icq_b200.h)."""

    _fields_ = [("K", C.c_int64), ("m", C.c_int64), ("d", C.c_int64), ("n", C.c_int64),
                ("gamma1", C.c_double), ("gamma2", C.c_double), ("pi1", C.c_double),
                ("pi2", C.c_double), ("alpha2", C.c_double), ("sigma_scale", C.c_double),
                ("epochs", C.c_int64), ("batch_size", C.c_int64),
                ("learning_rate", C.c_double), ("seed", C.c_uint64), ("sigma", C.c_float),
                ("F", C.c_int32), ("fast", C.c_uint32 * 64), ("file_bytes", C.c_int64)]


# exported symbols and their C signatures (kept in sync with include/icq_b200.h)
_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
SIGNATURES = {
    "icq_last_error": (C.c_char_p, []),
    "icq_abi_version": (_i32, []),
    "icq_kernel_launches": (C.c_int64, []),
    "icq_index_create": (_i32, [_vp, _i32, _i32, _i32, _vp, _i64, _vp, _i32, C.POINTER(_vp)]),
    "icq_index_create_u8": (_i32, [_vp, _i32, _i32, _i32, _vp, _i64, _vp, _i32, C.POINTER(_vp)]),
    "icq_index_create_device": (
        _i32, [_vp, _i32, _i32, _i32, _vp, _i64, _vp, _i32, _vp, C.POINTER(_vp)]),
    "icq_index_destroy": (_i32, [_vp]),
    "icq_index_info": (_i32, [_vp, C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i32),
                              C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i64)]),
    "icq_build_lut": (_i32, [_vp, _vp, _i32, _vp, _vp]),
    "icq_workspace_size": (_i32, [_vp, _i32, _i32, C.POINTER(C.c_size_t)]),
    "icq_search_two_step": (_i32, [_vp, _vp, _i32, _i32, C.c_double, _vp, _vp, _vp, _vp, _vp,
                                   C.POINTER(_i32), _vp, C.c_size_t, _vp]),
    "icq_search_exact": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, C.c_size_t, _vp]),
    "icq_search_with_lut": (_i32, [_vp, _vp, _i32, _i32, C.c_double, _i32, _vp, _vp, _vp, _vp,
                                   _vp, C.POINTER(_i32), _vp]),
    "icq_search_host": (_i32, [_vp, _vp, _i32, _i32, C.c_double, _i32, _vp, _vp, _vp,
                               C.POINTER(_i32)]),
    "icq_index_read_codes": (_i32, [_vp, _i64, _i64, _vp]),
    "icq_index_file_info_read": (_i32, [C.c_char_p, C.POINTER(IndexFileInfo)]),
    "icq_index_load": (_i32, [C.c_char_p, _vp, _vp, _vp, C.POINTER(IndexFileInfo), _vp,
                              C.POINTER(_vp)]),
    "icq_bruteforce": (_i32, [_vp, _i64, _i32, _vp, _i32, _i32, _vp, _vp, _vp]),
    "icq_encode": (_i32, [_vp, _i64, _i32, _vp, _vp, _i32, _i32, _vp, _i32, _vp,
                          C.POINTER(_i32), _vp]),
    "icq_profile_enable": (_i32, [_i32]),
    "icq_profile_read": (_i32, [C.POINTER(C.c_double), C.POINTER(_i32)]),
}

_lib = None


def lib():
    """Load (once) and return the CDLL; raises if the library was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().icq_last_error()
    return msg.decode() if msg else ""
