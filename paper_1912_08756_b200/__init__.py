"""B200-native ICQ query path (arXiv 1912.08756) — drop-in for icq.search.

Names mirror the reference package (/root/reference/pkg/src/icq/__init__.py:9-53):
``build_lut``, ``exact_score``, ``fast_score``, ``search_exact``,
``search_two_step``, ``OpCounter``, ``QueryResult``, ``SearchIndex``,
``ValidationError``.  The engines run hand-written sm_100a CUDA kernels
through the C ABI of libicq_b200.so (include/icq_b200.h).
"""

from .data import (
    CodebookSet,
    CodeMatrix,
    Config,
    DeviceError,
    SearchIndex,
    UnsupportedError,
    ValidationError,
)
from .search import (
    BatchResult,
    DeviceIndex,
    OpCounter,
    QueryResult,
    build_lut,
    device_index,
    exact_score,
    fast_score,
    search_exact,
    search_exact_batch,
    search_two_step,
    search_two_step_batch,
)

__all__ = [
    "BatchResult",
    "CodebookSet",
    "CodeMatrix",
    "Config",
    "DeviceError",
    "DeviceIndex",
    "OpCounter",
    "QueryResult",
    "SearchIndex",
    "UnsupportedError",
    "ValidationError",
    "build_lut",
    "device_index",
    "exact_score",
    "fast_score",
    "search_exact",
    "search_exact_batch",
    "search_two_step",
    "search_two_step_batch",
]
