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
    EmbeddedDataset,
    FormatError,
    SearchIndex,
    UnsupportedError,
    UnsupportedVersionError,
    ValidationError,
)
from .evaluate import (
    EvalReport,
    average_precision,
    code_length_bits,
    effective_code_length,
    recall_at,
    run_benchmark,
)
from .encode import assign_codes, encode_dataset, encode_device
from .io import DeviceSearchIndex, load_dataset, load_index, save_dataset, save_index
from .search import (
    BatchResult,
    DeviceIndex,
    OpCounter,
    QueryResult,
    build_lut,
    device_index,
    exact_score,
    fast_score,
    DeviceDataset,
    search_bruteforce,
    search_bruteforce_batch,
    search_exact,
    search_exact_batch,
    search_two_step,
    search_two_step_batch,
)

__all__ = [
    "BatchResult",
    "DeviceDataset",
    "DeviceSearchIndex",
    "assign_codes",
    "encode_dataset",
    "encode_device",
    "EmbeddedDataset",
    "EvalReport",
    "FormatError",
    "UnsupportedVersionError",
    "average_precision",
    "code_length_bits",
    "effective_code_length",
    "load_dataset",
    "load_index",
    "recall_at",
    "run_benchmark",
    "save_dataset",
    "save_index",
    "search_bruteforce",
    "search_bruteforce_batch",
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
