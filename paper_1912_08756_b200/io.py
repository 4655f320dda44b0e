"""Index and dataset files for the B200 query path (mirror of icq.data I/O).

* ``load_index(path)`` -- the reference's ``load_index`` (data.py:348-394),
  but the file goes straight to device memory: the native loader
  (icq_io.cu) validates header and tail with the reference's conditions and
  streams the (n, K) uint32 code block through pinned buffers into the GPU
  repack.  Returns a :class:`DeviceSearchIndex`, usable wherever the engines
  take a ``SearchIndex``; its host ``codes`` are fetched from the device only
  if someone asks for them.
* ``load_dataset(path)`` -- ICQD reader (data.py:279-299), host side (queries
  and raw vectors for brute-force truth).
* ``save_dataset`` / ``save_index`` -- byte-identical writers
  (data.py:266-277, :306-322) so tests and tools can produce files without the
  reference package.

Malformed files raise :class:`FormatError`, unknown versions
:class:`UnsupportedVersionError` (subclasses of the reference's classes when
``icq`` is importable, data.py:36-41).
"""

from __future__ import annotations

import ctypes as C
import struct
from pathlib import Path

import numpy as np

from . import _native
from .data import (CodebookSet, CodeMatrix, Config, DeviceError, EmbeddedDataset, FormatError,
                   UnsupportedError, UnsupportedVersionError, ValidationError)

INDEX_FORMAT_VERSION = 1
_DATASET_MAGIC = b"ICQD"
_INDEX_MAGIC = b"ICQI"
_CONFIG_STRUCT = struct.Struct("<IIddddddIIdQ")


def _raise(code: int, what: str):
    msg = f"{what}: {_native.last_error()}"
    if code == _native.ICQ_ERR_FORMAT:
        raise FormatError(msg)
    if code == _native.ICQ_ERR_VERSION:
        raise UnsupportedVersionError(msg)
    if code == _native.ICQ_ERR_VALIDATION:
        raise ValidationError(msg)
    if code == _native.ICQ_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise DeviceError(msg)


class DeviceSearchIndex:
    """A SearchIndex whose codes live on the device (from :func:`load_index`).

    Same fields as ``icq.SearchIndex`` (data.py:193-263): books, codes, xi,
    fast, sigma, lambdas, cfg, n, d.  ``codes`` is materialised from the
    device on first access (uint8 -> uint32 CodeMatrix).
    """

    def __init__(self, books, xi, fast, sigma, lambdas, cfg, n, device):
        self.books = CodebookSet(books)
        self.xi = xi
        self.fast = fast
        self.sigma = sigma
        self.lambdas = lambdas
        self.cfg = cfg
        self._n = n
        self._device = device
        self._codes = None

    @property
    def n(self) -> int:
        return self._n

    @property
    def d(self) -> int:
        return self.books.d

    @property
    def device(self):
        return self._device

    @property
    def codes(self) -> CodeMatrix:
        if self._codes is None:
            self._codes = CodeMatrix(self._device.read_codes().astype(np.uint32))
        return self._codes


def load_index(path) -> DeviceSearchIndex:
    """Read an ICQI index file into device memory (data.py:348-394)."""
    from .search import DeviceIndex

    L = _native.lib()
    p = str(Path(path)).encode()
    info = _native.IndexFileInfo()
    st = L.icq_index_file_info_read(p, C.byref(info))
    if st != _native.ICQ_OK:
        _raise(st, f"load_index({path})")
    K, m, d = int(info.K), int(info.m), int(info.d)
    books = np.empty((K, m, d), dtype=np.float32)
    xi = np.empty(d, dtype=np.uint8)
    lam = np.empty(d, dtype=np.float32)
    h = C.c_void_p()
    st = L.icq_index_load(p, books.ctypes.data, xi.ctypes.data, lam.ctypes.data, C.byref(info),
                          None, C.byref(h))
    if st != _native.ICQ_OK:
        _raise(st, f"load_index({path})")
    fast = np.array(list(info.fast)[: info.F], dtype=np.uint32)
    dev = DeviceIndex._adopt(h, K, m, d, int(info.n), int(info.F))
    cfg = Config(K=K, m=m, gamma1=info.gamma1, gamma2=info.gamma2, pi1=info.pi1, pi2=info.pi2,
                 alpha2=info.alpha2, sigma_scale=info.sigma_scale, epochs=int(info.epochs),
                 batch_size=int(info.batch_size), learning_rate=info.learning_rate,
                 seed=int(info.seed))
    # the stored float32 margin as a Python float (data.py:252, :380)
    return DeviceSearchIndex(books, xi, fast, float(info.sigma), lam, cfg, int(info.n), dev)


def save_index(index, path) -> None:
    """Write an ICQI file, byte-identical to the reference (data.py:306-322)."""
    books = np.asarray(index.books.codewords)
    K = books.shape[0]
    fast_mask = np.zeros(K, dtype=np.uint8)
    fast_mask[np.asarray(index.fast).astype(np.int64)] = 1
    cfg = index.cfg
    with open(path, "wb") as f:
        f.write(_INDEX_MAGIC)
        f.write(struct.pack("<I", INDEX_FORMAT_VERSION))
        f.write(_CONFIG_STRUCT.pack(cfg.K, cfg.m, cfg.gamma1, cfg.gamma2, cfg.pi1, cfg.pi2,
                                    cfg.alpha2, cfg.sigma_scale, cfg.epochs, cfg.batch_size,
                                    cfg.learning_rate, cfg.seed))
        f.write(struct.pack("<II", index.n, index.d))
        f.write(np.ascontiguousarray(books, dtype="<f4").tobytes())
        f.write(np.ascontiguousarray(index.codes.codes, dtype="<u4").tobytes())
        for arr, dt in ((index.xi, np.uint8), (fast_mask, np.uint8)):
            f.write(struct.pack("<I", len(arr)) + np.ascontiguousarray(arr, dtype=dt).tobytes())
        f.write(struct.pack("<I", index.d))
        f.write(np.ascontiguousarray(index.lambdas, dtype="<f4").tobytes())
        f.write(struct.pack("<f", index.sigma))


def save_dataset(ds: EmbeddedDataset, path) -> None:
    """Write an ICQD file (data.py:266-277); non-finite vectors are rejected."""
    if not np.all(np.isfinite(ds.vectors)):
        raise ValidationError("dataset vectors contain non-finite values")
    has_labels = ds.labels is not None
    with open(path, "wb") as f:
        f.write(_DATASET_MAGIC)
        f.write(struct.pack("<IIB", ds.n, ds.d, int(has_labels)))
        f.write(np.ascontiguousarray(ds.vectors, dtype="<f4").tobytes())
        if has_labels:
            f.write(np.ascontiguousarray(ds.labels, dtype="<u4").tobytes())


def load_dataset(path) -> EmbeddedDataset:
    """Read an ICQD file, validating magic, header and exact length (data.py:279-299)."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < 13:
        raise FormatError(f"dataset file too short ({len(raw)} bytes)")
    if raw[:4] != _DATASET_MAGIC:
        raise FormatError(f"bad dataset magic {raw[:4]!r}")
    n, d, has_labels = struct.unpack_from("<IIB", raw, 4)
    if has_labels not in (0, 1):
        raise FormatError(f"has_labels flag must be 0 or 1, got {has_labels}")
    expected = 13 + n * d * 4 + (n * 4 if has_labels else 0)
    if len(raw) != expected:
        raise FormatError(f"dataset payload is {len(raw)} bytes, expected {expected}")
    vectors = np.frombuffer(raw, dtype="<f4", count=n * d, offset=13).reshape(n, d)
    labels = None
    if has_labels:
        labels = np.frombuffer(raw, dtype="<u4", count=n, offset=13 + n * d * 4)
    return EmbeddedDataset(vectors.copy(), None if labels is None else labels.copy())


__all__ = ["DeviceSearchIndex", "load_index", "save_index", "load_dataset", "save_dataset",
           "INDEX_FORMAT_VERSION"]
