"""GPU ICM encoder with the reference's encode entry points.

Reference: /root/reference/pkg/src/icq/train.py
    assign_codes(ds, books, codes=None, max_sweeps=10) -> CodeMatrix   :196-243
    encode_dataset(index, ds) -> SearchIndex                           :256-274
Both run the float64 ICM encoder of libicq_b200.so (icq_encode, icq_encode.cu):
greedy residual build-up (or the given codes), then strict-improvement
sweeps until one changes nothing.  ``encode_device`` is the device-tensor
form used to encode large synthetic databases chunk by chunk without host
copies (tools/workloads.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .data import CodeMatrix, DeviceError, SearchIndex, UnsupportedError, ValidationError


def _raise(code: int, what: str):
    msg = f"{what}: {_native.last_error()}"
    if code == _native.ICQ_ERR_VALIDATION:
        raise ValidationError(msg)
    if code == _native.ICQ_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise DeviceError(msg)


def _vectors(ds) -> np.ndarray:
    """train.py:61-67."""
    if hasattr(ds, "vectors"):
        return ds.vectors
    arr = np.asarray(ds)
    if arr.ndim != 2:
        raise ValidationError(f"expected (n, d) vectors, got shape {arr.shape}")
    return arr


def _codewords(books) -> np.ndarray:
    return books.codewords if hasattr(books, "codewords") else np.asarray(books)


def _book_tables(books):
    """float64 codewords and their squared norms (train.py:207, :212), numpy order."""
    b = np.ascontiguousarray(_codewords(books), dtype=np.float64)
    if b.ndim != 3:
        raise ValidationError(f"codewords must be (K, m, d), got shape {b.shape}")
    return b, (b ** 2).sum(axis=2)


def encode_device(x, books, codes=None, max_sweeps: int = 10, stream=None):
    """(n, d) float32 cuda tensor -> (n, K) uint8 cuda tensor of ICM codes.

    ``codes``: optional (n, K) uint8 cuda tensor of starting codes.
    Returns (codes, sweeps run).
    """
    import torch

    if x.dtype != torch.float32 or x.dim() != 2 or not x.is_cuda:
        raise ValidationError("x must be a cuda float32 tensor of shape (n, d)")
    b, c_sq = _book_tables(books)
    K, m, d = b.shape
    if x.shape[1] != d:
        raise ValidationError(f"codebook d={d} does not match data d={x.shape[1]}")
    if m > 256:
        raise UnsupportedError(f"m={m} > 256 codewords (uint8 codes)")
    x = x.contiguous()
    dev = x.device
    bd = torch.from_numpy(b).to(dev)
    cs = torch.from_numpy(np.ascontiguousarray(c_sq)).to(dev)
    out = torch.empty((x.shape[0], K), dtype=torch.uint8, device=dev)
    cin = None
    if codes is not None:
        if codes.shape != (x.shape[0], K) or codes.dtype != torch.uint8:
            raise ValidationError(f"codes shape {tuple(codes.shape)} does not match ({x.shape[0]}, {K})")
        cin = codes.contiguous()
    used = C.c_int32(0)
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    st = _native.lib().icq_encode(x.data_ptr(), x.shape[0], d, bd.data_ptr(), cs.data_ptr(), K, m,
                                  cin.data_ptr() if cin is not None else None, int(max_sweeps),
                                  out.data_ptr(), C.byref(used), s)
    if st != _native.ICQ_OK:
        _raise(st, "icq_encode")
    return out, int(used.value)


def assign_codes(ds, books, codes=None, max_sweeps: int = 10) -> CodeMatrix:
    """Encode elements by iterated conditional modes over the codebooks (train.py:196-243)."""
    import torch

    x = _vectors(ds)
    b = _codewords(books)
    if np.asarray(b).shape[2] != x.shape[1]:
        raise ValidationError(f"codebook d={np.asarray(b).shape[2]} does not match data d={x.shape[1]}")
    x32 = np.ascontiguousarray(x, dtype=np.float32)
    if x.dtype != np.float32 and not np.array_equal(x32.astype(np.float64), np.asarray(x, dtype=np.float64)):
        raise UnsupportedError("the device encoder takes float32 vectors (the reference's "
                               "EmbeddedDataset storage type)")
    K = np.asarray(b).shape[0]
    cin = None
    if codes is not None:
        arr = np.asarray(codes.codes if hasattr(codes, "codes") else codes)
        if arr.shape != (x.shape[0], K):
            raise ValidationError(f"codes shape {arr.shape} does not match ({x.shape[0]}, {K})")
        if arr.size and (arr.min() < 0 or arr.max() > 255):
            raise ValidationError("codes reference codewords beyond m")
        cin = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.uint8)).cuda()
    out, _ = encode_device(torch.from_numpy(x32).cuda(), b, cin, max_sweeps)
    return CodeMatrix(out.cpu().numpy().astype(np.uint32))


def encode_dataset(index, ds):
    """Index new data with an already trained quantizer (train.py:256-274)."""
    x = _vectors(ds)
    if x.shape[1] != index.d:
        raise ValidationError(f"data d={x.shape[1]} does not match index d={index.d}")
    codes = assign_codes(x, index.books)
    return SearchIndex(books=index.books, codes=codes, xi=index.xi, fast=index.fast,
                       sigma=index.sigma, lambdas=index.lambdas, cfg=index.cfg)


__all__ = ["assign_codes", "encode_dataset", "encode_device"]
