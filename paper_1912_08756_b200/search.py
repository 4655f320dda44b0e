"""B200 query engines with the reference's call surface (mirror of icq.search).

Reference: /root/reference/pkg/src/icq/search.py.  Same names, arguments,
return types, op accounting and exceptions:

    build_lut(index, q, ops=None)              search.py:61-69
    exact_score / fast_score                   search.py:72-89 (per-row helpers)
    search_exact(index, q, k)                  search.py:97-109
    search_two_step(index, q, k, sigma=None)   search.py:112-165

plus batched variants (``search_two_step_batch`` / ``search_exact_batch``)
and ``DeviceIndex`` for device-resident (torch) inputs.  Every engine runs
the CUDA kernels of libicq_b200.so; there is no CPU fallback.  Results are
bitwise the reference's: float64 scores, ids ordered by (score, id),
refinement counts — the fp32 scan is certified against float64 on device.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .data import DeviceError, UnsupportedError, ValidationError


# per-query int64 diagnostics written by the replay kernel (icq_b200.h stats_dev)
STATS_FIELDS = 16
STATS_NAMES = ("insertions", "replay_candidates", "walked_items", "prologue_end",
               "prologue_cycles", "replay_cycles", "rescanned_slices", "wide_rounds",
               "prologue_f64_scored", "filter_candidates", "prologue_insertions",
               "refine_inputs", "prologue_filter_cycles", "prologue_score_cycles",
               "prologue_decide_cycles", "filter_skipped_items")


@dataclass
class OpCounter:
    """Addition counts for one query (search.py:22-34)."""

    fast_adds: int = 0
    exact_adds: int = 0
    lut_ops: int = 0
    evaluations: int = 0
    refinements: int = 0

    @property
    def total_adds(self) -> int:
        return self.fast_adds + self.exact_adds


@dataclass
class QueryResult:
    """Ranked neighbor ids and scores (ascending) plus the op counter (search.py:37-44)."""

    ids: np.ndarray
    scores: np.ndarray
    ops: OpCounter = field(default_factory=OpCounter)
    fallback: bool = False


@dataclass
class BatchResult:
    """Batched results: ids (Q, k) int64, scores (Q, k) float64, refinements (Q,)."""

    ids: np.ndarray
    scores: np.ndarray
    refinements: np.ndarray
    ops: list
    fallback: bool = False


FLAG_EXACT = 1       # icq_b200.h ICQ_FLAG_EXACT
FLAG_SIGMA_F32 = 2   # icq_b200.h ICQ_FLAG_SIGMA_F32


def _sigma_flags(sigma) -> tuple[float, int]:
    """sigma as the float64 the C ABI takes, plus the promotion flag.

    The reference computes ``bound + sigma`` (search.py:149) with whatever
    scalar type the caller passed.  A numpy float32 sigma makes numpy 2
    evaluate that sum -- and the comparison -- in float32 once the heap
    maximum is an inserted entry (NEP 50); ICQ_FLAG_SIGMA_F32 reproduces it
    on the device.  Python floats, ints and float64 stay float64; other
    reduced/extended numpy float types are rejected rather than silently
    computed differently.
    """
    if isinstance(sigma, np.floating) and not isinstance(sigma, np.float64):
        if isinstance(sigma, np.float32):
            return float(sigma), FLAG_SIGMA_F32
        raise UnsupportedError(f"sigma of type {type(sigma).__name__} is not supported "
                               "(use a Python float, np.float64 or np.float32)")
    return float(sigma), 0


def _raise(code: int, what: str):
    msg = f"{what}: {_native.last_error()}"
    if code == _native.ICQ_ERR_VALIDATION:
        raise ValidationError(msg)
    if code == _native.ICQ_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise DeviceError(msg)


def _check_query(q, d: int) -> np.ndarray:
    """search.py:47-53."""
    q = np.asarray(q, dtype=np.float64).reshape(-1)
    if q.shape != (d,):
        raise ValidationError(f"query shape {q.shape} does not match d={d}")
    if not np.all(np.isfinite(q)):
        raise ValidationError("query contains non-finite values")
    return q


def _check_queries(Q, d: int) -> np.ndarray:
    Q = np.asarray(Q, dtype=np.float64)
    if Q.ndim != 2 or Q.shape[1] != d:
        raise ValidationError(f"queries shape {Q.shape} does not match (nq, {d})")
    if not np.all(np.isfinite(Q)):
        raise ValidationError("query contains non-finite values")
    return np.ascontiguousarray(Q)


def _check_k(k: int, n: int) -> None:
    """search.py:56-58."""
    if not 1 <= k <= n:
        raise ValidationError(f"k={k} out of range [1, {n}]")


def _index_arrays(index):
    books = np.ascontiguousarray(index.books.codewords, dtype=np.float32)
    codes = index.codes.codes
    fast = np.ascontiguousarray(np.asarray(index.fast), dtype=np.uint32)
    return books, codes, fast


class DeviceIndex:
    """Device-resident index (codes repacked to uint8 fast/full row blocks).

    Owns an ``icq_index_t``.  Immutable; safe to share across threads.
    """

    def __init__(self, books: np.ndarray, codes: np.ndarray, fast: np.ndarray):
        L = _native.lib()
        books = np.ascontiguousarray(books, dtype=np.float32)
        if books.ndim != 3:
            raise ValidationError(f"codewords must be (K, m, d), got shape {books.shape}")
        K, m, d = books.shape
        codes = np.ascontiguousarray(codes)
        if codes.ndim != 2 or codes.shape[1] != K:
            raise ValidationError(f"codes must be (n, {K}), got shape {codes.shape}")
        fast = np.ascontiguousarray(np.asarray(fast), dtype=np.uint32).reshape(-1)
        h = C.c_void_p()
        n = codes.shape[0]
        if codes.dtype == np.uint8:
            st = L.icq_index_create_u8(books.ctypes.data, K, m, d, codes.ctypes.data, n,
                                       fast.ctypes.data, fast.size, C.byref(h))
        else:
            if codes.size and (codes.min() < 0):
                raise ValidationError("codes must be non-negative")
            c32 = np.ascontiguousarray(codes, dtype=np.uint32)
            st = L.icq_index_create(books.ctypes.data, K, m, d, c32.ctypes.data, n,
                                    fast.ctypes.data, fast.size, C.byref(h))
        if st != _native.ICQ_OK:
            _raise(st, "icq_index_create")
        self._h = h
        self.K, self.m, self.d, self.n, self.F = K, m, d, n, int(fast.size)
        self._fin = weakref.finalize(self, L.icq_index_destroy, h)

    @classmethod
    def from_device(cls, books: np.ndarray, codes_dev, fast: np.ndarray, stream=None):
        """Build from uint8 (n, K) codes already on the device (torch tensor)."""
        import torch

        L = _native.lib()
        books = np.ascontiguousarray(books, dtype=np.float32)
        K, m, d = books.shape
        if codes_dev.dtype != torch.uint8 or codes_dev.dim() != 2 or codes_dev.shape[1] != K:
            raise ValidationError("codes_dev must be a cuda uint8 tensor of shape (n, K)")
        codes_dev = codes_dev.contiguous()
        books_dev = torch.from_numpy(books).to(codes_dev.device)
        fast = np.ascontiguousarray(np.asarray(fast), dtype=np.uint32).reshape(-1)
        s = stream if stream is not None else torch.cuda.current_stream(codes_dev.device).cuda_stream
        h = C.c_void_p()
        st = L.icq_index_create_device(books_dev.data_ptr(), K, m, d, codes_dev.data_ptr(),
                                       codes_dev.shape[0], fast.ctypes.data, fast.size, s,
                                       C.byref(h))
        if st != _native.ICQ_OK:
            _raise(st, "icq_index_create_device")
        self = cls.__new__(cls)
        self._h = h
        self.K, self.m, self.d, self.n, self.F = K, m, d, int(codes_dev.shape[0]), int(fast.size)
        self._fin = weakref.finalize(self, L.icq_index_destroy, h)
        return self

    @classmethod
    def _adopt(cls, h, K: int, m: int, d: int, n: int, F: int):
        """Own an icq_index_t created elsewhere (icq_index_load)."""
        self = cls.__new__(cls)
        self._h = h
        self.K, self.m, self.d, self.n, self.F = K, m, d, n, F
        self._fin = weakref.finalize(self, _native.lib().icq_index_destroy, h)
        return self

    @property
    def handle(self):
        return self._h

    def read_codes(self, row0: int = 0, rows: int | None = None) -> np.ndarray:
        """(rows, K) uint8 codes back from the device."""
        rows = self.n - row0 if rows is None else rows
        out = np.empty((rows, self.K), dtype=np.uint8)
        st = _native.lib().icq_index_read_codes(self._h, row0, rows, out.ctypes.data)
        if st != _native.ICQ_OK:
            _raise(st, "icq_index_read_codes")
        return out

    def search_lut_device(self, lut, k: int, sigma: float = 0.0, exact: bool = False, out=None,
                          stats=False, stream=None, survivors=False):
        """Search on a precomputed device float64 LUT (nq, K, m); torch outputs."""
        import torch

        nq = lut.shape[0]
        dev = lut.device
        if out is None:
            out = {
                "ids": torch.empty((nq, k), dtype=torch.int64, device=dev),
                "scores": torch.empty((nq, k), dtype=torch.float64, device=dev),
                "refinements": torch.empty((nq,), dtype=torch.int64, device=dev),
            }
            if survivors:
                out["survivors"] = torch.empty((nq, (self.n + 31) // 32), dtype=torch.int32,
                                               device=dev)
            if stats:
                out["stats"] = torch.empty((nq, STATS_FIELDS), dtype=torch.int64, device=dev)
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        fb = C.c_int32(0)
        sig, flags = _sigma_flags(sigma)
        st = _native.lib().icq_search_with_lut(
            self._h, lut.data_ptr(), nq, k, sig, flags | (FLAG_EXACT if exact else 0),
            out["ids"].data_ptr(),
            out["scores"].data_ptr(), out["refinements"].data_ptr(),
            out["survivors"].data_ptr() if "survivors" in out else None,
            out["stats"].data_ptr() if "stats" in out else None, C.byref(fb), s)
        if st != _native.ICQ_OK:
            _raise(st, "icq_search_with_lut")
        out["fallback"] = bool(fb.value)
        return out

    # -- host-buffer path (used by the reference-shaped API) ------------------
    def search_host(self, Q: np.ndarray, k: int, sigma, exact: bool):
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        nq = Q.shape[0]
        ids = np.empty((nq, k), dtype=np.int64)
        scores = np.empty((nq, k), dtype=np.float64)
        refine = np.empty((nq,), dtype=np.int64)
        fb = C.c_int32(0)
        sig, flags = _sigma_flags(sigma)
        st = _native.lib().icq_search_host(self._h, Q.ctypes.data, nq, k, sig,
                                           flags | (FLAG_EXACT if exact else 0),
                                           ids.ctypes.data, scores.ctypes.data,
                                           refine.ctypes.data, C.byref(fb))
        if st != _native.ICQ_OK:
            _raise(st, "icq_search_host")
        return ids, scores, refine, bool(fb.value)

    # -- device path (torch tensors, current stream, no host sync) ------------
    def workspace_bytes(self, nq: int, k: int) -> int:
        b = C.c_size_t(0)
        st = _native.lib().icq_workspace_size(self._h, nq, k, C.byref(b))
        if st != _native.ICQ_OK:
            _raise(st, "icq_workspace_size")
        return int(b.value)

    def search_device(self, q, k: int, sigma: float = 0.0, exact: bool = False, out=None,
                      workspace=None, survivors=False, stats=False, stream=None):
        """Batched search on device tensors.  ``q``: torch float64 (nq, d) on cuda.

        Returns dict of torch tensors: ids (nq, k) int64, scores (nq, k) float64,
        refinements (nq,) int64, optionally survivors bitmap and stats.
        """
        import torch

        if q.dtype != torch.float64 or q.dim() != 2 or q.shape[1] != self.d or not q.is_cuda:
            raise ValidationError("q must be a cuda float64 tensor of shape (nq, d)")
        if not exact and _sigma_flags(sigma)[1]:  # float32 sigma: the flags entry point
            lut = self.build_lut_device(q, stream=stream)
            return self.search_lut_device(lut, k, sigma, out=out, stats=stats, stream=stream,
                                          survivors=survivors)
        q = q.contiguous()
        nq = q.shape[0]
        dev = q.device
        if out is None:
            out = {
                "ids": torch.empty((nq, k), dtype=torch.int64, device=dev),
                "scores": torch.empty((nq, k), dtype=torch.float64, device=dev),
                "refinements": torch.empty((nq,), dtype=torch.int64, device=dev),
            }
            if survivors:
                out["survivors"] = torch.empty((nq, (self.n + 31) // 32), dtype=torch.int32,
                                               device=dev)
            if stats:
                out["stats"] = torch.empty((nq, STATS_FIELDS), dtype=torch.int64, device=dev)
        need = self.workspace_bytes(nq, k)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=dev)
        s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        L = _native.lib()
        fb = C.c_int32(0)
        if exact:
            st = L.icq_search_exact(self._h, q.data_ptr(), nq, k, out["ids"].data_ptr(),
                                    out["scores"].data_ptr(), workspace.data_ptr(),
                                    workspace.numel(), s)
        else:
            st = L.icq_search_two_step(
                self._h, q.data_ptr(), nq, k, float(sigma), out["ids"].data_ptr(),
                out["scores"].data_ptr(), out["refinements"].data_ptr(),
                out["survivors"].data_ptr() if "survivors" in out else None,
                out["stats"].data_ptr() if "stats" in out else None, C.byref(fb),
                workspace.data_ptr(), workspace.numel(), s)
        if st != _native.ICQ_OK:
            _raise(st, "icq_search")
        if exact:  # search_exact refines every element (search.py:108)
            out["refinements"].fill_(self.n)
        out["fallback"] = bool(fb.value)
        return out

    def build_lut_device(self, q, stream=None):
        import torch

        q = q.contiguous()
        lut = torch.empty((q.shape[0], self.K, self.m), dtype=torch.float64, device=q.device)
        s = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
        st = _native.lib().icq_build_lut(self._h, q.data_ptr(), q.shape[0], lut.data_ptr(), s)
        if st != _native.ICQ_OK:
            _raise(st, "icq_build_lut")
        return lut


# ---------------------------------------------------------------------------
# per-SearchIndex device cache (SearchIndex is immutable by contract, SPEC 446)
# ---------------------------------------------------------------------------
_cache: dict = {}
_cache_lock = threading.Lock()


def device_index(index) -> DeviceIndex:
    """The DeviceIndex for a (reference or local) SearchIndex, uploaded once."""
    dev = getattr(index, "_device", None)  # io.load_index: already on the device
    if isinstance(dev, DeviceIndex):
        return dev
    books = index.books.codewords
    codes = index.codes.codes
    fast = np.asarray(index.fast)
    key = id(index)
    sig = (id(books), id(codes), tuple(int(x) for x in fast))
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None and hit[0] == sig:
            return hit[1]
    b, c, f = _index_arrays(index)
    if c.dtype != np.uint8 and int(index.cfg.m) <= 256:
        c = c.astype(np.uint8)
    dev = DeviceIndex(b, c, f)
    with _cache_lock:
        _cache[key] = (sig, dev)
        try:
            weakref.finalize(index, _cache.pop, key, None)
        except TypeError:
            pass
    return dev


def _ops_two_step(index, R: int, k: int) -> OpCounter:
    K, m, d, n = index.cfg.K, index.cfg.m, index.d, index.n
    F = int(np.asarray(index.fast).size)
    return OpCounter(fast_adds=(F - 1) * n, exact_adds=(K - 1) * (R + k), lut_ops=K * m * d,
                     evaluations=n, refinements=R)


def _ops_exact(index) -> OpCounter:
    K, m, d, n = index.cfg.K, index.cfg.m, index.d, index.n
    return OpCounter(exact_adds=(K - 1) * n, lut_ops=K * m * d, evaluations=n, refinements=n)


# ---------------------------------------------------------------------------
# reference-shaped API
# ---------------------------------------------------------------------------
def build_lut(index, q, ops: OpCounter | None = None) -> np.ndarray:
    """(K, m) float64 table of squared distances from q to every codeword (search.py:61-69)."""
    import torch

    q = _check_query(q, index.d)
    dev = device_index(index)
    lut = dev.build_lut_device(torch.from_numpy(q[None]).cuda())
    torch.cuda.current_stream().synchronize()
    if ops is not None:
        ops.lut_ops += index.cfg.K * index.cfg.m * index.d
    return lut[0].cpu().numpy()


def exact_score(lut: np.ndarray, code_row, ops: OpCounter | None = None) -> float:
    """Full reconstruction score of one row (search.py:72-78)."""
    K = lut.shape[0]
    score = float(np.sum(lut[np.arange(K), np.asarray(code_row)]))
    if ops is not None:
        ops.exact_adds += K - 1
    return score


def fast_score(lut: np.ndarray, code_row, fast, ops: OpCounter | None = None) -> float:
    """Partial score over the fast books of one row (search.py:81-89)."""
    fast = np.asarray(fast)
    score = float(np.sum(lut[fast, np.asarray(code_row)[fast]]))
    if ops is not None:
        ops.fast_adds += max(len(fast) - 1, 0)
    return score


def search_exact(index, q, k: int) -> QueryResult:
    """Scan every element with the full score; k best by (score, id) (search.py:97-109)."""
    _check_k(k, index.n)
    q = _check_query(q, index.d)
    ids, scores, _, _ = device_index(index).search_host(q[None], k, 0.0, exact=True)
    return QueryResult(ids=ids[0], scores=scores[0], ops=_ops_exact(index))


def search_two_step(index, q, k: int, sigma: float | None = None) -> QueryResult:
    """Prune with fast scores against the heap maximum, refine the rest (search.py:112-165)."""
    _check_k(k, index.n)
    if sigma is None:
        sigma = index.sigma
    if not sigma >= 0:
        raise ValidationError(f"sigma must be >= 0, got {sigma}")
    if np.asarray(index.fast).size == 0:
        res = search_exact(index, q, k)
        res.fallback = True
        return res
    q = _check_query(q, index.d)
    ids, scores, refine, _ = device_index(index).search_host(q[None], k, sigma, exact=False)
    R = int(refine[0])
    return QueryResult(ids=ids[0], scores=scores[0], ops=_ops_two_step(index, R, k))


def search_two_step_batch(index, queries, k: int, sigma: float | None = None) -> BatchResult:
    """All queries in one device call (host buffers in, host buffers out)."""
    _check_k(k, index.n)
    if sigma is None:
        sigma = index.sigma
    if not sigma >= 0:
        raise ValidationError(f"sigma must be >= 0, got {sigma}")
    Q = _check_queries(queries, index.d)
    exact = np.asarray(index.fast).size == 0
    ids, scores, refine, fb = device_index(index).search_host(Q, k, sigma, exact=exact)
    if exact:
        ops = [_ops_exact(index) for _ in range(Q.shape[0])]
        refine = np.full(Q.shape[0], index.n, dtype=np.int64)
    else:
        ops = [_ops_two_step(index, int(r), k) for r in refine]
    return BatchResult(ids=ids, scores=scores, refinements=refine, ops=ops, fallback=exact)


def search_exact_batch(index, queries, k: int) -> BatchResult:
    _check_k(k, index.n)
    Q = _check_queries(queries, index.d)
    ids, scores, _, _ = device_index(index).search_host(Q, k, 0.0, exact=True)
    n = index.n
    return BatchResult(ids=ids, scores=scores, refinements=np.full(Q.shape[0], n, dtype=np.int64),
                       ops=[_ops_exact(index) for _ in range(Q.shape[0])])


# ---------------------------------------------------------------------------
# brute-force ground truth (search.py:168-178)
# ---------------------------------------------------------------------------
class DeviceDataset:
    """Raw float32 vectors resident on the device (the brute-force scan's input)."""

    def __init__(self, vectors):
        import torch

        if isinstance(vectors, torch.Tensor):
            x = vectors
            if x.dtype != torch.float32 or x.dim() != 2:
                raise ValidationError("vectors must be a float32 (n, d) tensor")
            self.x = x.contiguous() if x.is_cuda else x.contiguous().cuda()
        else:
            x = np.ascontiguousarray(np.asarray(vectors), dtype=np.float32)
            if x.ndim != 2:
                raise ValidationError(f"vectors must be 2-d, got shape {x.shape}")
            self.x = torch.from_numpy(x).cuda()
        self.n, self.d = int(self.x.shape[0]), int(self.x.shape[1])

    def search_device(self, q, k: int, stream=None):
        """Batched scan: q torch float64 (nq, d) on cuda -> ids (nq, k), scores (nq, k)."""
        import torch

        _check_k(k, self.n)
        if q.dtype != torch.float64 or q.dim() != 2 or q.shape[1] != self.d or not q.is_cuda:
            raise ValidationError("q must be a cuda float64 tensor of shape (nq, d)")
        q = q.contiguous()
        nq = q.shape[0]
        ids = torch.empty((nq, k), dtype=torch.int64, device=q.device)
        scores = torch.empty((nq, k), dtype=torch.float64, device=q.device)
        s = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
        st = _native.lib().icq_bruteforce(self.x.data_ptr(), self.n, self.d, q.data_ptr(), nq, k,
                                          ids.data_ptr(), scores.data_ptr(), s)
        if st != _native.ICQ_OK:
            _raise(st, "icq_bruteforce")
        return {"ids": ids, "scores": scores}


_ds_cache: dict = {}


def _device_dataset(ds) -> DeviceDataset:
    if isinstance(ds, DeviceDataset):
        return ds
    x = ds.vectors if hasattr(ds, "vectors") else np.asarray(ds)
    key = id(x)
    hit = _ds_cache.get(key)
    if hit is not None and hit[0] is x:
        return hit[1]
    dd = DeviceDataset(x)
    _ds_cache.clear()  # one raw dataset at a time (they are large)
    _ds_cache[key] = (x, dd)
    return dd


def search_bruteforce(ds, q, k: int) -> QueryResult:
    """Exact squared Euclidean scan over raw vectors (search.py:168-178), on the GPU."""
    import torch

    dd = _device_dataset(ds)
    _check_k(k, dd.n)
    q = _check_query(q, dd.d)
    out = dd.search_device(torch.from_numpy(q[None]).cuda(), k)
    ops = OpCounter(exact_adds=(dd.d - 1) * dd.n, evaluations=dd.n, refinements=dd.n)
    return QueryResult(ids=out["ids"][0].cpu().numpy(), scores=out["scores"][0].cpu().numpy(),
                       ops=ops)


def search_bruteforce_batch(ds, queries, k: int) -> BatchResult:
    import torch

    dd = _device_dataset(ds)
    _check_k(k, dd.n)
    Q = _check_queries(queries, dd.d)
    out = dd.search_device(torch.from_numpy(Q).cuda(), k)
    ops = [OpCounter(exact_adds=(dd.d - 1) * dd.n, evaluations=dd.n, refinements=dd.n)
           for _ in range(Q.shape[0])]
    return BatchResult(ids=out["ids"].cpu().numpy(), scores=out["scores"].cpu().numpy(),
                       refinements=np.full(Q.shape[0], dd.n, dtype=np.int64), ops=ops)
