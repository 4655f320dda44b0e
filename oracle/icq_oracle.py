"""CPU oracle for the ICQ query path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the reference query engines of
``/root/reference/pkg/src/icq/search.py`` so the GPU path can be checked
against them.  It is imported only by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference``).  The
product package ``paper_1912_08756_b200`` never imports it; the product path
fails loudly when its CUDA library is missing.

Pinning: ``tests/golden/*.npz`` hold outputs of the real reference (generated
in the build container by ``tests/golden/make_golden.py`` with the reference
importable from ``/root/reference/pkg/src``); ``tests/test_oracle_golden.py``
asserts this oracle reproduces them bit for bit (ids, float64 scores,
refinement counts and op counters).

What it restates (reference file:line):

* ``lut``            — ``build_lut`` search.py:61-69: float64 direct difference,
                       ``(diff*diff).sum(axis=2)`` (numpy pairwise order).
* ``gather``         — ``_gather_scores`` search.py:92-94.
* ``two_step``       — ``search_two_step`` search.py:112-165: heap seeded with
                       ids 0..k-1 (:141-143), element i refined iff
                       ``fast[i] < bound + sigma`` where bound is the FAST score
                       of the current (exact, id) heap maximum (:149, :154),
                       inserted iff ``exact[i] < exact(heap max)`` (:152).
                       Instrumented: also returns the survivor (refined) ids,
                       which the reference only counts (:150).
* ``exact``          — ``search_exact`` search.py:97-109 (lexsort by score, id).
* ``pairwise_sum``   — numpy's float64 ``add.reduce`` order (identity 0 plus
                       pairwise blocks of 8 up to 128, recursive halving above),
                       written out so the CUDA kernels can mirror it exactly.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np


class OracleValidationError(ValueError):
    """Mirrors icq.data.ValidationError (data.py:32) for the oracle's checks."""


# ----------------------------------------------------------------------------
# numpy float64 add.reduce order, restated (numpy pairwise_sum; used by
# search.py:66 and :94).  Checked bitwise against ndarray.sum in the tests.
# ----------------------------------------------------------------------------
def pairwise_sum(a) -> float:
    a = [float(x) for x in a]
    return 0.0 + _pw(a, 0, len(a))


def _pw(a, lo, n):
    if n < 8:
        r = 0.0
        for i in range(n):
            r += a[lo + i]
        return r
    if n <= 128:
        r = [a[lo + j] for j in range(8)]
        i = 8
        top = n - (n % 8)
        while i < top:
            for j in range(8):
                r[j] += a[lo + i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += a[lo + i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _pw(a, lo, n2) + _pw(a, lo + n2, n - n2)


def pairwise_leaves(n: int):
    """Leaf ranges and postfix combine program of numpy's pairwise sum over n
    elements: returns list of ('leaf', start, length) / ('add',) ops."""
    prog = []

    def rec(lo, m):
        if m <= 128:
            prog.append(("leaf", lo, m))
            return
        m2 = m // 2
        m2 -= m2 % 8
        rec(lo, m2)
        rec(lo + m2, m - m2)
        prog.append(("add",))

    rec(0, n)
    return prog


# ----------------------------------------------------------------------------
# Engines
# ----------------------------------------------------------------------------
@dataclass
class OracleOps:
    fast_adds: int = 0
    exact_adds: int = 0
    lut_ops: int = 0
    evaluations: int = 0
    refinements: int = 0

    @property
    def total_adds(self) -> int:
        return self.fast_adds + self.exact_adds


@dataclass
class OracleResult:
    ids: np.ndarray
    scores: np.ndarray
    ops: OracleOps = field(default_factory=OracleOps)
    fallback: bool = False
    survivors: np.ndarray | None = None  # refined ids in scan order (two-step only)


def check_query(q, d: int) -> np.ndarray:
    """search.py:47-53."""
    q = np.asarray(q, dtype=np.float64).reshape(-1)
    if q.shape != (d,):
        raise OracleValidationError(f"query shape {q.shape} does not match d={d}")
    if not np.all(np.isfinite(q)):
        raise OracleValidationError("query contains non-finite values")
    return q


def check_k(k: int, n: int) -> None:
    """search.py:56-58."""
    if not 1 <= k <= n:
        raise OracleValidationError(f"k={k} out of range [1, {n}]")


def lut(books: np.ndarray, q) -> np.ndarray:
    """(K, m) float64 table of squared distances (search.py:61-69)."""
    books = np.asarray(books)
    q = check_query(q, books.shape[2])
    diff = books.astype(np.float64) - q[None, None, :]
    return (diff * diff).sum(axis=2)


def gather(table: np.ndarray, codes: np.ndarray, books: np.ndarray) -> np.ndarray:
    """Per-row sums of table entries over the given book columns (search.py:92-94)."""
    books = np.asarray(books, dtype=np.int64)
    return table[books[None, :], codes[:, books]].sum(axis=1)


def exact(books: np.ndarray, codes: np.ndarray, q, k: int) -> OracleResult:
    """search_exact, search.py:97-109."""
    codes = np.asarray(codes)
    n, K = codes.shape
    check_k(k, n)
    table = lut(books, q)
    m, d = books.shape[1], books.shape[2]
    scores = gather(table, codes, np.arange(K))
    order = np.lexsort((np.arange(n), scores))[:k]
    ops = OracleOps(exact_adds=(K - 1) * n, lut_ops=K * m * d, evaluations=n, refinements=n)
    return OracleResult(ids=order.astype(np.int64), scores=scores[order], ops=ops)


def _refine_mask(fs, bound, max_id, sigma, k):
    """``fs < bound + sigma`` with the reference's scalar types (search.py:149).

    The reference's heap caches np.float64 fast scores for the seeds
    (search.py:141, ``fast_all[i]``) and Python floats for inserted entries
    (:153, ``fast_list[i]``).  With a numpy float32 sigma, numpy 2 (NEP 50)
    computes ``bound + sigma`` in float32 when bound is a Python float and then
    compares ``fast_list[i] < float32`` in float32 too; with an np.float64
    bound everything stays float64.
    """
    if isinstance(sigma, np.float32) and max_id >= k:
        thr32 = np.float32(bound) + sigma
        return fs.astype(np.float32) < thr32
    return fs < bound + float(sigma)


def two_step(books, codes, fast, sigma, q, k: int, chunk: int = 4096) -> OracleResult:
    """search_two_step, search.py:112-165, instrumented with the survivor list.

    The prune loop is evaluated chunk-wise: within a chunk the heap (hence
    ``bound`` and the heap-max exact score ``T``) is constant until the first
    insertion, so every element before that insertion is decided by the same
    predicate (search.py:149) — identical to the element-by-element loop,
    which ``two_step_loop`` restates literally and the tests compare against.
    """
    codes = np.asarray(codes)
    n, K = codes.shape
    check_k(k, n)
    if not sigma >= 0:
        raise OracleValidationError(f"sigma must be >= 0, got {sigma}")
    fast = np.asarray(fast).astype(np.int64)
    if fast.size == 0:
        res = exact(books, codes, q, k)
        res.fallback = True
        return res
    table = lut(books, q)
    m, d = books.shape[1], books.shape[2]
    fast_all = gather(table, codes, fast)
    exact_all = gather(table, codes, np.arange(K))

    heap = [(-float(exact_all[i]), -i, float(fast_all[i])) for i in range(k)]
    heapq.heapify(heap)
    bound = heap[0][2]
    survivors = []
    pos = k
    while pos < n:
        end = min(n, pos + chunk)
        fs = fast_all[pos:end]
        es = exact_all[pos:end]
        while pos < end:
            off = pos - (end - len(fs))
            refined = _refine_mask(fs[off:], bound, -heap[0][1], sigma, k)
            ins = refined & (es[off:] < -heap[0][0])
            hit = np.flatnonzero(ins)
            stop = off + (int(hit[0]) + 1 if hit.size else len(fs) - off)
            survivors.extend((np.flatnonzero(refined[: stop - off]) + pos).tolist())
            if hit.size:
                i = pos + int(hit[0])
                heapq.heapreplace(heap, (-float(exact_all[i]), -i, float(fast_all[i])))
                bound = heap[0][2]
            pos = (end - len(fs)) + stop
    ranked = sorted((-e[0], -e[1]) for e in heap)
    R = len(survivors)
    ops = OracleOps(
        fast_adds=(fast.size - 1) * n,
        exact_adds=(K - 1) * (R + k),
        lut_ops=K * m * d,
        evaluations=n,
        refinements=R,
    )
    return OracleResult(
        ids=np.array([i for _, i in ranked], dtype=np.int64),
        scores=np.array([s for s, _ in ranked], dtype=np.float64),
        ops=ops,
        survivors=np.asarray(survivors, dtype=np.int64),
    )


def two_step_loop(books, codes, fast, sigma, q, k: int) -> OracleResult:
    """Literal element-by-element restatement of search.py:140-154 (slow)."""
    codes = np.asarray(codes)
    n, K = codes.shape
    check_k(k, n)
    fast = np.asarray(fast).astype(np.int64)
    if fast.size == 0:
        res = exact(books, codes, q, k)
        res.fallback = True
        return res
    table = lut(books, q)
    fast_all = gather(table, codes, fast)
    exact_all = gather(table, codes, np.arange(K))
    # seeds cache numpy scalars, inserted entries Python floats (search.py:141, :153)
    heap = [(-exact_all[i], -i, fast_all[i]) for i in range(k)]
    heapq.heapify(heap)
    fl = fast_all.tolist()
    el = exact_all.tolist()
    bound = heap[0][2]
    survivors = []
    for i in range(k, n):
        if fl[i] < bound + sigma:
            survivors.append(i)
            if el[i] < -heap[0][0]:
                heapq.heapreplace(heap, (-el[i], -i, fl[i]))
                bound = heap[0][2]
    ranked = sorted((-e[0], -e[1]) for e in heap)
    m, d = books.shape[1], books.shape[2]
    R = len(survivors)
    ops = OracleOps((fast.size - 1) * n, (K - 1) * (R + k), K * m * d, n, R)
    return OracleResult(
        ids=np.array([i for _, i in ranked], dtype=np.int64),
        scores=np.array([s for s, _ in ranked], dtype=np.float64),
        ops=ops,
        survivors=np.asarray(survivors, dtype=np.int64),
    )


def bruteforce(x, q, k: int) -> OracleResult:
    """search_bruteforce, search.py:168-178: float64 direct difference over raw
    vectors (numpy pairwise order along d), lexsort by (score, id)."""
    x = np.asarray(x)
    n, d = x.shape
    check_k(k, n)
    q = check_query(q, d)
    diff = x.astype(np.float64) - q[None, :]
    scores = (diff * diff).sum(axis=1)
    order = np.lexsort((np.arange(n), scores))[:k]
    ops = OracleOps(exact_adds=(d - 1) * n, evaluations=n, refinements=n)
    return OracleResult(ids=order.astype(np.int64), scores=scores[order], ops=ops)
