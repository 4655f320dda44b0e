"""CPU property tests of the stale filter thresholds the GPU pipeline relies on
(icq_common.cuh stale_core, icq_pipeline.cuh budgeted A_J), checked against
the reference loop (search.py:140-154) on seeded random indices with ties.

For every item i refined by the reference (fast_i < bound_i + sigma):
  * sigma == 0: fast_i < M_s for every earlier state s (M = max fast over the
    heap never increases), so M_P filters a superset of the refined items;
  * any sigma:  fast_i < U_s + sigma, U = max(M, T - Smin);
  * budget:     if at most J insertions happen in (s, i], then
                fast_i < A_J(s) = max fast over the J+1 largest-exact heap
                entries at s (sigma == 0).
"""

import numpy as np
import pytest

from _threshold_sim import replay


def _case(seed, n, K, F, m, dup):
    rng = np.random.default_rng(seed)
    d = 6
    books = rng.standard_normal((K, m, d))
    books[:F] *= 3.0
    codes = rng.integers(0, m, size=(n, K))
    if dup:
        codes[1::3] = codes[0::3][: len(codes[1::3])]
    q = rng.standard_normal(d)
    lut = ((books - q) ** 2).sum(-1)
    fast = lut[np.arange(F)[None, :], codes[:, :F]].sum(1)
    exact = lut[np.arange(K)[None, :], codes].sum(1)
    smin = lut[F:].min(1).sum() if F < K else 0.0
    return fast, exact, smin


def _trajectory(fast, exact, k, sigma):
    """Heap states after each insertion (sorted descending by (exact, id))."""
    n = fast.shape[0]
    order = np.lexsort((-np.arange(k), -exact[:k]))
    heap = [(exact[i], i, fast[i]) for i in order]  # descending
    states = [(k - 1, list(heap))]
    refined = []
    for i in range(k, n):
        bound = heap[0][2]
        if fast[i] < bound + sigma:
            refined.append(i)
            if exact[i] < heap[0][0]:
                heap = heap[1:] + [(exact[i], i, fast[i])]
                heap.sort(key=lambda t: (-t[0], -t[1]))
                states.append((i, list(heap)))
    return refined, states


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("sigma", [0.0, 1.0, 25.0])
def test_stale_thresholds_cover_refined_items(seed, sigma):
    n, K, F, m, k = 1500, 6, 2, 8, 10
    fast, exact, smin = _case(seed, n, K, F, m, dup=seed % 2 == 0)
    refined, states = _trajectory(fast, exact, k, sigma)
    # cross-check the sim's chunked replay (also used by the design probes)
    r = replay(fast, exact, k, sigma, smin)
    assert int(r[0].sum()) == len(refined)
    pos = np.array([s[0] for s in states])
    for si, (p0, heap) in enumerate(states):
        M = max(t[2] for t in heap)
        T = heap[0][0]
        U = max(M, T - smin)
        later = [i for i in refined if i > p0]
        for i in later:
            assert fast[i] < U + sigma + 1e-9 * abs(U)
            if sigma == 0.0:
                assert fast[i] < M
        if sigma == 0.0:
            for J in (0, 1, 3):
                AJ = max(t[2] for t in heap[: J + 1])
                for i in later:
                    ins_between = int(((pos > p0) & (pos < i)).sum())
                    if ins_between <= J:
                        assert fast[i] < AJ, (seed, J, i)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("sigma", [0.0, 1.0, 25.0, 1e9])
def test_count_mode_candidates_cover_insertions(seed, sigma):
    """Count mode lists only possible insertions: an item inserted after state
    s has exact < T_s and therefore fast < T_s - Smin (slow part >= Smin) --
    whatever sigma is (icq_pipeline.cuh prologue hand-off, count mode)."""
    n, K, F, m, k = 1500, 6, 2, 8, 10
    fast, exact, smin = _case(seed, n, K, F, m, dup=seed % 3 == 0)
    _, states = _trajectory(fast, exact, k, sigma)
    inserted = [s[0] for s in states[1:]]
    for p0, heap in states:
        T = heap[0][0]
        for i in inserted:
            if i > p0:
                assert exact[i] < T
                assert fast[i] < T - smin + 1e-9 * abs(T)
