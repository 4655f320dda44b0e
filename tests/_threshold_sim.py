"""Chunked restatement of the reference loop (search.py:140-154) that also
records the heap state after every insertion -- test infrastructure for the
stale-threshold properties (tests/test_threshold_theory.py)."""

import numpy as np


def replay(fast, exact, k, sigma, smin):
    """Chunked exact replay; returns refined mask and U/T/bound after each item
    (as step arrays at the insertion positions)."""
    n = fast.shape[0]
    order = np.lexsort((-np.arange(k), -exact[:k]))  # descending by (exact, id)
    he = exact[:k][order].copy()
    hi = np.arange(k)[order].copy()
    hf = fast[:k][order].copy()
    refined = np.zeros(n, dtype=bool)
    ins_pos = [k - 1]
    U_at = [max(hf.max(), he[0] - smin)]
    M_at = [hf.max()]
    T_at = [he[0]]
    B_at = [hf[0]]
    pos = k
    C = 256
    while pos < n:
        end = min(n, pos + C)
        f = fast[pos:end]
        e = exact[pos:end]
        thr = hf[0] + sigma
        ref = f < thr
        ins = ref & (e < he[0])
        if not ins.any():
            refined[pos:end] = ref
            pos = end
            C = min(C * 2, 1 << 20)
            continue
        j = int(np.argmax(ins))
        refined[pos:pos + j + 1] = ref[:j + 1]
        i = pos + j
        # replace the max (entry 0) and keep the array sorted descending
        xe, xi, xf = exact[i], i, fast[i]
        he, hi, hf = he[1:], hi[1:], hf[1:]
        # position: entries with key > x stay before it
        gt = (he > xe) | ((he == xe) & (hi > xi))
        g = int(gt.sum())
        he = np.insert(he, g, xe)
        hi = np.insert(hi, g, xi)
        hf = np.insert(hf, g, xf)
        ins_pos.append(i)
        U_at.append(max(hf.max(), he[0] - smin))
        M_at.append(hf.max())
        T_at.append(he[0])
        B_at.append(hf[0])
        pos = i + 1
        C = 256
    return refined, np.array(ins_pos), np.array(U_at), np.array(T_at), np.array(B_at), hi, he, np.array(M_at)
