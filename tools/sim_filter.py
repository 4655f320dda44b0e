"""Design probe (not product, not a test): how many items each candidate filter
passes on a bench workload, next to the reference's refined set.

For a few queries it computes float64 fast/exact scores of every item with
torch (GPU), replays search.py:140-154 in chunks (numpy, insertion by
insertion) and records the trajectory of bound, T and
U = max(max fast over the heap, T - Smin).  It then counts
the items a parallel filter would pass with

  * U at the end of a prologue of P items, for every later item;
  * block-stale thresholds: block b filtered with U at the end of block b-lag;

    python tools/sim_filter.py --config c4 --queries 4
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--queries", type=int, default=4)
    ap.add_argument("--sigma", type=float, default=None)
    ap.add_argument("--n", type=int, default=0, help="truncate the database (0 = full)")
    ap.add_argument("--sweeps", type=int, default=10)
    ap.add_argument("--only", type=str, default="", help="comma-separated query indices")
    args = ap.parse_args()

    import torch

    from tools.workloads import CONFIGS, build_database, index_rule, load_books, queries

    w = CONFIGS[args.config]
    books, meta = load_books(w)
    fast_books, sigma, _, _ = index_rule(w, meta, args.sigma)
    codes = build_database(w, books, sweeps=args.sweeps)
    if args.n:
        codes = codes[:args.n]
    n = codes.shape[0]
    Q = queries(w)[:args.queries]
    B = torch.as_tensor(books, device="cuda", dtype=torch.float64)
    ci = codes.long()
    fb = torch.as_tensor(fast_books.astype(np.int64), device="cuda")
    slow = torch.as_tensor([b for b in range(w.K) if b not in set(fast_books.tolist())],
                           device="cuda", dtype=torch.long)
    out = []
    sel = [int(x) for x in args.only.split(",")] if args.only else list(range(Q.shape[0]))
    for qi in sel:
        q = Q[qi]
        lut = ((B - q[None, None, :]) ** 2).sum(-1)  # (K, m)
        fast = torch.zeros(n, dtype=torch.float64, device="cuda")
        for b in fb.tolist():
            fast += lut[b][ci[:, b]]
        exact = torch.zeros(n, dtype=torch.float64, device="cuda")
        for b in range(w.K):
            exact += lut[b][ci[:, b]]
        smin = float(lut[slow].min(1).values.sum()) if slow.numel() else 0.0
        f = fast.cpu().numpy()
        e = exact.cpu().numpy()
        refined, ins_pos, U_at, T_at, B_at, hi, he, M_at = replay(f, e, w.k, sigma, smin)
        R = int(refined.sum())
        res = {"q": qi, "n": n, "refined": R, "insertions": len(ins_pos) - 1,
               "last_insertion": int(ins_pos[-1]),
               "insertions_after": {str(P): int((ins_pos >= P).sum()) for P in
                                    (1 << 14, 1 << 16, 1 << 18, 1 << 20, 1 << 22)}}

        def U_before(p):
            # U in force when item p is examined (after all insertions < p)
            j = np.searchsorted(ins_pos, p, side="left") - 1
            return U_at[max(j, 0)]

        # U at the end of a prologue of P items
        cands = {}
        for P in (1 << 14, 1 << 16, 1 << 18, 1 << 20):
            if P >= n:
                continue
            u = U_before(P) + sigma
            cands[str(P)] = int((f[P:] < u).sum())
        res["cand_after_prologue"] = cands
        if sigma == 0.0:
            # sigma = 0: M = max fast over the heap is itself non-increasing
            mc = {}
            for P in (1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20):
                if P >= n:
                    continue
                j = np.searchsorted(ins_pos, P, side="left") - 1
                mc[str(P)] = int((f[P:] < M_at[max(j, 0)]).sum())
            res["cand_after_prologue_M"] = mc
            j = np.searchsorted(ins_pos, np.arange(n), side="left") - 1
            res["cand_live_M"] = int((f < M_at[np.maximum(j, 0)]).sum())
            res["final_M"] = float(M_at[-1])
        # block-stale: block b filtered with U before block b-lag
        blk = {}
        for bs in (1 << 16, 1 << 18, 1 << 20):
            for lag in (1, 2):
                tot = 0
                for s in range(0, n, bs):
                    src = max(0, s - (lag - 1) * bs)
                    u = U_before(src) + sigma
                    tot += int((f[s:s + bs] < u).sum())
                blk[f"{bs}/{lag}"] = tot
        res["cand_block_stale"] = blk
        # live threshold candidates (U at item i) = best possible superset
        j = np.searchsorted(ins_pos, np.arange(n), side="left") - 1
        ulive = U_at[np.maximum(j, 0)] + sigma
        res["cand_live_U"] = int((f < ulive).sum())
        blive = B_at[np.maximum(j, 0)] + sigma
        res["cand_live_bound"] = int((f < blive).sum())
        res["final_T"] = float(T_at[-1])
        res["final_U"] = float(U_at[-1])
        res["smin"] = smin
        out.append(res)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
