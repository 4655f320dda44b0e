"""Per-query pruning diagnostics on a BASELINE workload (GPU box; not product).

    python tools/diag_query.py c5 [--sigma S] [--nq 512] [--deep 6]

Runs one batch through the device pipeline with stats, prints the per-query
stat distribution, then for the heaviest queries (by replay cycles) and a few
typical ones replays search.py:148-154 on the host from device-computed
float64 fast/exact scores, reporting where the insertions fall after the
prologue end P and how many items each threshold would pass: the stale M at
P, the final live bound, and the maximum live bound seen after P.
"""

from __future__ import annotations

import argparse
import heapq
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from tools.workloads import CONFIGS, build_database, index_rule, load_books, queries  # noqa: E402


def host_trajectory(fast, exact, k, sigma, P, heap_at_P=None):
    heap = [(-float(exact[i]), -i, float(fast[i])) for i in range(k)]
    heapq.heapify(heap)
    bound = heap[0][2]
    pos = k
    n = fast.shape[0]
    traj = []
    M_at_P = None
    chunk = 1 << 16
    while pos < n:
        if M_at_P is None and pos >= P:
            M_at_P = max(e[2] for e in heap)
            if heap_at_P is not None:
                heap_at_P.extend(sorted(((-e[0], -e[1], e[2]) for e in heap), reverse=True))
        end = min(n, pos + chunk)
        if M_at_P is None and end > P:
            end = P
        fs = fast[pos:end]
        es = exact[pos:end]
        off = 0
        while off < fs.shape[0]:
            thr = bound + sigma
            ref = fs[off:] < thr
            ins = ref & (es[off:] < -heap[0][0])
            hit = np.flatnonzero(ins)
            if hit.size == 0:
                break
            i = pos + off + int(hit[0])
            heapq.heapreplace(heap, (-float(exact[i]), -i, float(fast[i])))
            bound = heap[0][2]
            traj.append((i, bound, -heap[0][0]))
            off += int(hit[0]) + 1
        pos = end
    return traj, M_at_P


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--sigma", type=float, default=None)
    ap.add_argument("--nq", type=int, default=0)
    ap.add_argument("--deep", type=int, default=6)
    args = ap.parse_args()
    import torch

    import paper_1912_08756_b200 as icqb
    from paper_1912_08756_b200.search import STATS_NAMES

    w = CONFIGS[args.config]
    books, meta = load_books(w)
    fast, sigma, _, _ = index_rule(w, meta, args.sigma)
    codes = build_database(w, books, sweeps=10)
    Qall = queries(w)
    nq = args.nq or w.batch
    qb = Qall[:nq]
    dev = icqb.DeviceIndex.from_device(books, codes, fast)
    lut = dev.build_lut_device(qb)
    out = dev.search_lut_device(lut, w.k, sigma, stats=True)
    torch.cuda.synchronize()
    st = out["stats"].cpu().numpy()
    ref = out["refinements"].cpu().numpy()
    S = {nm: st[:, i] for i, nm in enumerate(STATS_NAMES)}
    pct = lambda a: [float(np.percentile(a, p)) for p in (0, 50, 90, 99, 100)]
    print(json.dumps({nm: pct(v) for nm, v in S.items()} | {"refinements": pct(ref)}, indent=0))
    order = np.argsort(-S["replay_cycles"])
    for qi in order[:12]:
        print("heavy", int(qi), {nm: int(S[nm][qi]) for nm in STATS_NAMES}, "refined", int(ref[qi]))
    if args.deep <= 0:
        return
    pick = list(order[: args.deep]) + list(order[len(order) // 2: len(order) // 2 + 2])
    K = w.K
    fidx = torch.as_tensor(fast.astype(np.int64), device="cuda")
    for qi in pick:
        L = lut[qi]  # (K, m) float64
        cl = codes.long()
        # fast sums in the reference's order (sequential in book order)
        f = torch.zeros(w.n, dtype=torch.float64, device="cuda")
        for b in fidx.tolist():
            f += L[b][cl[:, b]]
        e = torch.zeros(w.n, dtype=torch.float64, device="cuda")
        for b in range(K):
            e += L[b][cl[:, b]]
        fh, eh = f.cpu().numpy(), e.cpu().numpy()
        P = int(S["prologue_end"][qi])
        hP = []
        traj, M = host_trajectory(fh, eh, w.k, sigma, P, hP)
        after = [t for t in traj if t[0] >= P]
        bmax = max([t[1] for t in after], default=None)
        rest = fh[P:]
        row = {"q": int(qi), "P": P, "replay_cycles": int(S["replay_cycles"][qi]),
               "skipped": int(S["filter_skipped_items"][qi]),
               "refinements": int(ref[qi]), "insertions_total": len(traj),
               "insertions_after_P": len(after),
               "first_ins_after_P": [int(t[0]) for t in after[:12]],
               "M_at_P": M, "pass_M": int((rest < M + sigma).sum()),
               "bound_at_P": float(traj[-len(after) - 1][1]) if len(after) < len(traj) else None,
               "pass_bound_final": int((rest < traj[-1][1] + sigma).sum()) if traj else None,
               "max_bound_after_P": bmax,
               "pass_max_bound_after_P": int((rest < bmax + sigma).sum()) if bmax else None,
               "fast_pct": [float(np.percentile(rest, p)) for p in (0.01, 0.1, 1, 10, 50)]}
        # policies: filter threshold theta = A_J(heap at P) + sigma; the replay
        # walks item by item while the live bound + sigma exceeds theta
        pol = {}
        for J in (0, 2, 8, 32, w.k - 1):
            A = max(e[2] for e in hP[: J + 1])
            theta = A + sigma
            walked, spikes, start = 0, 0, None
            for (i, b, _) in after:
                if b + sigma > theta and start is None:
                    start, spikes = i, spikes + 1
                elif b + sigma <= theta and start is not None:
                    walked += i - start
                    start = None
            if start is not None:
                walked += w.n - start
            pol[J] = {"list": int((rest < theta).sum()), "spikes": spikes, "walked": walked}
        row["policies"] = pol
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
