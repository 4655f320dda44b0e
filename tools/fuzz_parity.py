"""Randomised parity soak (run on the GPU box): random index shapes, margins,
k and planning knobs through the C ABI, against the oracle -- ids, float64
scores, refinement counts and survivor sets, bitwise.

    python tools/fuzz_parity.py [seconds] [seed]      (FUZZ_BIG=1: 120k - 1.2M items)
"""
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402

import paper_1912_08756_b200 as icqb  # noqa: E402
from oracle import icq_oracle as O  # noqa: E402

KNOBS = {
    "ICQ_COUNT_MODE": ["0", "1"],
    "ICQ_CM_PREFIX": ["0", "3000", "9000", "40000"],
    "ICQ_PRO_MAX": ["2048", "4096", "16384"],
    "ICQ_PRO_MIN": ["0", "2048"],
    "ICQ_PRO_MAX_CM": ["0", "5000", "1000000"],
    "ICQ_LIST_J": ["-1", "0", "3"],
    "ICQ_LIST_DIV": ["128", "4"],
    "ICQ_CL": ["1", "0"],
    "ICQ_CL_CAP": ["1048576", "500"],
    "ICQ_MAX_PAGES": ["128", "1"],
    "ICQ_MAX_PAGES_CM": ["512", "1", "3"],
    "ICQ_POOL_PAGES": ["8192", "2", "40"],
    "ICQ_ROUNDS": ["4", "1", "2"],
    "ICQ_WALK_CAP": ["131072", "1", "3000"],
    "ICQ_RANGE_ITEMS": ["32768", "65536"],
    "ICQ_RANGE_MAJOR": ["0", "1"],
    "ICQ_RANGE_GROUP": ["1", "2"],
    "ICQ_COUNT_RANGES": ["1", "2"],
    "ICQ_COUNT_DIV": ["256", "8", "0"],
    "ICQ_COUNT_MIN": ["262144", "100"],
    "ICQ_DEBUG": ["0", "64", "1", "16"],
    "ICQ_QBATCH": ["2048", "3"],
}


def surv_ids(row, n):
    bits = np.unpackbits(row.astype(np.uint32).view(np.uint8), bitorder="little")[:n]
    return np.flatnonzero(bits)


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rng = np.random.default_rng(seed)
    t0 = time.time()
    it = fails = 0
    while time.time() - t0 < budget:
        it += 1
        sizes = [120000, 400000, 1200000] if os.environ.get("FUZZ_BIG") else [300, 2500, 9000, 40000, 120000]
        n = int(rng.choice(sizes))
        K = int(rng.choice([2, 4, 8, 16]))
        m = int(rng.choice([4, 16, 256]))
        F = int(rng.integers(1, K + 1)) if rng.random() < 0.3 else int(rng.choice([1, 2, 4])[()] if K >= 4 else 1)
        F = min(F, K)
        d = int(rng.choice([4, 16, 40]))
        books = rng.standard_normal((K, m, d)).astype(np.float32)
        books[:F] *= float(rng.choice([1.0, 4.0]))
        codes = rng.integers(0, m, size=(n, K)).astype(np.uint8)
        if rng.random() < 0.2:
            codes[1::2] = codes[0::2]
        fast = np.sort(rng.choice(K, size=F, replace=False)).astype(np.uint32)
        env = {k: str(rng.choice(v)) for k, v in KNOBS.items() if rng.random() < 0.45}
        for key in KNOBS:
            os.environ.pop(key, None)
        os.environ.update(env)
        nq = int(rng.integers(1, 6))
        Q = rng.standard_normal((nq, d))
        k = int(rng.choice([1, 7, 100, 300]))
        k = min(k, n)
        sigma = rng.choice([0.0, 0.3, 2.0, 30.0, 1e18])
        sigma = np.float32(sigma) if rng.random() < 0.15 and sigma < 1e10 else float(sigma)
        try:
            dev = icqb.DeviceIndex(books, codes, fast)
            out = dev.search_device(torch.from_numpy(Q).cuda(), k, sigma, survivors=True, stats=True)
            torch.cuda.synchronize()
            for i in range(nq):
                ref = O.two_step(books, codes, fast, sigma, Q[i], k)
                ok = (np.array_equal(out["ids"][i].cpu().numpy(), ref.ids)
                      and np.array_equal(out["scores"][i].cpu().numpy(), ref.scores)
                      and int(out["refinements"][i]) == ref.ops.refinements
                      and np.array_equal(surv_ids(out["survivors"][i].cpu().numpy(), n), ref.survivors))
                if not ok:
                    fails += 1
                    print("MISMATCH", dict(n=n, K=K, m=m, F=F, d=d, k=k, sigma=repr(sigma), q=i, fast=fast.tolist(),
                                           seed=seed, it=it), env, flush=True)
                    break
        except Exception as e:  # noqa: BLE001
            fails += 1
            print("ERROR", repr(e)[:300], dict(n=n, K=K, m=m, F=F, d=d, k=k, sigma=repr(sigma), seed=seed, it=it),
                  env, flush=True)
    print(f"fuzz: {it} cases, {fails} failures, {time.time() - t0:.0f} s, seed {seed}")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
