"""Debug helper: GPU survivors vs the oracle on a random case in a pipeline mode
(env knobs of icq_capi.cu), with the float64 fast score / bound context of
every mismatching item."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from oracle import icq_oracle as O  # noqa: E402
import paper_1912_08756_b200 as icqb  # noqa: E402

n, d, K, m, F = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (5000, 16, 8, 256, 2)))
os.environ.setdefault("ICQ_PRO_MAX", "2048")
os.environ.setdefault("ICQ_PRO_MIN", "0")
rng = np.random.default_rng(n + d + K + m + F)
books = rng.standard_normal((K, m, d)).astype(np.float32)
books[:F] *= 4.0
codes = rng.integers(0, m, size=(n, K)).astype(np.uint8)
fast = np.arange(F, dtype=np.uint32)
dev = icqb.DeviceIndex(books, codes, fast)
Q = rng.standard_normal((6, d))
qd = torch.from_numpy(Q).cuda()
for k in (1, 10, 100):
    for sigma in (0.0, 1.0, 25.0):
        out = dev.search_device(qd, k, sigma, survivors=True, stats=True)
        torch.cuda.synchronize()
        for i in range(6):
            bm = out['survivors'][i].cpu().numpy().astype(np.uint32)
            got = np.flatnonzero(np.unpackbits(bm.view(np.uint8), bitorder='little')[:n])
            ref = O.two_step(books, codes, fast, sigma, Q[i], k)
            miss = np.setdiff1d(ref.survivors, got)
            extra = np.setdiff1d(got, ref.survivors)
            if miss.size or extra.size:
                st = out['stats'][i].cpu().numpy().tolist()
                lut = ((books.astype(np.float64) - Q[i]) ** 2).sum(-1)
                f64 = lut[np.arange(F)[None, :], codes[:, :F]].sum(1)
                print(f"k={k} sigma={sigma} q={i} miss={miss[:8].tolist()} extra={extra[:8].tolist()} "
                      f"P={st[3]} stats={st[:11]}")
                for j in list(miss[:4]) + list(extra[:4]):
                    print(f"   item {j}: fast64={f64[j]!r} f32sum={np.float32(lut[np.arange(F), codes[j, :F]].astype(np.float32)).sum()!r}")

# expected filter candidates for the first query at k=10, sigma=0
from tools.sim_filter import replay  # noqa: E402
out = dev.search_device(qd, 10, 0.0, survivors=True, stats=True)
torch.cuda.synchronize()
for i in range(6):
    st = out['stats'][i].cpu().numpy()
    P = int(st[3])
    hi = np.array([st[11]], dtype=np.int64).astype(np.int32).view(np.float32)[0]
    lut = ((books.astype(np.float64) - Q[i]) ** 2).sum(-1)
    f64 = lut[np.arange(F)[None, :], codes[:, :F]].sum(1)
    e64 = lut[np.arange(K)[None, :], codes].sum(1)
    res = replay(f64[:P], e64[:P], 10, 0.0, 0.0)
    M = f64[res[5]].max()
    f32 = lut.astype(np.float32)[np.arange(F)[None, :], codes[:, :F]].sum(1)
    print(f"q={i} P={P} hi={hi!r} M={M!r} expected_cands={(f64[P:] < M).sum()} "
          f"f32<hi={(f32[P:] < hi).sum()} gpu_listed={st[9]}")
