"""Debug helper: per-query filter diagnostics on a bench workload (rounds,
prologue end, filter threshold, overflowed slices) next to a float64
recount of the items under the threshold."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from tools.workloads import CONFIGS, build_database, index_rule, load_books, queries  # noqa: E402
import paper_1912_08756_b200 as icqb  # noqa: E402

cfg = sys.argv[1]
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = CONFIGS[cfg]
books, meta = load_books(w)
fast, sigma, _, _ = index_rule(w, meta, None)
codes = build_database(w, books, sweeps=10)
dev = icqb.DeviceIndex.from_device(books, codes, fast)
Q = queries(w)[:w.batch]
lut = dev.build_lut_device(Q)
out = dev.search_lut_device(lut, w.k, sigma, stats=True)
torch.cuda.synchronize()
st = out['stats'].cpu().numpy()
fb = st[:, 6]
print(cfg, 'rounds', np.bincount(st[:, 2].astype(int)), 'P mean', st[:, 3].mean(),
      'rescans', (fb & 0xfffff).sum(), 'ovf_pages', ((fb >> 20) & 0xfffff).sum(), 'ovf_pool', (fb >> 40).sum())
B = torch.as_tensor(books, device='cuda', dtype=torch.float64)
ci = codes.long()
for qi in range(nq):
    lut64 = ((B - Q[qi][None, None, :]) ** 2).sum(-1)
    f = sum(lut64[b][ci[:, b]] for b in fast.tolist())
    P = int(st[qi, 3])
    hi = np.array([st[qi, 11]], dtype=np.int64).astype(np.int32).view(np.float32)[0]
    under = int((f[P:] < float(hi)).sum().item())
    print(qi, 'P', P, 'rounds', int(st[qi, 2]), 'hi', float(hi), 'items<hi after P', under,
          'ovf', int((fb[qi] >> 20) & 0xfffff), int(fb[qi] >> 40), 'ins', int(st[qi, 0]), 'pro_ins', int(st[qi, 10]))
