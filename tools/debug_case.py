"""Debug helper: compare GPU survivors with the oracle on a golden case."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from _golden import load
from oracle import icq_oracle as O
import paper_1912_08756_b200 as icqb

name = sys.argv[1] if len(sys.argv) > 1 else 'trained_k16f4'
c = load(name)
dev = icqb.DeviceIndex(c.books, c.codes.astype(np.uint8), c.fast)
for qi in range(len(c.queries)):
    for k in (10, 100):
        for sigma in (0.0, 2.0):
            q = torch.from_numpy(c.queries[qi:qi+1]).cuda()
            out = dev.search_device(q, k, sigma, survivors=True, stats=True)
            torch.cuda.synchronize()
            bm = out['survivors'][0].cpu().numpy().astype(np.uint32)
            bits = np.unpackbits(bm.view(np.uint8), bitorder='little')[:c.n]
            got = np.flatnonzero(bits)
            ref = O.two_step(c.books, c.codes, c.fast, sigma, c.queries[qi], k)
            st = out['stats'][0].cpu().numpy()
            miss = np.setdiff1d(ref.survivors, got); extra = np.setdiff1d(got, ref.survivors)
            print(qi, k, sigma, 'ref', ref.survivors.size, 'gpu', got.size, 'miss', miss[:10], 'extra', extra[:10], 'stats', st.tolist())
