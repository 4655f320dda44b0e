import sys, numpy as np, torch
sys.path.insert(0, '.')
from tools.workloads import CONFIGS, build_database, index_rule, load_books, queries
import paper_1912_08756_b200 as icqb
for cfg in sys.argv[1:]:
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
    print(cfg, 'P', st[:, 3][:8], 'rescans', (fb & 0xfffff)[:8], 'ovf_pages', ((fb >> 20) & 0xfffff)[:8], 'ovf_pool', (fb >> 40)[:8], 'listed', st[:, 9][:8])
    print(cfg, 'totals: rescans', (fb & 0xfffff).sum(), 'ovf_pages', ((fb >> 20) & 0xfffff).sum(), 'ovf_pool', (fb >> 40).sum())
    # float64 reference of the filter threshold for the first queries
    from tools.sim_filter import replay
    B = torch.as_tensor(books, device='cuda', dtype=torch.float64)
    ci = codes.long()
    for qi in range(4):
        lut64 = ((B - Q[qi][None, None, :]) ** 2).sum(-1)
        f = sum(lut64[b][ci[:, b]] for b in fast.tolist()).cpu().numpy()
        e = sum(lut64[b][ci[:, b]] for b in range(w.K)).cpu().numpy()
        P = int(st[qi, 3])
        res = replay(f[:P], e[:P], w.k, sigma, 0.0)
        M = f[res[5]].max()
        hi = np.array([st[qi, 11]], dtype=np.int64).astype(np.int32).view(np.float32)[0]
        print(cfg, qi, 'wide', st[qi, 7], 'hi', hi, 'M', M, 'refined<P', int(res[0].sum()), 'cands', int((f[P:] < M).sum()),
              'lut min/max', float(lut64.min()), float(lut64.max()))
        l32 = lut64.float()
        fb = fast.tolist()
        a = l32[fb[0]][ci[:, fb[0]]] + l32[fb[1]][ci[:, fb[1]]]
        b = l32[fb[2]][ci[:, fb[2]]] + l32[fb[3]][ci[:, fb[3]]] if len(fb) == 4 else 0
        f32 = (a + b).cpu().numpy()
        print('   f32<hi after P:', int((f32[P:] < hi).sum()), ' f64<hi:', int((f[P:] < hi).sum()),
              ' f64 quantiles', np.quantile(f[P:], [0, 0.001, 0.01, 0.5]).tolist(), 'first items f64', f[:4].tolist())
