"""Debug helper (GPU box): one failing parity case of the rounds mode."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))


def main():
    import torch

    import paper_1912_08756_b200 as icqb
    from oracle import icq_oracle as O
    from paper_1912_08756_b200.search import STATS_NAMES
    from test_gpu_parity import _random_case

    n, d, K, m, F, dup = 5000, 16, 8, 256, 2, False
    rng = np.random.default_rng(n + d + K + m + F)
    books, codes, fast = _random_case(rng, n, d, K, m, F, dup)
    dev = icqb.DeviceIndex(books, codes, fast)
    Q = rng.standard_normal((6, d))
    qd = torch.from_numpy(Q).cuda()
    k, sigma = 10, 0.0
    for cap in ("1", "100000000"):
        os.environ.update(ICQ_PRO_MAX="2048", ICQ_PRO_MIN="0", ICQ_WALK_CAP=cap, ICQ_ROUNDS="4")
        out = dev.search_device(qd, k, sigma, survivors=True, stats=True)
        st = out["stats"].cpu().numpy()
        for i in range(6):
            ref = O.two_step(books, codes, fast, sigma, Q[i], k)
            ok = np.array_equal(out["ids"][i].cpu().numpy(), ref.ids)
            print(cap, i, ok, int(out["refinements"][i]), ref.ops.refinements,
                  {nm: int(st[i, j]) for j, nm in enumerate(STATS_NAMES) if j in (0, 1, 2, 3, 6, 7, 9)})
            if not ok:
                bits = np.unpackbits(out["survivors"][i].cpu().numpy().view(np.uint8),
                                     bitorder="little")[:n]
                got = np.flatnonzero(bits)
                miss = np.setdiff1d(ref.survivors, got)
                extra = np.setdiff1d(got, ref.survivors)
                print("   missing", miss[:20], "extra", extra[:20])


if __name__ == "__main__":
    main()
