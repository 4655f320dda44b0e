"""Small driver for ncu: one config's data, then LUT + scan launches on a
query subset (first launch = warm-up).  Not a benchmark (see bench.py)."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tools.workloads import CONFIGS, build_database, index_rule, load_books, queries  # noqa: E402
import paper_1912_08756_b200 as icqb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--nq", type=int, default=296)
ap.add_argument("--launches", type=int, default=2)
ap.add_argument("--sigma", type=float, default=None)
args = ap.parse_args()
w = CONFIGS[args.config]
books, meta = load_books(w)
fast, sigma, _, _ = index_rule(w, meta, args.sigma)
codes = build_database(w, books)
Q = queries(w)[: args.nq]
dev = icqb.DeviceIndex.from_device(books, codes, fast)
for _ in range(args.launches):
    lut = dev.build_lut_device(Q)
    out = dev.search_lut_device(lut, w.k, sigma, stats=True)
torch.cuda.synchronize()
st = out["stats"].double().mean(0).tolist()
print("stats", dict(zip(icqb.search.STATS_NAMES, st)))
