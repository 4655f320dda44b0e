"""Aggregate an ncu source page (cuda,sass CSV) into per-source-line stall samples."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur_file = None
cur_line = None
cur_src = None
agg = defaultdict(lambda: [0, 0, ""])
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:  # source line row
        cur_line = r[0]
        cur_src = r[1]
        continue
    # sass row: columns shifted by 2
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ex = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    key = (cur_file, cur_line)
    agg[key][0] += s
    agg[key][1] = max(agg[key][1], ex)
    agg[key][2] = cur_src
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for (f, l), (s, ex, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot:5.1f}% {s:7d} ex={ex:9d} {f}:{l} {src.strip()[:80]}")
