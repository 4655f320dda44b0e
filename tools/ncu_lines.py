"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
into per-source-line instruction counts and stall samples (with the top
stall reasons).  Usage: ncu_lines.py <csv> [top] [per-unit divisor]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
rows = list(csv.reader(open(path)))
hdr = None
cur = None
fname = "?"
agg = defaultdict(lambda: {"ex": 0, "s": 0, "r": defaultdict(int)})
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:70])
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ex = int(d.get("Instructions Executed", "0") or 0)
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    a = agg[cur]
    a["ex"] += ex
    a["s"] += s
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                a["r"][k[6:]] += int(v or 0)
            except ValueError:
                pass
tot_s = sum(a["s"] for a in agg.values()) or 1
tot_ex = sum(a["ex"] for a in agg.values())
print(f"instructions {tot_ex} ({tot_ex / div:.1f} per unit), stall samples {tot_s}")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1]["s"])[:top]:
    rs = sorted(a["r"].items(), key=lambda kv: -kv[1])[:2]
    rtxt = " ".join(f"{k}:{100 * v / max(1, a['s']):.0f}%" for k, v in rs)
    print(f"{100 * a['s'] / tot_s:5.1f}% {a['ex'] / div:8.1f}/u  {key[0]}:{key[1]:>4} [{rtxt}] {key[2]}")
