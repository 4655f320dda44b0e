"""Per-region / per-line stall samples from an ncu cuda,sass source CSV."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
regions = [tuple(x.split(":")) for x in sys.argv[2:]]  # name:lo:hi (lines of icq_scan.cu)
rows = list(csv.reader(open(path)))
hdr = None
agg = defaultdict(int)
ex = defaultdict(int)
src = {}
f = None
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        try:
            cur = (f, int(r[0]))
            src[cur] = r[1]
        except ValueError:
            pass
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        agg[cur] += int(d["Warp Stall Sampling (All Samples)"] or 0)
        ex[cur] = max(ex[cur], int(d["Instructions Executed"] or 0))
    except (ValueError, KeyError):
        pass
tot = sum(agg.values())
print("total", tot)
for name, lo, hi in regions:
    rng = [k for k in agg if k[0] == "icq_scan.cu" and int(lo) <= k[1] <= int(hi)]
    s = sum(agg[k] for k in rng)
    print(f"== {name} {100 * s / max(tot, 1):.1f}%")
    for k in sorted(rng, key=lambda k: -agg[k])[:14]:
        print(f"{agg[k]:6d} ex={ex[k]:9d} {k[1]} {src[k].strip()[:88]}")
