"""Print a one-line summary of bench.py's JSON line (stdin): config, value,
filter roofline fraction, per-step median/max and per-kernel milliseconds."""
import json
import sys

lines = [ln for ln in sys.stdin.read().strip().splitlines() if ln.startswith("{")]
if not lines:
    print("no bench line")
    sys.exit(1)
d = json.loads(lines[-1])
tag = sys.argv[1] if len(sys.argv) > 1 else ""
print(tag, d["config"]["workload"].split(":")[0], round(d["value"]),
      round((d.get("roofline") or {}).get("frac") or 0, 3), d.get("step_ms_median_max"),
      {k: round(v, 3) for k, v in (d.get("kernels_ms_per_step") or {}).items()},
      "e2e", round((d.get("e2e") or {}).get("value") or 0))
