"""Summarise ncu captures from gpurun_out/ into profiles/ (run in the build
container after tools/profile_bench.sh ran on the GPU box).

    python tools/profile_summary.py <config> <tag>

Writes
  profiles/<tag>_<cfg>_launches.csv      per-launch device times (ncu launch list)
  profiles/<tag>_<cfg>_<kernel>.txt      key --set full metrics + hottest source lines
  profiles/traffic.json                  DRAM bytes per filter launch (bench.py roofline.traffic)
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "nsecond": 1e-9, "second": 1.0}

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]


def raw_metrics(rep: Path) -> dict:
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            out[h] = v
            continue
        if u in UNITS:
            out[h] = x * UNITS[u]
            out[h + "@unit"] = "s" if "second" in u or u in ("ns", "us", "ms", "s") else "bytes"
        else:
            out[h] = x
            out[h + "@unit"] = u
    return out


def main():
    cfg, tag = sys.argv[1], sys.argv[2]
    PROF.mkdir(exist_ok=True)
    launches = OUT / f"launches_{cfg}_{tag}.csv"
    if launches.exists():
        lines = [ln for ln in launches.read_text().splitlines() if not ln.startswith("==")]
        rows = list(csv.reader(lines))
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        with open(PROF / f"{tag}_{cfg}_launches.csv", "w") as f:
            f.write("kernel,ns\n")
            tot = {}
            for r in rows[1:]:
                name = r[ki].split("(")[0].replace("void ", "")
                f.write(f"{name},{r[vi]}\n")
                tot[name] = tot.get(name, 0.0) + float(r[vi])
            f.write("# share of device time: " + ", ".join(
                f"{k} {100 * v / sum(tot.values()):.1f}%" for k, v in tot.items()) + "\n")
            # the search step's own kernels: the pipeline instantiation launched
            # most often (bench.py's setup also runs the exact engine once, <16>)
            cnt = {}
            for r in rows[1:]:
                name = r[ki].split("(")[0].replace("void ", "")
                if "icq_filter_kernel" in name:
                    cnt[name] = cnt.get(name, 0) + 1
            if cnt:
                targ = max(cnt, key=cnt.get).split("icq_filter_kernel")[1]
                step = {k: v for k, v in tot.items() if k.endswith(targ) or "lut_build" in k}
                f.write(f"# share of the search step ({targ} pipeline + LUT build): " + ", ".join(
                    f"{k} {100 * v / sum(step.values()):.1f}%" for k, v in step.items()) + "\n")
    traffic = {}
    tpath = PROF / "traffic.json"
    if tpath.exists():
        traffic = json.loads(tpath.read_text())
    for rep in sorted(OUT.glob(f"full_{cfg}_{tag}_*.ncu-rep")):
        kern = rep.stem.split(f"full_{cfg}_{tag}_")[1]
        m = raw_metrics(rep)
        src = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv",
                              "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
        tmp = OUT / f"{kern}_src.csv"
        tmp.write_text(src)
        hot = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_lines.py"), str(tmp), "25"],
                             capture_output=True, text=True).stdout
        with open(PROF / f"{tag}_{cfg}_{kern}.txt", "w") as f:
            f.write(f"ncu --set full --clock-control none capture of {kern} ({cfg}, {tag}); one launch\n")
            for k in KEYS:
                if k in m:
                    f.write(f"{k} = {m[k]} {m.get(k + '@unit', '')}\n")
            f.write("\nhottest source lines (stall samples, instructions per launch):\n")
            f.write(hot)
        if kern == "icq_filter":
            rd = m.get("dram__bytes_read.sum", 0.0)
            wr = m.get("dram__bytes_write.sum", 0.0)
            traffic[cfg] = {
                "source": f"profiles/{tag}_{cfg}_{kern}.txt (ncu --set full, one filter launch = one bench batch)",
                "dram_bytes_read_per_launch": rd,
                "dram_bytes_write_per_launch": wr,
                "dram_bytes_per_launch_at_bench_batch": rd + wr,
                "note": "the fast-code stream is L2-resident across the queries of a batch; DRAM "
                        "traffic is first touches, the L2 flush write-back and candidate pages",
            }
    tpath.write_text(json.dumps(traffic, indent=2) + "\n")
    print("wrote", sorted(p.name for p in PROF.glob(f"{tag}_{cfg}_*")))


if __name__ == "__main__":
    main()
