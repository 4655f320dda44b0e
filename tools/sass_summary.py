"""Opcode summary of the built library's kernels (cuobjdump -sass), written to
profiles/<tag>_sass_opcodes.txt: per kernel the instruction count, the
memory / gather opcodes and the top opcodes.

    python tools/sass_summary.py r02 [kernel-substring ...]
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_1912_08756_b200" / "lib" / "libicq_b200.so"
WATCH = ("LDG", "LDS", "STS", "STG", "LDGSTS", "UBLKCP", "UTMALDG", "PRMT", "FADD2", "FADD", "DADD",
         "DMUL", "IMAD", "SHF", "LEA", "VIMNMX3", "VIMNMX", "VOTE", "SHFL", "BAR", "ATOMG", "RED", "LDL", "STL")


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    want = sys.argv[2:] or ["icq_filter_kernelILi2E", "icq_filter_kernelILi4E", "icq_count_kernelILi2E",
                            "icq_dense_kernelILi2E", "icq_refine_kernelILi2E", "icq_cl_gather_kernelILi2E",
                            "icq_replay_kernelILi2E", "icq_prologue_kernelILi2E", "lut_build_kernel",
                            "encode_step_kernel"]
    txt = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    out = [f"SASS opcode summary of {LIB.name} (cuobjdump -sass, sm_100a)", ""]
    cur, ops = None, collections.Counter()

    def flush():
        if cur is None or not any(w in cur for w in want):
            return
        total = sum(ops.values())
        fam = collections.Counter()
        for k, v in ops.items():
            fam[k.split(".")[0]] += v
        out.append(f"{cur}: {total} instructions")
        out.append("  memory/gather: " + ", ".join(f"{w} {fam[w]}" for w in WATCH if fam.get(w)))
        wide = {k: v for k, v in ops.items() if k.startswith(("LDG.E.128", "LDG.E.64", "LDS.128", "LDS.64"))}
        if wide:
            out.append("  wide loads: " + ", ".join(f"{k} {v}" for k, v in sorted(wide.items())))
        out.append("  top: " + ", ".join(f"{k} {v}" for k, v in fam.most_common(12)))
        out.append("")

    for ln in txt.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            flush()
            cur, ops = m.group(1), collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", ln)
        if m and cur:
            ops[m.group(1)] += 1
    flush()
    (ROOT / "profiles").mkdir(exist_ok=True)
    p = ROOT / "profiles" / f"{tag}_sass_opcodes.txt"
    p.write_text("\n".join(out) + "\n")
    print("wrote", p, len(out), "lines")


if __name__ == "__main__":
    main()
