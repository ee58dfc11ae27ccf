"""ptxas -v resource lines and a SASS opcode census of the tile-pass kernels
(the evidence for tcgen05 / TMA / TMEM use and for register spills).
usage: python tools/census.py  -> profiles/r02_ptxas.txt, profiles/r02_sass_census.txt"""
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2604_03816_b200", "csrc")
OBJ = os.path.join(ROOT, "paper_2604_03816_b200", "lib", "obj")
TUS = ["svb_inst_tile.cu", "svb_inst_reg64.cu", "svb_inst_reg64_tc.cu", "svb_inst_reg128.cu", "svb_inst_gemm.cu"]
KEEP = ("UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP", "SYNCS", "HMMA", "DFMA", "FFMA", "F2FP",
        "HADD2", "STS", "LDS", "STG", "LDG", "BAR", "SHFL", "LDL", "STL")


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    ptx_lines = ["# ptxas -v of the tile-pass kernels (round 2 build, sm_100a)", ""]
    for tu in TUS:
        r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                            "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I", CSRC,
                            "-I", os.path.join(ROOT, "include"), "-Xptxas", "-v", "-c",
                            os.path.join(CSRC, tu), "-o", os.devnull], capture_output=True, text=True)
        cur = None
        for line in r.stderr.splitlines():
            m = re.search(r"Compiling entry function '([^']+)'", line)
            if m:
                cur = m.group(1)
                continue
            if cur and ("registers" in line or "spill" in line):
                ptx_lines.append((cur, line.strip()))
    names = sorted({x[0] for x in ptx_lines if isinstance(x, tuple)})
    dm = demangle(names)
    out = [x if isinstance(x, str) else f"{dm[x[0]][:90]:90s} {x[1]}" for x in ptx_lines]
    open(os.path.join(ROOT, "profiles", "r02_ptxas.txt"), "w").write("\n".join(out) + "\n")

    cen = ["# SASS opcode census (static instruction counts) of the tile-pass kernels, round 2 build",
           "# (tcgen05 MMA = UTCHMMA, TMEM load/store = LDTM/STTM, TMA = UTMALDG / UBLKCP, mbarrier = SYNCS,",
           "#  local memory = LDL/STL)", ""]
    for tu in TUS:
        obj = os.path.join(OBJ, tu.replace(".cu", ".o"))
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        fn, cnt = None, Counter()
        rows = []
        for line in sass.splitlines():
            m = re.search(r"Function : (\S+)", line)
            if m:
                if fn:
                    rows.append((fn, cnt))
                fn, cnt = m.group(1), Counter()
                continue
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
            if m and fn:
                cnt[m.group(2)] += 1
        if fn:
            rows.append((fn, cnt))
        dm = demangle([r[0] for r in rows])
        for f, c in rows:
            total = sum(c.values())
            cen.append(f"{dm[f][:80]:80s} total={total} " + " ".join(f"{k}={c[k]}" for k in KEEP if c[k]))
    open(os.path.join(ROOT, "profiles", "r02_sass_census.txt"), "w").write("\n".join(cen) + "\n")


if __name__ == "__main__":
    sys.exit(main())
