"""Warp-stall samples and executed instructions grouped by SASS opcode (ncu
source page) for one kernel of a report.

usage: python tools/ncu_opstall.py report.ncu-rep [kernel_index (0)] [top (14)]
"""
import csv
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]
want = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 14
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
# sections: a "Kernel Name" row, a header row, then the instruction rows
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "hdr": None, "data": []}
        sections.append(cur)
    elif cur is not None and cur["hdr"] is None:
        cur["hdr"] = r
    elif cur is not None and len(r) >= len(cur["hdr"]):
        cur["data"].append(r)
sec = sections[want]
h = sec["hdr"]
ci = h.index("Warp Stall Sampling (All Samples)")
si = h.index("Source")
ie = h.index("Instructions Executed")
stall_cols = [(k, h.index(k)) for k in h if k.startswith("stall_") and "Not Issued" not in k]
by = defaultdict(Counter)
samp = Counter()
inst = Counter()
for r in sec["data"]:
    toks = r[si].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    samp[op] += float(r[ci] or 0)
    inst[op] += float(r[ie] or 0)
    for k, j in stall_cols:
        by[op][k[6:]] += float(r[j] or 0)
tot = sum(samp.values()) or 1.0
itot = sum(inst.values()) or 1.0
print(f"# {sec['name']}: {itot:.4g} warp instructions")
for op, v in samp.most_common(top):
    print(f"{op:10s} samples {100 * v / tot:5.1f}%  inst {inst[op]:.3g} ({100 * inst[op] / itot:4.1f}%)  "
          f"top: {[(k, round(100 * x / tot, 1)) for k, x in by[op].most_common(3)]}")
