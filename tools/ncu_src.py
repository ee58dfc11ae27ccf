"""Summarise an ncu source page: top stall lines + instruction mix."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[1]; data = rows[2:]
ci = h.index('Warp Stall Sampling (All Samples)'); si = h.index('Source'); ai = h.index('Address')
ie = h.index('Instructions Executed')
stall_cols = [k for k in h if k.startswith('stall_')]
tot = sum(float(r[ci] or 0) for r in data)
totinst = sum(float(r[ie] or 0) for r in data)
print("samples", tot, "instructions", totinst)
for r in sorted(data, key=lambda r: -float(r[ci] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    st = sorted(((float(r[h.index(k)] or 0), k) for k in stall_cols), reverse=True)[:2]
    print(r[ai][-5:], r[si][:58].ljust(58), r[ci], [(k[6:], int(v)) for v, k in st if v])
agg = Counter()
for r in data:
    for k in stall_cols:
        agg[k] += float(r[h.index(k)] or 0)
print("stall totals:", [(k[6:], round(100 * v / tot, 1)) for k, v in agg.most_common(8)])
c = Counter()
for r in data:
    toks = r[si].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    c[op.split('.')[0]] += float(r[ie] or 0)
print("mix:", [(k, round(100 * v / totinst, 1)) for k, v in c.most_common(14)])
