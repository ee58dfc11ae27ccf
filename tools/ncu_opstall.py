"""Warp-stall samples grouped by SASS opcode (ncu source page)."""
import csv, subprocess, sys
from collections import Counter, defaultdict
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[1]; data = rows[2:]
ci = h.index('Warp Stall Sampling (All Samples)'); si = h.index('Source')
ie = h.index('Instructions Executed')
stall_cols = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
by = defaultdict(Counter); samp = Counter(); inst = Counter()
for r in data:
    toks = r[si].split()
    if not toks: continue
    op = (toks[1] if toks[0].startswith('@') else toks[0]).split('.')[0]
    samp[op] += float(r[ci] or 0); inst[op] += float(r[ie] or 0)
    for k in stall_cols:
        by[op][k[6:]] += float(r[h.index(k)] or 0)
tot = sum(samp.values())
for op, v in samp.most_common(12):
    print(f"{op:10s} samples {100*v/tot:5.1f}%  inst {inst[op]:.3g}  top: {[(k, round(100*x/tot,1)) for k, x in by[op].most_common(4)]}")
