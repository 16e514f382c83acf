"""Opcode mix + stall samples of a kernel from `ncu --page source --csv --print-source sass`.
usage: python profiles/sass_mix.py source.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
ops, stall = collections.Counter(), collections.Counter()
tot = stot = 0
for r in rows[2:]:
    if len(r) <= iE: continue
    s = r[iS].strip()
    op = s.split()[0] if s else "?"
    if op.startswith("@"): op = s.split()[1]
    n = int(r[iE] or 0); w = int(r[iW] or 0)
    ops[op] += n; tot += n; stall[op] += w; stot += w
print(f"total warp instructions {tot:,}  stall samples {stot:,}")
for op, n in ops.most_common(top):
    print(f"{op:28s} {n:14,} {100*n/tot:6.2f}%   stall {100*stall[op]/max(stot,1):6.2f}%")
