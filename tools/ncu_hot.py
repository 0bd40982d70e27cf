"""Top SASS instructions by stall samples from an ncu source-page CSV."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":   # next kernel instance: stop at the first
        break
    if len(r) > 2 and r[0].startswith("0x"):
        data.append(r)
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
tot = sum(int(r[si] or 0) for r in data)
print("total samples", tot, "instructions", sum(int(r[ie] or 0) for r in data))
top = sorted(data, key=lambda r: -int(r[si] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]
idx = {r[0]: i for i, r in enumerate(data)}
for r in top:
    print("%6.2f%%  %-8s %s" % (100.0 * int(r[si]) / tot, r[ie], r[1].strip()[:90]))
# group by opcode
from collections import Counter
c = Counter()
ci = Counter()
for r in data:
    op = r[1].strip().split()[0] if r[1].strip() else "?"
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    c[op.split(".")[0]] += int(r[si] or 0)
    ci[op.split(".")[0]] += int(r[ie] or 0)
print("by opcode (stall samples):", ", ".join("%s=%.1f%%" % (k, 100.0 * v / tot) for k, v in c.most_common(14)))
print("by opcode (instr executed):", ", ".join("%s=%d" % (k, v) for k, v in ci.most_common(14)))
