"""Per-kernel share of one bench step from an ncu launch list (gpu__time_duration).

Steps are delimited by bench.py's untimed L2 flush (a torch fill kernel).
Prints a markdown table for the step with the most of our launches."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
steps, cur = [], []
for r in rows[hi + 1:]:
    name = r[ki]
    if name.startswith("void at::") or "elementwise" in name or "fill" in name.lower():
        if cur:
            steps.append(cur)
        cur = []
        continue
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    us = v / 1000.0 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1000.0
    short = name.split("(")[0].replace("setbwte::sortk::", "").replace("setbwte::", "")
    short = short.replace("void ", "")
    cur.append((short, us))
if cur:
    steps.append(cur)
cands = [st for st in steps if not any(n.startswith("decode") for n, _ in st)] or steps
step = max(cands, key=len)
agg = collections.OrderedDict()
for n, us in step:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
print("| kernel | launches | total us | share |")
print("|---|---|---|---|")
for n, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print("| %s | %d | %.1f | %.3f |" % (n, c, us, us / tot))
print("| **step total (serialised, cold)** | %d | %.1f | 1.000 |" % (len(step), tot))
