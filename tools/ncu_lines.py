"""Stall samples and instructions per CUDA source line from
`ncu -i X --page source --csv --print-source cuda,sass` output."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
line = None
samp = defaultdict(int)
inst = defaultdict(int)
src = {}
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) < 4:
        continue
    if r[0]:
        line = int(r[0])
        src[line] = r[1]
    if r[2].startswith("0x") or (len(r) > 2 and r[2]):
        try:
            samp[line] += int(r[si] or 0)
            inst[line] += int(r[ie] or 0)
        except (ValueError, IndexError):
            pass
tot = sum(samp.values()) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for l in sorted(samp, key=lambda l: -samp[l])[:n]:
    print("%6.2f%% %9d  %5d  %s" % (100.0 * samp[l] / tot, inst[l], l, src.get(l, "").strip()[:90]))
