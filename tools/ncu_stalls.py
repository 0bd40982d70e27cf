"""Warp-state stall breakdown (cycles per issued instruction) from an ncu report."""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0][-30:]
    vals = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                vals.append((float(r[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    vals.sort(reverse=True)
    print(name, " ".join("%s=%.2f" % (b, a) for a, b in vals[:8]))
