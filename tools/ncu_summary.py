"""Summarise an ncu report: per kernel time, DRAM bytes, throughputs, top stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
data = rows[2:]
col = {n: i for i, n in enumerate(h)}


def g(r, n):
    i = col.get(n)
    return r[i] if i is not None else ""


stall_cols = [n for n in h if n.startswith("smsp__average_warp_latency_issue_stalled_") and
              n.endswith(".ratio")] or \
             [n for n in h if n.startswith("smsp__average_warps_issue_stalled_") and
              n.endswith("_per_issue_active.ratio")]
for r in data:
    name = g(r, "Kernel Name").split("(")[0].split("::")[-1][:26]
    t = float(g(r, "gpu__time_duration.sum") or 0)
    rd = float(g(r, "dram__bytes_read.sum") or 0)
    wr = float(g(r, "dram__bytes_write.sum") or 0)
    print("%-26s t=%8.1fus dram=%7.1fMB  dramGB/s=%7.0f  sm%%=%5.1f mem%%=%5.1f warps%%=%5.1f regs=%s L2hit=%s" % (
        name, t * 1e3 if t < 100 else t / 1e3, rd + wr,
        (rd + wr) / (t if t < 100 else t / 1e3) if t else 0,
        float(g(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed") or 0),
        float(g(r, "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed") or 0),
        float(g(r, "sm__warps_active.avg.pct_of_peak_sustained_active") or 0),
        g(r, "launch__registers_per_thread"), g(r, "lts__t_sector_hit_rate.pct")))
    st = []
    for n in stall_cols:
        try:
            st.append((float(r[col[n]]), n.split("stalled_")[1].split(".")[0].replace("_per_issue_active", "")))
        except ValueError:
            pass
    st.sort(reverse=True)
    print("     stalls:", ", ".join("%s=%.1f" % (b, a) for a, b in st[:6]))
print("units:", rows[1][col["gpu__time_duration.sum"]], rows[1][col["dram__bytes_read.sum"]])
