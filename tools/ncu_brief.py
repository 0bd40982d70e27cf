"""One line per kernel of an ncu report, unit-normalised: time (us), DRAM MB,
DRAM GB/s, L2 hit %, SM / memory throughput %, achieved occupancy %, regs,
and the top stall reasons.  Usage: python tools/ncu_brief.py rep.ncu-rep ..."""
import csv
import io
import subprocess
import sys

SCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6,
         "nsecond": 1e-3, "second": 1e6, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
         "Gbyte": 1e3, "Tbyte": 1e6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}


def rows_of(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    return rows[0], rows[1], rows[2:]


def val(h, u, r, name, unit_scale=True):
    if name not in h:
        return None
    i = h.index(name)
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:
        return None
    return v * SCALE.get(u[i], 1.0) if unit_scale else v


for rep in sys.argv[1:]:
    h, u, data = rows_of(rep)
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0][:40]
        t = val(h, u, r, "gpu__time_duration.sum")
        rd = val(h, u, r, "dram__bytes_read.sum") or 0
        wr = val(h, u, r, "dram__bytes_write.sum") or 0
        l2 = val(h, u, r, "lts__t_sector_hit_rate.pct", False)
        sm = val(h, u, r, "sm__throughput.avg.pct_of_peak_sustained_elapsed", False)
        mem = val(h, u, r, "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", False)
        occ = val(h, u, r, "sm__warps_active.avg.pct_of_peak_sustained_active", False)
        regs = val(h, u, r, "launch__registers_per_thread", False)
        inst = val(h, u, r, "smsp__inst_executed.sum", False)
        stalls = []
        for i, n in enumerate(h):
            pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
            if n.startswith(pre) and n.endswith(suf):
                try:
                    stalls.append((float(r[i]), n[len(pre):-len(suf)]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("%-40s %9.1f us  DRAM %8.1f MB  %6.0f GB/s  L2hit %5.1f  sm %5.1f  mem %5.1f  occ %5.1f  regs %s  Minst %.1f"
              % (name, t or 0, rd + wr, (rd + wr) / (t or 1) * 1e3, l2 or 0, sm or 0,
                 mem or 0, occ or 0, int(regs or 0), (inst or 0) / 1e6))
        print("    stalls: " + ", ".join("%s=%.1f" % (n, v) for v, n in stalls[:6]))
