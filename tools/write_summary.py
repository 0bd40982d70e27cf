"""Write profiles/<round>_summary.md (+ copies of the raw artefacts and
profiles/traffic.json) from the gpurun_out/ files of tools/make_profiles.sh.

    python tools/write_summary.py r01
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
r = sys.argv[1] if len(sys.argv) > 1 else "r01"

# the ncu --set full captures of tools/make_profiles.sh, in order
CAPTURES = [("digit_scatter", "first 8-bit pass of block 0 (16,777,312 active elements)",
             16.0 * 16777312),
            ("bitonic_kernel<8>", "block 0", None),
            ("compute_ranks", "block 5", None),
            ("gather", "block 5", None),
            ("insert", "block 5", None),
            ("digit_hist", "first pass of block 0 (generates key word 0)", None),
            ("tiny", "first launch", None)]


def raw(rep, metrics):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (v[h.index(k)], u[h.index(k)]) for k in h if k in metrics or k == "Kernel Name"}


def num(x, unit):
    x = float(x)
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e3, "us": 1.0,
             "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}
    return x * scale.get(unit, 1.0)


def launches_table(path):
    rows = [row for row in csv.reader(open(path)) if len(row) > 10 and row[0].isdigit()]
    agg = {}
    for row in rows:
        name = row[4].split("(")[0].replace("void ", "").replace("setbwte::", "")
        unit = row[-2]
        t = num(row[-1], unit if unit else "ns")
        if unit == "nsecond" or unit == "ns":
            t = float(row[-1]) / 1000.0
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    total = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append("| %s | %d | %.1f | %.3f |" % (k, n, t, t / total))
    lines.append("| **all launches (serialised, cold)** | %d | %.1f | 1.000 |" %
                 (sum(v[0] for v in agg.values()), total))
    return "\n".join(lines), agg, total


def main():
    bench = json.load(open(os.path.join(OUT, r + "_bench.json")))
    ref = json.load(open(os.path.join(OUT, r + "_ref.json")))
    gpu = open(os.path.join(OUT, r + "_gpu.txt")).read().strip() if os.path.exists(
        os.path.join(OUT, r + "_gpu.txt")) else ""
    for f in (r + "_bench.json", r + "_ref.json", r + "_launches.csv"):
        shutil.copy(os.path.join(OUT, f), os.path.join(PROF, f))
    table, agg, total = launches_table(os.path.join(OUT, r + "_launches.csv"))
    metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "sm__throughput.avg.pct_of_peak_sustained_elapsed",
               "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
               "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
               "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]
    traffic = {}
    full_lines = ["%-22s %8s %9s %8s %6s %6s %6s %5s %9s %6s" %
                  ("kernel", "us", "DRAM MB", "GB/s", "sm%", "mem%", "warp%", "regs", "Minst", "L2hit")]
    for i, (key, launch, alg) in enumerate(CAPTURES):
        rep = os.path.join(OUT, "%s_full_%d.ncu-rep" % (r, i))
        if not os.path.exists(rep):
            continue
        m = raw(rep, metrics)
        if not m:
            continue
        if i == 0:  # the dominant kernel's full report is kept (the others stay in gpurun_out/)
            shutil.copy(rep, os.path.join(PROF, os.path.basename(rep)))
        t = num(*m["gpu__time_duration.sum"])
        d = num(*m["dram__bytes_read.sum"]) + num(*m["dram__bytes_write.sum"])
        full_lines.append("%-22s %8.1f %9.1f %8.0f %6.1f %6.1f %6.1f %5s %9.2f %6.1f" % (
            key, t, d / 1e6, d / t / 1e3, float(m["sm__throughput.avg.pct_of_peak_sustained_elapsed"][0]),
            float(m["gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
            float(m["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
            m["launch__registers_per_thread"][0], float(m["smsp__inst_executed.sum"][0]) / 1e6,
            float(m["lts__t_sector_hit_rate.pct"][0])))
        ent = {"dram_bytes_per_launch": d, "launch": launch + ", ncu --set full %s_full_%d" % (r, i)}
        if alg:
            ent["algorithmic_bytes_per_launch"] = alg
        traffic[key] = ent
    json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    roof = bench.get("roofline", {})
    dom = roof.get("kernel")
    share_ncu = None
    for k, (n, t) in agg.items():
        if dom and dom in k.replace("_kernel", "").replace("sortk::", ""):
            share_ncu = t / total
    md = ["# Round %s profile summary (B200, sm_100a) -- c2 workload" % r[1:], "",
          "Produced by `tools/make_profiles.sh %s` on one B200 (gpurun) and `tools/write_summary.py %s`." % (r, r),
          "GPU / clocks at start: `%s`." % gpu.replace("\n", " | "), "",
          "## Bench line (our arm)", "", "```", json.dumps(bench), "```", "",
          "## Reference arm (the CPU oracle on the box's host cores)", "", "```", json.dumps(ref), "```", "",
          "## Per-kernel share (ncu launch list of `bench.py --steps 2 --warmup 3 --no-cpu-baseline`: "
          "10 c2 builds incl. the e2e ones; cold-cache, serialised)", "",
          "Dominant kernel in the bench: `%s`, CUDA-event share of the pipelined step %.3f; "
          "its share of the serialised launch list below: %s." % (
              dom, roof.get("share_of_step") or 0.0, "%.3f" % share_ncu if share_ncu else "n/a"),
          "Raw list: `profiles/%s_launches.csv`." % r, "", table, "",
          "## ncu --set full, one launch each (`profiles/%s_full_0.ncu-rep` = digit_scatter)" % r, "", "```"] + \
        full_lines + ["```", ""]
    rd = os.path.join(PROF, r + "_reading.md")
    if os.path.exists(rd):
        md += ["", open(rd).read()]
    open(os.path.join(PROF, r + "_summary.md"), "w").write("\n".join(md))
    print("wrote", os.path.join(PROF, r + "_summary.md"))


if __name__ == "__main__":
    main()
