"""Write profiles/r02_summary.md (+ copies of the raw artefacts and the
traffic entries bench.py reads) from the gpurun_out/ files of
tools/make_profiles_r02.sh.

    python tools/write_summary_r02.py
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
r = "r02"
N_C3 = 134217789  # suffixes of a full c3 block (2^27 + the last string)

# tools/make_profiles_r02.sh's ncu --set full captures (tools/prof_c3.sh order)
CAPTURES = [("sort_local_digit", "local_digit_kernel<256> of block 0 (its third digit level, "
             "~2048-member segments; DRAM bytes as captured)", None),
            ("gather", "block 8", (5.375 + 32.0 + 4.0) * N_C3),  # g read as one 32 B sector
            ("compute_ranks", "block 8", None),
            ("digit_scatter", "second 8-bit pass of block 0", 16.0 * N_C3),
            ("insert", "block 10", None),
            ("digit_hist", "second pass of block 0", 8.0 * N_C3),
            ("pack", "block 5", 1.375 * N_C3)]


KEEP_REPORTS = (0, 1, 2)  # local_digit, gather, compute_ranks


def sh(cmd):
    return subprocess.run(cmd, capture_output=True, text=True, shell=isinstance(cmd, str)).stdout


def brief(rep):
    return sh([sys.executable, os.path.join(ROOT, "tools", "ncu_brief.py"), rep])


def dram_bytes(rep):
    out = sh(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
              "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"])
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None, None
    h, u, v = rows[0], rows[1], rows[2]
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
          "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}

    def g(n):
        i = h.index(n)
        return float(v[i].replace(",", "")) * sc.get(u[i], 1.0)
    return g("dram__bytes_read.sum") + g("dram__bytes_write.sum"), g("gpu__time_duration.sum")


def line(path):
    try:
        return open(path).read().strip().splitlines()[-1]
    except Exception:
        return None


def main():
    os.makedirs(PROF, exist_ok=True)
    md = ["# Round 02 profile summary (B200, sm_100a) -- c3 workload (the metric's config)", "",
          "Produced by `tools/make_profiles_r02.sh` on one B200 (gpurun) and "
          "`tools/write_summary_r02.py`.", ""]
    gpu = os.path.join(OUT, r + "_gpu.txt")
    if os.path.exists(gpu):
        md += ["GPU / clocks at start: `%s`." % " | ".join(open(gpu).read().split("\n")[:2]), ""]
    for name, f in (("Bench line (our arm, c3 default)", r + "_bench.json"),
                    ("Bench line (our arm, c2)", r + "_bench_c2.json"),
                    ("Reference arm (the CPU oracle on the box's host cores)", r + "_ref.json")):
        ln = line(os.path.join(OUT, f))
        if ln:
            shutil.copy(os.path.join(OUT, f), os.path.join(PROF, f))
            md += ["## " + name, "", "```", ln, "```", ""]
    lc = os.path.join(OUT, r + "_launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(PROF, r + "_launches.csv"))
        tab = sh([sys.executable, os.path.join(ROOT, "tools", "summarize_launches.py"), lc])
        md += ["## Per-kernel share of one c3 step (ncu launch list of `bench.py --steps 2 --warmup 3 "
               "--no-cpu-baseline`; cold-cache, serialised)", "",
               "Raw list: `profiles/%s_launches.csv`." % r, "", tab, ""]
    md += ["## ncu --set full, one launch each (c3, `tools/prof_c3.sh`)", "", "```"]
    traffic = {}
    tpath = os.path.join(PROF, "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for i, (kname, what, alg) in enumerate(CAPTURES):
        rep = os.path.join(OUT, "%s_full_%d.ncu-rep" % (r, i))
        if not os.path.exists(rep):
            continue
        md.append(brief(rep).rstrip())
        if i in KEEP_REPORTS:  # the largest reports stay in gpurun_out/ only
            shutil.copy(rep, os.path.join(PROF, "%s_full_%d.ncu-rep" % (r, i)))
        dram, t = dram_bytes(rep)
        if dram:
            ent = {"dram_bytes_per_launch": dram, "launch": "c3 %s, ncu --set full %s_full_%d" % (
                what, r, i), "time_s": t}
            if alg:
                ent["algorithmic_bytes_per_launch"] = alg
            traffic[kname] = ent
    md += ["```", ""]
    json.dump(traffic, open(tpath, "w"), indent=1)
    extra = os.path.join(PROF, r + "_reading.md")
    if os.path.exists(extra):
        md += [open(extra).read()]
    open(os.path.join(PROF, r + "_summary.md"), "w").write("\n".join(md) + "\n")
    print("wrote", os.path.join(PROF, r + "_summary.md"))


if __name__ == "__main__":
    main()
