#!/usr/bin/env python
"""bench.py -- set-bwte BWT build throughput on B200 (BASELINE.json metric).

One STEP = one whole pass of the hot path over one batch: clear the index and
append the workload's reads (Algorithm 1 over all its blocks: pack, ConstructSA,
B_int, ComputeRanks, g->g_sa gather, Insert + dictionary rebuild), inputs
already resident in HBM.  Default workload = BASELINE configs[2] ("c3"), the
config BASELINE.json's metric ("at 1/2/4/8 B200") is quoted on: 20M uniform
reads x 100 bp, blocks of M = 2^27 suffixes (K = 16).  configs[1] (c2) and the
others are selected with --workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU, NCCL): every rank builds the same index;
ComputeRanks is split by string across ranks and g is all-gathered by the
library itself over NCCL (setbwte_set_comm) -> strong scaling
of one build.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BWT build Mbases/s at 1/2/4/8 B200; ComputeRanks queries/s; % HBM roofline"
UNIT = "Mbases/s"

WORKLOADS = {
    # name: (description, generator kwargs, block_suffixes)
    "c1": ("c1: 1,000 uniform reads x 100 bp, K=4 blocks", dict(m=1000, L=100), 25250),
    "c2": ("c2: 1M uniform reads x 100 bp (100 Mbp), M=2^24-suffix blocks",
           dict(m=1_000_000, L=100), 1 << 24),
    "c3": ("c3: 20M uniform reads x 100 bp (2 Gbp), M=2^27-suffix blocks",
           dict(m=20_000_000, L=100), 1 << 27),
    "c4": ("c4: 1M uniform reads of length U[1000,10000] (~5.5 Gbp), M=2^30-suffix blocks",
           dict(m=1_000_000, lo=1000, hi=10000), 1 << 30),
    "c5": ("c5: append 10M uniform reads x 100 bp (seed 2) into an existing 50M-read index "
           "(seed 1) whose B_ext is host-tiered (pinned host memory), M=2^27-suffix blocks",
           dict(m=10_000_000, L=100, base_m=50_000_000), 1 << 27),
}

# which library kernels make up which stage of Table 2's taxonomy
STAGE_OF = {
    "pack": "pack", "slot_offsets": "pack", "partition": "pack",
    "sort_init": "sort", "sort_tiny": "sort", "sort_small": "sort", "sort_medium": "sort",
    "sort_warp": "sort", "sort_ctl": "sort",
    "sort_chunkify": "sort", "digit_hist": "sort", "digit_scan": "sort", "digit_scatter": "sort",
    "compute_ranks": "rank", "slices": "rank", "gather": "gather", "gather_part": "gather",
    "gather_fetch": "gather", "insert": "insert",
    "sb_scan": "insert",
}


# algorithmic bytes of ConstructSA per suffix for uniform
# reads (24 B per active suffix-pass x 1.044 passes + 4 B SA write, rounded)
SORT_MODEL_B_PER_SUFFIX = 29.0


def stage_fractions(kern: dict, stages: dict, peak_gbs: float, n_suf: int):
    """Per stage (Table 2's taxonomy): algorithmic bytes / stage
    time / HBM peak, with the times of the serialised warm-up step (every
    stage on one stream, every launch timed).  Sort: SURVEY 8(d)'s model
    bytes (29 B/suffix) and the library's own count (every 8-bit digit pass
    and finish pass it ran); gather / insert / pack: the library's counts
    (DESIGN.md section 7); rank: LF steps/s against the measured random
    32-byte sector ceiling (profiles/r01_microbench.json) and HBM bytes."""
    def kb(names):
        return sum(v["bytes"] for k, v in kern.items() if k in names)
    out = {"timing": "serialised warm-up step (stage_ms_per_step)"}
    sort_names = [k for k in kern if k.startswith(("sort_", "digit_"))]
    for st, names in (("sort", sort_names), ("gather", ["gather", "gather_part", "gather_fetch"]),
                      ("insert", ["insert", "sb_scan"]), ("pack", ["pack", "slot_offsets"]),
                      ("rank", ["compute_ranks"])):
        ms = stages.get(st, 0.0)
        if ms <= 0:
            continue
        b = kb(names)
        e = {"ms": round(ms, 4), "bytes_lib": b,
             "frac_lib": round(b / (ms / 1e3) / 1e9 / peak_gbs, 4)}
        if st == "sort":
            mb = SORT_MODEL_B_PER_SUFFIX * n_suf
            e["bytes_model"] = mb
            e["frac_model"] = round(mb / (ms / 1e3) / 1e9 / peak_gbs, 4)
        if st == "rank":
            mbp = os.path.join(ROOT, "profiles", "r01_microbench.json")
            cr = kern.get("compute_ranks")
            if cr and os.path.exists(mbp):
                ceil = json.load(open(mbp)).get("gather32_hbm_gsectors_s")
                if ceil:
                    q = cr["units"] / (ms / 1e3)
                    e["lf_steps_per_s"] = q
                    e["frac_random_sector_ceiling"] = round(q / (ceil * 1e9), 4)
        out[st] = e
    return out


def golden_digest(workload: str):
    p = os.path.join(ROOT, "tests", "golden", "%s_bwt_digest.json" % workload)
    return json.load(open(p)) if os.path.exists(p) else None


def gen(workload: str, seed: int = 1):
    import synth
    _, kw, _ = WORKLOADS[workload]
    if "base_m" in kw:  # c5: the appended reads (the base index is built untimed)
        return synth.uniform(kw["m"], kw["L"], seed=2)
    if "L" in kw:
        return synth.uniform(kw["m"], kw["L"], seed=seed)
    return synth.uniform_var(kw["m"], kw["lo"], kw["hi"], seed=seed)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        """Start sampling; returns once nvidia-smi produces lines (its start-up
        can take longer than a short timed region), so every timed step is
        covered.  The lines seen while waiting are dropped."""
        self.ready = threading.Event()
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            self.ready.wait(timeout=10.0)
            self.lines = []
        except Exception:
            self.proc = None

    paused = False

    def pause(self):
        self.paused = True

    def resume(self):
        self.paused = False

    def _read(self):
        for line in self.proc.stdout:
            self.ready.set()
            if not self.paused:
                self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# reference arm: the oracle (the slow CPU program) on the box's host cores
# ---------------------------------------------------------------------------
def sample_reads(offsets, max_reads, max_bases):
    """The oracle's bounded sample: the longest prefix of the workload's reads
    with at most max_reads reads and max_bases bases (at least one read)."""
    m = len(offsets) - 1
    k = int(np.searchsorted(np.asarray(offsets, dtype=np.uint64), np.uint64(max_bases), side="right")) - 1
    return max(1, min(max_reads, m, k))


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return 0
    import oracle
    wl = args.workload
    data, offsets = gen(wl)
    m_sample = sample_reads(offsets, args.ref_sample_reads, args.ref_sample_bases)
    o = offsets[: m_sample + 1]
    d = data[: int(o[-1])]
    bases = float(o[-1])
    cores = cpu_count()
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.bwt("ACGT", d, o, threads=cores)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = sum(times)
    value = bases * len(times) / t / 1e6
    sample = "first %d reads (%d bases) of %s per step" % (m_sample, int(bases), wl)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * t / len(times), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": WORKLOADS[wl][0], "sample": sample},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    from paper_1410_0562_b200 import SetBWTE

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = args.workload
    desc, _, M = WORKLOADS[wl]
    if args.block_suffixes:
        M = args.block_suffixes
    data, offsets = gen(wl)
    m = len(offsets) - 1
    bases = int(offsets[-1])
    d_data = torch.from_numpy(data).to(dev)
    d_off = torch.from_numpy(offsets.view(np.int64)).to(dev)
    stream = torch.cuda.current_stream(dev)

    def new_index():
        ix = SetBWTE("ACGT", block_suffixes=M)
        after = ("insert_split", "shard_dict", "sort_split")  # need the partition first
        for kv in args.option:
            k, v = kv.split("=", 1)
            if k not in after:
                ix.set_option(k, int(v))
        ix.set_stream(stream)
        if world > 1:
            # N > 1: ComputeRanks split by string and block k sorted on rank
            # k mod N (its SA_int broadcast); Insert replicated (--option
            # insert_split=1 / shard_dict=2 select the split / sharded forms)
            # the exchange runs inside the library on NCCL, on its stream
            from paper_1410_0562_b200.dist import nccl_comm
            ix.set_comm(nccl_comm(), rank, world)
            ix.set_option("sort_split", 1)
        for kv in args.option:
            k, v = kv.split("=", 1)
            if k in after:
                ix.set_option(k, int(v))
        return ix

    base = None
    if "base_m" in WORKLOADS[wl][1]:
        import synth
        bd, bo = synth.uniform(WORKLOADS[wl][1]["base_m"], WORKLOADS[wl][1]["L"], seed=1)
        base = (torch.from_numpy(bd).to(dev), torch.from_numpy(bo.view(np.int64)).to(dev),
                len(bo) - 1, bd, bo)

    idx = new_index()

    def prepare():
        """Untimed: the index the step appends to (empty, or c5's host-tiered base)."""
        nonlocal idx
        if base is None:
            idx.clear()
        else:
            idx.close()
            idx = new_index()
            idx.append_device(base[0], base[1], base[2])
            idx.set_option("host_tier", 1)
        torch.cuda.synchronize(dev)

    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        idx.append_device(d_data, d_off, m)

    # warm-up: the LAST warm-up step runs with every stage on one stream and
    # every launch timed (per-kernel breakdown, dominant kernel: with the sort
    # lanes running, a launch's begin event can fire on an idle lane stream
    # before the host has submitted the kernel; and the first step pays each
    # kernel's lazy module load); the timed steps then put CUDA events around
    # the dominant kernel's launches only (events around every launch perturb
    # the pipeline by ~20 %)
    lanes_opt = [int(kv.split("=", 1)[1]) for kv in args.option if kv.startswith("sort_lanes=")]
    warm_kern = {}
    for w in range(args.warmup):
        prepare()
        prof_step = w == args.warmup - 1
        if prof_step:
            idx.set_option("sort_lanes", 0)
            idx.set_profile(1)
        else:
            idx.set_option("sort_lanes", lanes_opt[-1] if lanes_opt else 255)
            idx.set_profile(0)
        l2_flush.zero_()
        step()
        if prof_step:
            for k, v in idx.stats()["kernels"].items():
                a = warm_kern.setdefault(k, {"launches": 0, "ms": 0.0, "bytes": 0.0, "units": 0})
                for f in a:
                    a[f] += v[f]
    idx.set_option("sort_lanes", lanes_opt[-1] if lanes_opt else 255)
    torch.cuda.synchronize(dev)
    dom_name = max(warm_kern.items(), key=lambda kv: kv[1]["ms"])[0] if warm_kern else None

    def set_timed_profile():
        if dom_name:
            idx.set_profile(2, dom_name)

    kern = {}
    launches = 0
    blocks = None
    sampler = ClockSampler(local_rank)
    sampler.start()                          # returns once samples flow
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    times = []
    for _ in range(args.steps):
        if base is not None:
            sampler.pause()
        prepare()                            # untimed
        set_timed_profile()
        if base is not None:
            sampler.resume()
        l2_flush.zero_()                     # flush L2 between timed iterations (untimed)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        st = idx.stats()
        launches += st["launches"]
        blocks = st["blocks"]
        for k, v in st["kernels"].items():
            a = kern.setdefault(k, {"launches": 0, "ms": 0.0, "bytes": 0.0, "units": 0})
            for f in a:
                a[f] += v[f]
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    t_local = sum(times) / 1000.0
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    else:
        t = t_local
    value = bases * args.steps / t / 1e6

    # ---- end to end through the public API: pinned host in, BWT back out ----
    pin_data = torch.from_numpy(data).pin_memory()
    pin_off = torch.from_numpy(offsets.view(np.int64)).pin_memory()
    n_total = bases + m + (int(base[4][-1]) + base[2] if base is not None else 0)
    pin_out = torch.empty(n_total, dtype=torch.uint8).pin_memory()
    np_data = pin_data.numpy()
    np_off = pin_off.numpy().view(np.uint64)
    e2e_times = []
    for i in range(args.warmup + args.steps):
        prepare()
        idx.set_profile(0)
        l2_flush.zero_()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        idx.append(np_data, np_off)          # H2D of the step's inputs inside
        idx.bwt(pin_out)                      # D2H of the step's result
        e1.record(stream)
        e1.synchronize()
        if i >= args.warmup:
            e2e_times.append(e0.elapsed_time(e1))
    te = sum(e2e_times) / 1000.0
    if world > 1:
        tt = torch.tensor([te], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
    e2e_value = bases * len(e2e_times) / te / 1e6
    h2d = data.nbytes + offsets.nbytes
    d2h = n_total

    # ---- roofline of the dominant kernel ----
    peak, peak_src = load_peaks()
    dname = dom_name
    dk = kern[dname]
    per_launch_bytes = dk["bytes"] / max(dk["launches"], 1)
    avg_ms = dk["ms"] / max(dk["launches"], 1)
    achieved = per_launch_bytes / (avg_ms / 1000.0) / 1e9 if avg_ms > 0 else None
    # DRAM traffic of one captured launch of this kernel (ncu --set full,
    # profiles/traffic.json) next to that launch's algorithmic bytes
    traffic = None
    traffic_note = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        ent = json.load(open(tr_path)).get(dname)
        if ent:
            # the captured launch's DRAM bytes, scaled to this run's average
            # launch by the ratio of algorithmic bytes (the capture is one
            # full-size launch; the average mixes full and partial passes)
            dram = ent.get("dram_bytes_per_launch")
            alg = ent.get("algorithmic_bytes_per_launch")
            traffic = round(dram * per_launch_bytes / alg, 1) if dram and alg else dram
            traffic_note = {"captured_dram_bytes": dram, "captured_algorithmic_bytes": alg,
                            "launch": ent.get("launch"),
                            "scaled": bool(dram and alg)}
    roof = {"kernel": dname, "bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
            "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4) if achieved else None, "traffic": traffic,
            "traffic_launch": traffic_note,
            "bytes_per_launch": per_launch_bytes, "avg_launch_ms": round(avg_ms, 5),
            "share_of_step": round(dk["ms"] / (t_local * 1000.0), 4), "peak_source": peak_src}
    stages = {}
    for k, v in warm_kern.items():
        sname = STAGE_OF.get(k) or ("sort" if k.startswith(("sort_", "digit_")) else
                                    "insert" if k.startswith("insert") else "other")
        stages[sname] = stages.get(sname, 0.0) + v["ms"]
    cr = warm_kern.get("compute_ranks")
    qps = (cr["units"] / (cr["ms"] / 1000.0)) if cr and cr["ms"] > 0 else None
    stage_frac = stage_fractions(warm_kern, stages, peak, n_suf=bases + m)

    # ---- oracle beside it (rank 0, N = 1 only), + parity of this run ----
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and base is None:
        import oracle
        cores = cpu_count()
        m_s = sample_reads(offsets, args.cpu_sample_reads, args.cpu_sample_bases)
        o_s = offsets[: m_s + 1]
        d_s = data[: int(o_s[-1])]
        t0 = time.perf_counter()
        want = oracle.bwt("ACGT", d_s, o_s, threads=cores)
        dt = time.perf_counter() - t0
        cpu = {"value": round(float(o_s[-1]) / dt / 1e6, 3), "unit": UNIT, "cores": cores,
               "kind": "oracle",
               "sample": "first %d reads (%d bases) of %s, one build" % (m_s, int(o_s[-1]), wl)}
        if m_s == m:
            parity = "bit-exact" if bytes(pin_out.numpy()[:n_total]) == want else "MISMATCH"
    if rank == 0 and parity is None:
        # full-size parity through the oracle-written digest (tests/golden,
        # tools/make_golden_digests.py: bucketed oracle, BLAKE2b-128)
        gd = golden_digest(wl)
        if gd is not None and gd["n"] == n_total:
            import hashlib
            h = hashlib.blake2b(digest_size=16)
            h.update(memoryview(pin_out.numpy()[:n_total]))
            parity = ("bit-exact (BLAKE2b-128 of the whole BWT == oracle digest)"
                      if h.hexdigest() == gd["digest"]["hex"] else "MISMATCH")
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000.0 * t / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            # integer path: 2-bit symbols, u32 ranks / positions while the index
            # has < 2^32 symbols (u64 beyond)
            "dtype": "u32" if n_total < (1 << 32) else "u64", "data": "synthetic",
            "config": {"workload": desc, "reads": m, "bases": bases, "block_suffixes": M,
                       "host_tier": bool(idx.stats().get("host_tier")),
                       "blocks": blocks, "parallelism": "dp%d (ComputeRanks split by string)" % world,
                       "l2": "flushed between timed steps (256 MiB write, untimed)"},
            "compute_ranks_queries_per_s": qps, "stage_ms_per_step": stages,
            "stage_frac": stage_frac,
            "profile_note": "stage/kernel ms and queries/s from the last warm-up step, run with "
                            "every stage on one stream and every launch timed (serialised, so they "
                            "add up to more than ms_per_step); roofline from the timed steps "
                            "(pipelined, events on the dominant kernel only)",
            "kernel_ms_per_step": {k: round(v["ms"], 4) for k, v in
                                   sorted(warm_kern.items(), key=lambda kv: -kv[1]["ms"])},
            "roofline": roof, "cpu_baseline": cpu, "parity_vs_oracle": parity,
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    idx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--block-suffixes", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-reads", type=int, default=1_000_000)
    ap.add_argument("--cpu-sample-bases", type=int, default=100_000_000)
    ap.add_argument("--ref-sample-reads", type=int, default=100_000)
    ap.add_argument("--ref-sample-bases", type=int, default=10_000_000)
    ap.add_argument("--option", action="append", default=[],
                    help="library option key=value (setbwte_set_option), repeatable")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
