"""Stage overlap of one pipelined append (setbwte_set_profile mode 3).

    python tools/timeline.py [--workload c3] [--json out.json]

Builds the workload twice untimed (warm-up), then once with every launch
bracketed by events (which perturbs the pipeline by ~20 %), and reports, over
the append's span, how long the sort lanes' kernels, the main stream's
kernels (ComputeRanks / gather / Insert) and the pack ran -- alone, together,
or not at all (GPU idle)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1410_0562_b200 import SetBWTE  # noqa: E402

SORT = ("sort_", "digit_")
MAIN = ("compute_ranks", "gather", "insert", "sb_scan", "slices")
PACK = ("pack", "slot_offsets", "partition")


def cat(name):
    if name.startswith(SORT):
        return "sort"
    if name.startswith(MAIN):
        return "main"
    if name.startswith(PACK):
        return "pack"
    return "other"


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def overlap_profile(tl):
    """Time in ms with (sort busy, main busy) in each of the four states."""
    ev = []
    for name, _, t0, t1 in tl:
        c = cat(name)
        if c in ("sort", "main"):
            ev.append((t0, 1, c))
            ev.append((t1, -1, c))
    ev.sort()
    busy = {"sort": 0, "main": 0}
    acc = {"both": 0.0, "sort only": 0.0, "main only": 0.0, "neither": 0.0}
    last = ev[0][0] if ev else 0.0
    for t, d, c in ev:
        key = ("both" if busy["sort"] and busy["main"] else "sort only" if busy["sort"]
               else "main only" if busy["main"] else "neither")
        acc[key] += t - last
        busy[c] += d
        last = t
    return acc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    desc, _, M = bench.WORKLOADS[a.workload]
    data, offsets = bench.gen(a.workload)
    dd = torch.from_numpy(data).cuda()
    do = torch.from_numpy(offsets.view(np.int64)).cuda()
    idx = SetBWTE("ACGT", block_suffixes=M)
    idx.set_stream(torch.cuda.current_stream())
    for _ in range(2):
        idx.clear()
        idx.append_device(dd, do)
    torch.cuda.synchronize()
    idx.clear()
    idx.set_profile(3)
    idx.append_device(dd, do)
    torch.cuda.synchronize()
    st = idx.stats()
    idx.set_profile(0)
    tl = st["timeline"]
    span = max(t1 for _, _, _, t1 in tl) - min(t0 for _, _, t0, _ in tl)
    per = {}
    for name, _, t0, t1 in tl:
        per.setdefault(cat(name), []).append((t0, t1))
    res = {"workload": desc, "launches": len(tl), "span_ms": round(span, 3),
           "busy_ms": {c: round(sum(b - a for a, b in union(v)), 3) for c, v in per.items()},
           "kernel_sum_ms": {c: round(sum(b - a for a, b in v), 3) for c, v in per.items()},
           "overlap_ms": {k: round(v, 3) for k, v in overlap_profile(tl).items()}}
    # when each block's main-stream work starts and ends
    main_iv = sorted((t0, t1, n) for n, _, t0, t1 in tl if cat(n) == "main")
    res["first_main_ms"] = round(main_iv[0][0], 3) if main_iv else None
    print(json.dumps(res, indent=1))
    if a.json:
        json.dump({"summary": res, "timeline": tl}, open(a.json, "w"))


if __name__ == "__main__":
    main()
