"""Kernel-level ComputeRanks scaling on ONE GPU ("report
kernel-level ComputeRanks scaling (queries/s per GPU x P)"): with the
partition of setbwte_set_comm / set_partition, rank 0 of P ranks computes g
for its suffix-balanced 1/P of a block's strings.  This times exactly that
kernel -- c3's last block (2^27 suffixes, 1.33 M reads) ranked into the index
of the first 18.67 M reads (~1.9 G symbols) -- for P = 1, 2, 4, 8; the
exchange (an NCCL all-gather-v of g) is not in it.

    python tools/rank_scaling.py  -> one JSON line
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1410_0562_b200 import SetBWTE  # noqa: E402

d, o = synth.uniform(20_000_000, 100, seed=1)
cut = 20_000_000 - 1_328_889
oo = np.asarray(o, dtype=np.uint64)
idx = SetBWTE("ACGT", block_suffixes=1 << 27)
idx.append(d[: int(oo[cut])], oo[: cut + 1])
bd, bo = d[int(oo[cut]):], oo[cut:] - oo[cut]
out = {"what": "compute_ranks kernel time of rank 0 of P (its 1/P of c3's last block), one B200",
       "index_symbols": idx.size()[0], "block_suffixes": int(bo[-1]) + len(bo) - 1}
res = {}
for P in (1, 2, 4, 8):
    idx.set_partition(0, P, (lambda *a: None) if P > 1 else None)
    idx.set_profile(1)
    best = None
    for _ in range(3):
        idx.compute_ranks(bd, bo)
        k = idx.stats()["kernels"]["compute_ranks"]
        if best is None or k["ms"] < best["ms"]:
            best = k
    res[P] = {"ms": round(best["ms"], 4), "lf_steps": best["units"],
              "lf_steps_per_s_per_gpu": best["units"] / (best["ms"] / 1e3)}
t1 = res[1]["ms"]
for P, r in res.items():
    r["speedup_vs_1"] = round(t1 / r["ms"], 3)
    r["aggregate_lf_steps_per_s"] = r["lf_steps_per_s_per_gpu"] * P
out["P"] = res
print(json.dumps(out))
