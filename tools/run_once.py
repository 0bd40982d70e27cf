"""Build one workload once through the C-ABI (for ncu / sanitizer runs)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1410_0562_b200 import SetBWTE  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reads", type=int, default=1_000_000)
ap.add_argument("--len", type=int, default=100)
ap.add_argument("--M", type=int, default=1 << 24)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--genome", type=int, default=0)
ap.add_argument("--var", action="store_true", help="c4-style read lengths U[1000, 10000]")
ap.add_argument("--option", action="append", default=[], help="library option key=value")
a = ap.parse_args()
if a.var:
    d, o = synth.uniform_var(a.reads, 1000, 10000, seed=1)
elif a.genome:
    d, o = synth.genome_sampled(a.reads, a.len, a.genome, seed=1)
else:
    d, o = synth.uniform(a.reads, a.len, seed=1)
dd = torch.from_numpy(d).cuda()
do = torch.from_numpy(o.view(np.int64)).cuda()
idx = SetBWTE("ACGT", block_suffixes=a.M)
for kv in a.option:
    k, v = kv.split("=", 1)
    idx.set_option(k, int(v))
for _ in range(a.repeat):
    idx.clear()
    idx.append_device(dd, do)
torch.cuda.synchronize()
print("ok", idx.size(), idx.stats()["sort"])
