"""Break the e2e step into its parts (append from device / host, BWT read-back)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1410_0562_b200 import SetBWTE  # noqa: E402

d, o = synth.uniform(1_000_000, 100, seed=1)
pd = torch.from_numpy(d).pin_memory()
po = torch.from_numpy(o.view(np.int64)).pin_memory()
dd, do = pd.cuda(), po.cuda()
out = torch.empty(int(o[-1]) + len(o) - 1, dtype=torch.uint8).pin_memory()
idx = SetBWTE("ACGT", block_suffixes=1 << 24)


def t(f, n=5):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1000 * min(ts)


print("append_device ms", t(lambda: (idx.clear(), idx.append_device(dd, do))))
print("append_host   ms", t(lambda: (idx.clear(), idx.append(pd.numpy(), po.numpy().view(np.uint64)))))
print("bwt_host      ms", t(lambda: idx.bwt(out)))
dev_out = torch.empty_like(out, device="cuda")
print("bwt_device    ms", t(lambda: idx.bwt_device(dev_out)))
print("h2d 100MB     ms", t(lambda: dd.copy_(pd, non_blocking=True)))
print("d2h 101MB     ms", t(lambda: out.copy_(dev_out, non_blocking=True)))
