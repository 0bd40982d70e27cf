"""Where the end-to-end step's time goes (python tools/e2e_probe.py [c2|c3]) (GPU box): wall-clock of
append_device / append from pinned host / bwt into pinned host / bwt_device."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1410_0562_b200 import SetBWTE  # noqa: E402

WL = sys.argv[1] if len(sys.argv) > 1 else "c2"
data, offsets = bench.gen(WL)
m = len(offsets) - 1
dev = torch.device("cuda:0")
d_data = torch.from_numpy(data).to(dev)
d_off = torch.from_numpy(offsets.view(np.int64)).to(dev)
pin_data = torch.from_numpy(data).pin_memory()
pin_off = torch.from_numpy(offsets.view(np.int64)).pin_memory()
np_data, np_off = pin_data.numpy(), pin_off.numpy().view(np.uint64)
idx = SetBWTE("ACGT", block_suffixes=bench.WORKLOADS[WL][2])
pin_out = torch.empty(int(offsets[-1]) + m, dtype=torch.uint8).pin_memory()
d_out = torch.empty_like(pin_out, device=dev)


def t(f, reps=4 if WL != "c2" else 12):
    out = []
    for _ in range(reps):
        idx.clear()
        torch.cuda.synchronize()
        a = time.perf_counter()
        f()
        torch.cuda.synchronize()
        out.append((time.perf_counter() - a) * 1e3)
    return "min %.2f med %.2f ms  all %s" % (min(out), sorted(out)[len(out) // 2],
                                            " ".join("%.1f" % x for x in out))


for _ in range(3):
    idx.clear()
    idx.append_device(d_data, d_off, m)
torch.cuda.synchronize()
print("append_device      ", t(lambda: idx.append_device(d_data, d_off, m)))
print("append pinned host ", t(lambda: idx.append(np_data, np_off)))
print("append pageable    ", t(lambda: idx.append(data, offsets)))
print("append+bwt pinned  ", t(lambda: (idx.append(np_data, np_off), idx.bwt(pin_out))))
print("append_device again", t(lambda: idx.append_device(d_data, d_off, m)))
idx.clear()
idx.append_device(d_data, d_off, m)
torch.cuda.synchronize()


def tb(f, reps=6):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        f()
        torch.cuda.synchronize()
        out.append((time.perf_counter() - a) * 1e3)
    return "min %.2f med %.2f ms" % (min(out), sorted(out)[len(out) // 2])


print("bwt pinned host    ", tb(lambda: idx.bwt(pin_out)))
print("bwt device         ", tb(lambda: idx.bwt_device(d_out)))
print("torch H2D inputs   ", tb(lambda: (d_data.copy_(pin_data, non_blocking=True), d_off.copy_(pin_off, non_blocking=True))))
print("torch D2H BWT      ", tb(lambda: pin_out.copy_(d_out, non_blocking=True)))
import os
print("cpus", os.cpu_count(), "load", os.getloadavg())
