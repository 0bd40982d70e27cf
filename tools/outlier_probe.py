"""Find slow c2 append_device calls and print their sort statistics (GPU box)."""
import gc
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1410_0562_b200 import SetBWTE  # noqa: E402

gcoff = "--nogc" in sys.argv
wl = ([a.split("=")[1] for a in sys.argv if a.startswith("wl=")] or ["c2"])[0]
iters = int(([a.split("=")[1] for a in sys.argv if a.startswith("iters=")] or ["60"])[0])
data, offsets = bench.gen(wl)
m = len(offsets) - 1
dev = torch.device("cuda:0")
d_data = torch.from_numpy(data).to(dev)
d_off = torch.from_numpy(offsets.view(np.int64)).to(dev)
idx = SetBWTE("ACGT", block_suffixes=bench.WORKLOADS[wl][2])
for kv in sys.argv[1:]:
    if "=" in kv and not kv.startswith(("wl=", "iters=")):
        k, v = kv.split("=")
        idx.set_option(k, int(v))
prof = "--prof" in sys.argv
if prof:
    idx.set_profile(1)
if gcoff:
    gc.disable()
import resource


def steal():
    f = open("/proc/stat").readline().split()
    return int(f[8]), int(f[4])  # steal, idle (jiffies)


ts = []
for i in range(iters):
    s0 = steal()
    r0 = resource.getrusage(resource.RUSAGE_SELF)
    idx.clear()
    torch.cuda.synchronize()
    a = time.perf_counter()
    idx.append_device(d_data, d_off, m)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - a) * 1e3
    s1 = steal()
    r1 = resource.getrusage(resource.RUSAGE_SELF)
    st = idx.stats()
    ts.append(dt)
    info = "steal %d idle %d nivcsw %d nvcsw %d minflt %d" % (
        s1[0] - s0[0], s1[1] - s0[1], r1.ru_nivcsw - r0.ru_nivcsw, r1.ru_nvcsw - r0.ru_nvcsw,
        r1.ru_minflt - r0.ru_minflt)
    if prof:
        ks = sorted(st["kernels"].items(), key=lambda kv: -kv[1]["ms"])
        info += " ksum %.2f ms top %s" % (sum(v["ms"] for _, v in ks),
                                          " ".join("%s=%.2f" % (k, v["ms"]) for k, v in ks[:4]))
    if i >= 3 and (dt > 1.4 * np.median(ts) or i % 10 == 0):
        print("%s %d: %.1f ms  %s" % ("slow" if dt > 9 else "ok  ", i, dt, info))
ts = np.array(ts[3:])
print("median %.2f mean %.2f p90 %.2f max %.2f" % (np.median(ts), ts.mean(), np.percentile(ts, 90), ts.max()))
