"""The library's world > 1 path (ComputeRanks split by string,
all-gather-v of g, and Insert split by output range with all-gathered
dictionary slices) on ONE GPU: P handles in one process, each with its own
rank, driven from P host threads.  The exchange callback is a host-side
loopback (stream sync, device copies, a threading.Barrier), so no kernel ever
waits on another rank -- only the host does.  Every rank must end with the
oracle's BWT."""
import threading

import numpy as np
import pytest

import oracle
import synth

A = "ACGT"
pytestmark = pytest.mark.gpu


def _loopback(world):
    import torch

    from paper_1410_0562_b200.dist import _CAI

    bar = threading.Barrier(world, timeout=120)
    store = [None] * world

    def make(rank):
        def cb(buf_ptr, bpr, world_, stream_ptr):
            total = sum(bpr)
            torch.cuda.ExternalStream(stream_ptr).synchronize()  # this rank's slice is done
            buf = torch.as_tensor(_CAI(buf_ptr, total), device="cuda")
            off = sum(bpr[:rank])
            store[rank] = buf[off:off + bpr[rank]].clone()
            torch.cuda.synchronize()
            bar.wait()
            o = 0
            for q in range(world_):
                if q != rank and bpr[q]:
                    buf[o:o + bpr[q]].copy_(store[q])
                o += bpr[q]
            torch.cuda.synchronize()
            bar.wait()  # nobody reuses `store` before everyone copied
        return cb

    return make


def _run_ranks(world, split, appends, M):
    from paper_1410_0562_b200 import SetBWTE
    make = _loopback(world)
    idx = []
    for r in range(world):
        h = SetBWTE(A, block_suffixes=M)
        h.set_partition(r, world, make(r))
        h.set_option("insert_split", split)
        idx.append(h)
    errs = [None] * world

    def run(r):
        try:
            for d, o in appends:
                idx[r].append(d, o)
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert errs == [None] * world, errs
    return [h.bwt() for h in idx]


def _split_appends(d, o, cuts):
    o = np.asarray(o, dtype=np.uint64)
    out = []
    bounds = [0] + list(cuts) + [len(o) - 1]
    for a, b in zip(bounds[:-1], bounds[1:]):
        oo = o[a:b + 1]
        out.append((d[int(oo[0]):int(oo[-1])], oo - oo[0]))
    return out


@pytest.mark.parametrize("world,split", [(2, 0), (2, 1), (3, 1)])
@pytest.mark.parametrize("seed", range(3))
def test_multirank_random_sets(world, split, seed):
    d, o = synth.random_set(12000 + seed, max_m=64, max_len=60)
    want = oracle.bwt(A, d, o)
    m = len(o) - 1
    apps = _split_appends(d, o, [m // 3] if m > 3 else [])
    for got in _run_ranks(world, split, apps, M=150):
        assert got == want


@pytest.mark.parametrize("world,split", [(2, 1), (4, 1), (4, 0)])
def test_multirank_c1(world, split):
    d, o = synth.uniform(1000, 100, seed=1)
    want = oracle.bwt(A, d, o, threads=None)
    apps = _split_appends(d, o, [300, 700])
    for got in _run_ranks(world, split, apps, M=25250):
        assert got == want
