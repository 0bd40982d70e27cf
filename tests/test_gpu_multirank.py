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


def _run_ranks(world, split, appends, M, shard=False, keep=False, sort_split=False, lanes=None):
    from paper_1410_0562_b200 import SetBWTE
    make = _loopback(world)
    idx = []
    for r in range(world):
        h = SetBWTE(A, block_suffixes=M)
        h.set_partition(r, world, make(r))
        h.set_option("insert_split", split)
        if shard:
            h.set_option("shard_dict", 1)
        if sort_split:
            h.set_option("sort_split", 1)
        if lanes is not None:
            h.set_option("sort_lanes", lanes)
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
    out = [h.bwt() for h in idx]
    return (out, idx) if keep else out


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


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("seed", range(3))
def test_sharded_dictionary_random_sets(world, seed):
    """NEXT-3: B_ext sharded by output superblock range; every rank holds only
    its shard and reads the others' through their device pointers."""
    d, o = synth.random_set(18000 + seed, max_m=64, max_len=60)
    want = oracle.bwt(A, d, o)
    m = len(o) - 1
    apps = _split_appends(d, o, [m // 2] if m > 2 else [])
    for got in _run_ranks(world, 1, apps, M=120, shard=True):
        assert got == want


def test_sharded_dictionary_c1_queries():
    d, o = synth.uniform(3000, 100, seed=9)
    want = oracle.bwt(A, d, o, threads=None)
    apps = _split_appends(d, o, [1000, 2000])
    outs, idx = _run_ranks(3, 1, apps, M=40000, shard=True, keep=True)
    for got in outs:
        assert got == want
    # rank / count queries read every shard
    rng = np.random.default_rng(2)
    B = np.frombuffer(want, dtype=np.uint8)
    for k in rng.integers(0, len(want) + 1, size=6):
        for c in "$ACGT":
            assert idx[1].rank(c, int(k)) == int((B[:int(k)] == ord(c)).sum())
    starts = rng.integers(0, len(d) - 10, size=30)
    pats = [bytes(d[a:a + 7]).decode() for a in starts]
    assert np.array_equal(idx[2].count(pats), oracle.count(A, d, o, pats))


@pytest.mark.parametrize("world,shard,lanes", [(2, False, None), (3, True, None), (2, True, 0),
                                               (4, False, 1)])
def test_sort_split(world, shard, lanes):
    """Block k sorted on rank k mod P only; its SA_int is shared through the
    exchange (NEXT-1 across GPUs)."""
    d, o = synth.uniform(4000, 100, seed=31)
    want = oracle.bwt(A, d, o, threads=None)
    apps = _split_appends(d, o, [1500])
    for got in _run_ranks(world, 1, apps, M=30000, shard=shard, sort_split=True, lanes=lanes):
        assert got == want
