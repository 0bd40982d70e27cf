"""Multi-process host logic of data-parallel ComputeRanks, on
CPU with the gloo backend, world_size 2: suffix-balanced string slices and the
all-gather-v that assembles g on every rank.  Per-rank g slices come from the
oracle (this exercises the exchange, not the kernels)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1410_0562_b200.dist import allgather_slices, balanced_slices


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank,
                                world_size=world)
        d, o = synth.random_set(11, max_m=40, max_len=30)
        strings = synth.to_strings(d, o)
        cut = len(strings) // 3
        full_g = oracle.compute_ranks("ACGT", d, o, m_ext=cut)   # block = strings[cut:]
        blk = strings[cut:]
        slot_off = np.zeros(len(blk) + 1, dtype=np.int64)
        slot_off[1:] = np.cumsum([len(s) + 1 for s in blk])
        sl = balanced_slices(slot_off, 0, len(blk), world)
        # each rank fills only its slice of the (u64) g buffer, as the library does
        buf = torch.zeros(int(slot_off[-1]) * 8, dtype=torch.uint8)
        a, b = int(slot_off[sl[rank]]), int(slot_off[sl[rank + 1]])
        mine = torch.from_numpy(full_g[a:b].astype(np.uint64).view(np.uint8).copy())
        buf[a * 8:b * 8] = mine
        bytes_per_rank = [8 * int(slot_off[sl[r + 1]] - slot_off[sl[r]]) for r in range(world)]
        allgather_slices(buf, bytes_per_rank)
        got = buf.numpy().view(np.uint64)
        q.put((rank, bool(np.array_equal(got, full_g)), sl))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None))


def test_allgather_v_assembles_g_on_every_rank():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, sl in res:
        assert ok is True, (rank, ok)
    # both ranks computed the same slices, covering all strings
    assert res[0][2] == res[1][2]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_balanced_slices_partition(world):
    d, o = synth.uniform_var(200, 1, 300, seed=world)
    lens = np.diff(o.astype(np.int64))
    slot_off = np.zeros(len(lens) + 1, dtype=np.int64)
    slot_off[1:] = np.cumsum(lens + 1)
    sl = balanced_slices(slot_off, 0, len(lens), world)
    assert sl[0] == 0 and sl[-1] == len(lens)
    assert all(a <= b for a, b in zip(sl[:-1], sl[1:]))
    # every slice starts at the first string reaching its suffix target
    total = slot_off[-1]
    for r in range(1, world):
        target = total * r // world
        j = sl[r]
        assert slot_off[j] >= target and (j == 0 or slot_off[j - 1] < target)
