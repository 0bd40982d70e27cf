"""NEXT-3 in the one-process-per-rank model: the sharded dictionary with
shard_dict = 2, where ranks are separate processes and exchange CUDA IPC
handles of their shards.  Two processes on ONE GPU, exchanging through gloo on
the host (the callback syncs its stream, copies its slice to the host, and
all-gathers with torch.distributed); no kernel waits on another process.  Both
ranks must end with the oracle's BWT."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

A = "ACGT"
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, seed, q):
    try:
        import torch
        import torch.distributed as dist

        from paper_1410_0562_b200 import SetBWTE
        from paper_1410_0562_b200.dist import _CAI

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank,
                                world_size=world)

        def cb(buf_ptr, bpr, world_, stream_ptr):
            torch.cuda.ExternalStream(stream_ptr).synchronize()
            buf = torch.as_tensor(_CAI(buf_ptr, sum(bpr)), device="cuda")
            off = sum(bpr[:rank])
            mine = buf[off:off + bpr[rank]].cpu().numpy().tobytes()
            parts = [None] * world_
            dist.all_gather_object(parts, mine)
            o = 0
            for r in range(world_):
                if r != rank and bpr[r]:
                    src = torch.frombuffer(bytearray(parts[r]), dtype=torch.uint8)
                    buf[o:o + bpr[r]].copy_(src)
                o += bpr[r]
            torch.cuda.synchronize()

        d, o = synth.random_set(seed, max_m=80, max_len=70)
        idx = SetBWTE(A, block_suffixes=300)
        idx.set_partition(rank, world, cb)
        idx.set_option("shard_dict", 2)
        m = len(o) - 1
        cut = m // 2
        oo = np.asarray(o, dtype=np.uint64)
        idx.append(d[: int(oo[cut])], oo[: cut + 1])
        idx.append(d[int(oo[cut]):], oo[cut:] - oo[cut])
        got = idx.bwt()
        ok = got == oracle.bwt(A, d, o)
        # queries read every shard through the opened IPC handles
        B = np.frombuffer(got, dtype=np.uint8)
        k = len(got) // 2
        ok = ok and idx.rank("A", k) == int((B[:k] == ord("A")).sum())
        idx.close()
        dist.destroy_process_group()
        q.put((rank, bool(ok), None))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("seed", [19000, 19001])
def test_sharded_dictionary_across_processes(seed):
    import torch.multiprocessing as mp
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, (rank, err)
