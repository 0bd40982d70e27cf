"""The in-library exchange (setbwte_set_comm) and the Python
all-gather helper.

* NCCL: a world-1 NCCL communicator (this pool gives one GPU per run, and NCCL
  refuses two ranks on one device) with option "force_exchange", so every
  block runs the partitioned ComputeRanks (slices precomputed once per append)
  and the exchange is a real ncclGroupStart / ncclBroadcast / ncclGroupEnd on
  the library's stream.  The BWT must equal the oracle's.
* make_allgather (dist.py) without set_stream: two processes on one GPU over
  gloo; the callback must order its collectives after the library's stream
  (it used torch's current stream).  No kernel waits on the other
  process -- gloo exchanges through the host.
"""
import os
import socket
import tempfile

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


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    f = tempfile.NamedTemporaryFile(delete=False)
    f.close()
    store = dist.FileStore(f.name, 1)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    from paper_1410_0562_b200.dist import nccl_comm
    comm = nccl_comm()
    yield comm
    dist.destroy_process_group()
    os.unlink(f.name)


def test_set_comm_validates(nccl_world1):
    from paper_1410_0562_b200 import SetBWTE, SetBWTEError
    idx = SetBWTE(A)
    with pytest.raises(SetBWTEError) as e:
        idx.set_comm(nccl_world1, 0, 2)          # communicator has 1 rank
    assert e.value.name == "E_INVALID_ARG"
    with pytest.raises(SetBWTEError):
        idx.set_comm(nccl_world1, 1, 1)          # rank out of range
    idx.set_comm(nccl_world1, 0, 1)
    idx.set_comm(0, 0, 1)                        # detach
    idx.close()


@pytest.mark.parametrize("seed,M,g8", [(21000, 600, 0), (21001, 25250, 0), (21002, 2000, 1)])
def test_nccl_exchange_path_matches_oracle(nccl_world1, seed, M, g8):
    from paper_1410_0562_b200 import SetBWTE
    if seed == 21001:
        d, o = synth.uniform(1000, 100, seed=1)   # c1
    else:
        d, o = synth.random_set(seed, max_m=120, max_len=90)
    idx = SetBWTE(A, block_suffixes=M)
    idx.set_comm(nccl_world1, 0, 1)
    idx.set_option("force_exchange", 1)
    if g8:
        idx.set_option("g_width", 8)
    m = len(o) - 1
    cut = m // 3
    oo = np.asarray(o, dtype=np.uint64)
    idx.append(d[: int(oo[cut])], oo[: cut + 1])           # first append: B_ext empty
    idx.append(d[int(oo[cut]):], oo[cut:] - oo[cut])       # ranks against a real B_ext
    assert idx.bwt() == oracle.bwt(A, d, o)
    idx.close()


def test_nccl_exchange_with_insert_and_sort_split(nccl_world1):
    """Every exchange of the world > 1 path through NCCL: g slices, the
    sorting rank's SA_int (sort_split) and the dictionary slices + superblock
    totals (insert_split)."""
    from paper_1410_0562_b200 import SetBWTE
    d, o = synth.random_set(21010, max_m=100, max_len=80)
    idx = SetBWTE(A, block_suffixes=700)
    idx.set_comm(nccl_world1, 0, 1)
    idx.set_option("force_exchange", 1)
    idx.set_option("insert_split", 1)
    idx.set_option("sort_split", 1)
    m = len(o) - 1
    oo = np.asarray(o, dtype=np.uint64)
    idx.append(d[: int(oo[m // 2])], oo[: m // 2 + 1])
    idx.append(d[int(oo[m // 2]):], oo[m // 2:] - oo[m // 2])
    assert idx.bwt() == oracle.bwt(A, d, o)
    idx.close()


def _worker(rank, world, port, seed, q):
    try:
        import torch
        import torch.distributed as dist

        from paper_1410_0562_b200 import SetBWTE
        from paper_1410_0562_b200.dist import make_allgather

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank,
                                world_size=world)
        d, o = synth.random_set(seed, max_m=100, max_len=80)
        idx = SetBWTE(A, block_suffixes=400)     # the library's own stream: no set_stream
        idx.set_partition(rank, world, make_allgather())
        m = len(o) - 1
        cut = m // 2
        oo = np.asarray(o, dtype=np.uint64)
        idx.append(d[: int(oo[cut])], oo[: cut + 1])
        idx.append(d[int(oo[cut]):], oo[cut:] - oo[cut])
        ok = idx.bwt() == oracle.bwt(A, d, o)
        idx.close()
        dist.destroy_process_group()
        q.put((rank, bool(ok), None))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("seed", [21100, 21101])
def test_make_allgather_without_set_stream(seed):
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
