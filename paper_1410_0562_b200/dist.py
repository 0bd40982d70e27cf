"""Multi-process plumbing for data-parallel ComputeRanks.

Each rank holds a replica of B_ext and computes g for its own contiguous,
suffix-balanced slice of every block's strings (Alg.2 P:110 "for all j" is
independent per string); the slices are then assembled on every rank by one
exchange -- an all-gather-v of the g slices.  The library calls back into
``make_allgather``'s function with the device buffer; the exchange itself is a
sequence of NCCL broadcasts (one per source rank) through torch.distributed,
queued on the library's stream.  The production form is ``SetBWTE.set_comm``
with ``nccl_comm(group)``: the library then issues the NCCL group itself, on
its own stream, with no Python call per block.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class _CAI:
    """A raw device buffer exposed through __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
            "strides": None,
        }


def allgather_slices(buf: torch.Tensor, bytes_per_rank, group=None):
    """All-gather-v in place: rank r's slice is buf[off_r : off_r + bytes_per_rank[r]]
    (already filled on rank r); afterwards every slice is filled on every rank."""
    off = 0
    for r, nb in enumerate(bytes_per_rank):
        if nb:
            src = dist.get_global_rank(group, r) if group is not None else r
            dist.broadcast(buf[off:off + nb], src=src, group=group)
        off += nb
    return buf


def make_allgather(group=None):
    """Callback for SetBWTE.set_partition: (buf_ptr, bytes_per_rank, world, stream_ptr)."""

    def _cb(buf_ptr: int, bytes_per_rank, world: int, stream_ptr: int):
        total = sum(bytes_per_rank)
        buf = torch.as_tensor(_CAI(buf_ptr, total), device="cuda")
        # the slices are only QUEUED on the library's stream: issue the
        # collectives on that same stream, so they run after ComputeRanks wrote
        # this rank's slice and before the gather reads the others
        with torch.cuda.stream(torch.cuda.ExternalStream(stream_ptr)):
            allgather_slices(buf, bytes_per_rank, group)

    return _cb


def nccl_comm(group=None) -> int:
    """Address of the ncclComm_t behind a torch.distributed NCCL group (the
    default group if None), for SetBWTE.set_comm.  The communicator is created
    eagerly if the group has not used it yet."""
    g = group if group is not None else dist.group.WORLD
    dev = torch.device("cuda", torch.cuda.current_device())
    backend = g._get_backend(dev)
    ptr = int(backend._comm_ptr())
    if ptr == 0:
        # lazily initialised communicator: one tiny collective creates it
        t = torch.zeros(1, device=dev)
        dist.all_reduce(t, group=g)
        torch.cuda.synchronize(dev)
        ptr = int(backend._comm_ptr())
    return ptr


def balanced_slices(slot_off, j0: int, j1: int, parts: int):
    """Host mirror of the library's slice rule (pack.cu slices_kernel): slice r
    starts at the first string whose slot offset reaches S0 + r*(S1-S0)/parts."""
    import bisect
    S0, S1 = int(slot_off[j0]), int(slot_off[j1])
    out = []
    for r in range(parts):
        target = S0 + (S1 - S0) * r // parts
        out.append(bisect.bisect_left(list(slot_off[j0:j1 + 1]), target) + j0)
    out.append(j1)
    return out
