"""Multi-process plumbing for data-parallel ComputeRanks.

Each rank holds a replica of B_ext and computes g for its own contiguous,
suffix-balanced slice of every block's strings (Alg.2 P:110 "for all j" is
independent per string); the slices are then assembled on every rank by one
exchange -- an all-gather-v of the g slices.  The library calls back into
``make_allgather``'s function with the device buffer; the exchange itself is a
sequence of NCCL broadcasts (one per source rank) through torch.distributed,
queued on the library's stream.
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
        # the library's stream is torch's current stream (bench sets it), so the
        # collectives are ordered after ComputeRanks and before the gather.
        allgather_slices(buf, bytes_per_rank, group)

    return _cb


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
