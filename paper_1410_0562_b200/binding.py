"""Thin ctypes binding of libsetbwte.so (include/setbwte.h).

Argument marshalling only: every step of the set-bwte path runs in the CUDA
kernels of the library.  There is NO CPU fallback -- if the library is missing
or no CUDA device is present, calls raise.  Device buffers are passed as torch
CUDA tensors (their data_ptr), host buffers as numpy arrays / bytes.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SETBWTE_LIB") or os.path.join(_PKG, "libsetbwte.so")

STATUS = {
    0: "OK", 1: "E_INVALID_ARG", 2: "E_INVALID_CHAR", 3: "E_OUT_OF_RANGE", 4: "E_NOMEM",
    5: "E_CUDA", 6: "E_UNSUPPORTED", 7: "E_STATE", 8: "E_NCCL",
}

_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, _u64p, ctypes.c_int,
                                ctypes.c_void_p, ctypes.c_void_p)
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)

#: every symbol include/setbwte.h declares
EXPORTS = [
    "setbwte_create", "setbwte_destroy", "setbwte_strerror", "setbwte_append",
    "setbwte_append_device", "setbwte_prepend", "setbwte_prepend_device", "setbwte_merge",
    "setbwte_clear", "setbwte_size", "setbwte_bwt", "setbwte_bwt_device",
    "setbwte_rank", "setbwte_rank_batch", "setbwte_count", "setbwte_count_device",
    "setbwte_construct_sa", "setbwte_compute_ranks",
    "setbwte_set_option", "setbwte_set_profile", "setbwte_set_stream", "setbwte_set_partition",
    "setbwte_set_comm", "setbwte_set_allocator", "setbwte_stats",
    "setbwte_last_error",
]


class SetBWTEError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__("%s: %s%s" % (where, self.name, (" (" + detail + ")") if detail else ""))


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsetbwte.so and declare argument types.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError("libsetbwte.so not built (%s); run __graft_entry__.build()" % path)
    lib = ctypes.CDLL(path)
    vp, c64 = ctypes.c_void_p, ctypes.c_uint64
    sig = {
        "setbwte_create": ([ctypes.c_char_p, ctypes.POINTER(vp)], ctypes.c_int),
        "setbwte_destroy": ([vp], None),
        "setbwte_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "setbwte_append": ([vp, _u8p, _u64p, c64], ctypes.c_int),
        "setbwte_append_device": ([vp, vp, vp, c64], ctypes.c_int),
        "setbwte_prepend": ([vp, _u8p, _u64p, c64], ctypes.c_int),
        "setbwte_prepend_device": ([vp, vp, vp, c64], ctypes.c_int),
        "setbwte_merge": ([vp, vp], ctypes.c_int),
        "setbwte_clear": ([vp], ctypes.c_int),
        "setbwte_size": ([vp, _u64p, _u64p], ctypes.c_int),
        "setbwte_bwt": ([vp, vp, c64, _u64p], ctypes.c_int),
        "setbwte_bwt_device": ([vp, vp, c64, _u64p], ctypes.c_int),
        "setbwte_rank": ([vp, ctypes.c_uint8, c64, _u64p], ctypes.c_int),
        "setbwte_rank_batch": ([vp, vp, vp, c64, vp], ctypes.c_int),
        "setbwte_count": ([vp, _u8p, _u64p, c64, _u64p], ctypes.c_int),
        "setbwte_count_device": ([vp, vp, vp, c64, vp], ctypes.c_int),
        "setbwte_construct_sa": ([vp, _u8p, _u64p, c64, _u32p, _u8p], ctypes.c_int),
        "setbwte_compute_ranks": ([vp, _u8p, _u64p, c64, _u64p], ctypes.c_int),
        "setbwte_set_option": ([vp, ctypes.c_char_p, c64], ctypes.c_int),
        "setbwte_set_stream": ([vp, vp], ctypes.c_int),
        "setbwte_set_profile": ([vp, ctypes.c_int, ctypes.c_char_p], ctypes.c_int),
        "setbwte_set_partition": ([vp, ctypes.c_int, ctypes.c_int, ALLGATHER_FN, vp],
                                  ctypes.c_int),
        "setbwte_set_comm": ([vp, vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "setbwte_set_allocator": ([vp, ALLOC_FN, FREE_FN, vp], ctypes.c_int),
        "setbwte_stats": ([vp, ctypes.c_char_p, c64, _u64p], ctypes.c_int),
        "setbwte_last_error": ([vp, _u64p, _u8p], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name, None)
        if f is None:  # an older library build (A/B variants): the call is unavailable
            continue
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _host_u8(data):
    if isinstance(data, (bytes, bytearray)):
        data = np.frombuffer(bytes(data), dtype=np.uint8)
    arr = np.ascontiguousarray(data, dtype=np.uint8)
    if arr.size == 0:
        arr = np.zeros(1, dtype=np.uint8)
    return arr, arr.ctypes.data_as(_u8p)


def _host_u64(a):
    arr = np.ascontiguousarray(a, dtype=np.uint64)
    return arr, arr.ctypes.data_as(_u64p)


class SetBWTE:
    """An incrementally built string-set BWT / FM-index on one CUDA device.

    >>> idx = SetBWTE("ACGT"); idx.append_strings(["AC", "G"]); idx.bwt()
    b'CG$A$'
    """

    def __init__(self, alphabet: str = "ACGT", block_suffixes: int | None = None,
                 profile: bool = False):
        self._lib = load_library()
        h = ctypes.c_void_p()
        self._check(self._lib.setbwte_create(alphabet.encode(), ctypes.byref(h)), "create")
        self._h = h
        self._allgather_ref = None
        self.alphabet = alphabet
        if block_suffixes is not None:
            self.set_option("block_suffixes", block_suffixes)
        if profile:
            self.set_option("profile", 1)

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.setbwte_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc, where):
        if rc != 0:
            detail = ""
            if rc == 2 and getattr(self, "_h", None):
                pos, byte = self.last_error()
                detail = "byte %d = %r" % (pos, bytes([byte]))
            raise SetBWTEError(rc, where, detail)

    # -- options -------------------------------------------------------------
    def set_option(self, key: str, value: int):
        self._check(self._lib.setbwte_set_option(self._h, key.encode(), int(value)), "set_option")

    def set_profile(self, mode: int, kernel: str | None = None):
        """0 off, 1 time every launch, 2 time only launches of `kernel`, 3 every
        launch plus a timeline (stats()["timeline"]: [kernel, stream, start ms,
        end ms] per launch, from the append's start)."""
        self._check(self._lib.setbwte_set_profile(self._h, mode,
                                                  kernel.encode() if kernel else None),
                    "set_profile")

    def set_stream(self, stream):
        """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None."""
        ptr = None if stream is None else int(getattr(stream, "cuda_stream", stream))
        self._check(self._lib.setbwte_set_stream(self._h, ptr), "set_stream")

    def set_partition(self, rank: int, world: int, allgather=None):
        """allgather(buf_ptr, bytes_per_rank: list[int], world, stream_ptr) -> None."""
        if allgather is None:
            cb = ALLGATHER_FN()
        else:
            def _cb(buf, bpr, world_, stream, ctx):
                try:
                    allgather(int(buf), [int(bpr[i]) for i in range(world_)], world_,
                              int(stream or 0))
                    return 0
                except Exception:  # surfaced as SETBWTE_E_STATE
                    import traceback
                    traceback.print_exc()
                    return 1
            cb = ALLGATHER_FN(_cb)
        self._allgather_ref = cb
        self._check(self._lib.setbwte_set_partition(self._h, rank, world, cb, None),
                    "set_partition")

    def set_comm(self, nccl_comm: int, rank: int, world: int):
        """In-library NCCL exchange (setbwte_set_comm): nccl_comm is an
        ncclComm_t address (paper_1410_0562_b200.dist.nccl_comm(group)); 0
        detaches."""
        self._check(self._lib.setbwte_set_comm(self._h, ctypes.c_void_p(int(nccl_comm) or None),
                                               int(rank), int(world)), "set_comm")

    def set_allocator(self, alloc=None, free=None):
        """Route the handle's device allocations through alloc(nbytes) -> int
        device pointer (0 = out of memory) and free(ptr).  None, None restores
        cudaMalloc.  See setbwte_set_allocator."""
        if alloc is None and free is None:
            a, f = ALLOC_FN(), FREE_FN()
        else:
            def _a(nbytes, ctx):
                try:
                    return int(alloc(int(nbytes))) or None
                except Exception:  # surfaced as SETBWTE_E_NOMEM
                    return None

            def _f(ptr, ctx):
                free(int(ptr))
            a, f = ALLOC_FN(_a), FREE_FN(_f)
        self._check(self._lib.setbwte_set_allocator(self._h, a, f, None), "set_allocator")
        # earlier callbacks stay referenced: buffers they produced are
        # released through them
        self._alloc_refs = getattr(self, "_alloc_refs", []) + [a, f]

    def use_torch_allocator(self, device=None):
        """Share PyTorch's CUDA caching allocator (memory shows up in
        torch.cuda.memory_allocated and is reused across calls)."""
        import torch
        dev = torch.cuda.current_device() if device is None else device
        self.set_allocator(lambda n: torch.cuda.caching_allocator_alloc(n, device=dev),
                           torch.cuda.caching_allocator_delete)

    # -- append --------------------------------------------------------------
    def append(self, data, offsets):
        """Append strings given as a u8 host array + u64 CSR offsets (m+1)."""
        d, dp = _host_u8(data)
        o, op = _host_u64(offsets)
        self._check(self._lib.setbwte_append(self._h, dp, op, len(o) - 1), "append")

    def append_strings(self, strings):
        bs = [s.encode() if isinstance(s, str) else bytes(s) for s in strings]
        off = np.zeros(len(bs) + 1, dtype=np.uint64)
        if bs:
            off[1:] = np.cumsum([len(b) for b in bs])
        self.append(b"".join(bs), off)

    def append_device(self, data_t, offsets_t, m: int | None = None):
        """Append from torch CUDA tensors (uint8 data, int64/uint64 offsets)."""
        if m is None:
            m = offsets_t.numel() - 1
        self._check(self._lib.setbwte_append_device(self._h, data_t.data_ptr(),
                                                    offsets_t.data_ptr(), m), "append_device")

    def prepend(self, data, offsets):
        """Reverse orientation: add strings BEFORE every indexed string."""
        d, dp = _host_u8(data)
        o, op = _host_u64(offsets)
        self._check(self._lib.setbwte_prepend(self._h, dp, op, len(o) - 1), "prepend")

    def prepend_strings(self, strings):
        bs = [s.encode() if isinstance(s, str) else bytes(s) for s in strings]
        off = np.zeros(len(bs) + 1, dtype=np.uint64)
        if bs:
            off[1:] = np.cumsum([len(b) for b in bs])
        self.prepend(b"".join(bs), off)

    def prepend_device(self, data_t, offsets_t, m: int | None = None):
        if m is None:
            m = offsets_t.numel() - 1
        self._check(self._lib.setbwte_prepend_device(self._h, data_t.data_ptr(),
                                                     offsets_t.data_ptr(), m), "prepend_device")

    def merge(self, other: "SetBWTE"):
        """BWT merge: append the strings of `other` (from its BWT) after ours."""
        self._check(self._lib.setbwte_merge(self._h, other._h), "merge")

    def clear(self):
        self._check(self._lib.setbwte_clear(self._h), "clear")

    # -- queries ---------------------------------------------------------------
    def size(self):
        n, m = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self._lib.setbwte_size(self._h, ctypes.byref(n), ctypes.byref(m)), "size")
        return int(n.value), int(m.value)

    def bwt(self, out=None) -> bytes:
        """The BWT as bytes; or written into `out` (numpy u8 array / pinned torch tensor)."""
        n = ctypes.c_uint64()
        self._check(self._lib.setbwte_bwt(self._h, None, 0, ctypes.byref(n)), "bwt")
        if out is None:
            buf = np.empty(max(int(n.value), 1), dtype=np.uint8)
            self._check(self._lib.setbwte_bwt(self._h, buf.ctypes.data, buf.size,
                                              ctypes.byref(n)), "bwt")
            return buf[: n.value].tobytes()
        ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        cap = out.numel() if hasattr(out, "numel") else out.size
        self._check(self._lib.setbwte_bwt(self._h, ptr, cap, ctypes.byref(n)), "bwt")
        return int(n.value)

    def bwt_device(self, out_t) -> int:
        n = ctypes.c_uint64()
        self._check(self._lib.setbwte_bwt_device(self._h, out_t.data_ptr(), out_t.numel(),
                                                 ctypes.byref(n)), "bwt_device")
        return int(n.value)

    def rank(self, c: str, k: int) -> int:
        out = ctypes.c_uint64()
        self._check(self._lib.setbwte_rank(self._h, ord(c), int(k), ctypes.byref(out)), "rank")
        return int(out.value)

    def rank_batch(self, c_t, k_t, out_t):
        """Device batch: c_t uint8, k_t int64/uint64, out_t int64/uint64 CUDA tensors."""
        self._check(self._lib.setbwte_rank_batch(self._h, c_t.data_ptr(), k_t.data_ptr(),
                                                 c_t.numel(), out_t.data_ptr()), "rank_batch")
        return out_t

    def count(self, patterns):
        """FM-index count of each pattern (list of str/bytes) -> numpy u64 array."""
        bs = [p.encode() if isinstance(p, str) else bytes(p) for p in patterns]
        off = np.zeros(len(bs) + 1, dtype=np.uint64)
        if bs:
            off[1:] = np.cumsum([len(b) for b in bs])
        d, dp = _host_u8(b"".join(bs))
        o, op = _host_u64(off)
        out = np.zeros(max(len(bs), 1), dtype=np.uint64)
        self._check(self._lib.setbwte_count(self._h, dp, op, len(bs), out.ctypes.data_as(_u64p)),
                    "count")
        return out[:len(bs)]

    def count_device(self, pat_t, off_t, out_t):
        self._check(self._lib.setbwte_count_device(self._h, pat_t.data_ptr(), off_t.data_ptr(),
                                                   off_t.numel() - 1, out_t.data_ptr()),
                    "count_device")
        return out_t

    def construct_sa(self, data, offsets):
        """ConstructSA + B_int of one block (not added to the index)."""
        d, dp = _host_u8(data)
        o, op = _host_u64(offsets)
        m = len(o) - 1
        n = int(o[-1]) + m if m else 0
        sa = np.zeros(max(n, 1), dtype=np.uint32)
        bint = np.zeros(max(n, 1), dtype=np.uint8)
        self._check(self._lib.setbwte_construct_sa(self._h, dp, op, m, sa.ctypes.data_as(_u32p),
                                                   bint.ctypes.data_as(_u8p)), "construct_sa")
        return sa[:n], bint[:n].tobytes()

    def compute_ranks(self, data, offsets):
        """ComputeRanks of one block against the current index (index unchanged)."""
        d, dp = _host_u8(data)
        o, op = _host_u64(offsets)
        m = len(o) - 1
        n = int(o[-1]) + m if m else 0
        g = np.zeros(max(n, 1), dtype=np.uint64)
        self._check(self._lib.setbwte_compute_ranks(self._h, dp, op, m, g.ctypes.data_as(_u64p)),
                    "compute_ranks")
        return g[:n]

    def stats(self) -> dict:
        n = ctypes.c_uint64()
        self._check(self._lib.setbwte_stats(self._h, None, 0, ctypes.byref(n)), "stats")
        buf = ctypes.create_string_buffer(int(n.value))
        self._check(self._lib.setbwte_stats(self._h, buf, n.value, ctypes.byref(n)), "stats")
        return json.loads(buf.value.decode())

    def last_error(self):
        pos, byte = ctypes.c_uint64(), ctypes.c_uint8()
        self._lib.setbwte_last_error(self._h, ctypes.byref(pos), ctypes.byref(byte))
        return int(pos.value), int(byte.value)
