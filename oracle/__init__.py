"""CPU ORACLE for set-bwte (arXiv 1410.0562) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_1410_0562_b200``) never imports it, and it imports nothing from the
product path.  The arithmetic lives in ``oracle.cpp`` (plain C++, library sort
as the only primitive); this module is ctypes marshalling plus the build.

Functions and the passage each follows (P:<line> = /root/reference/PAPER.md):

* ``bwt``           -- Eq.(1) P:33-35 on T = S_0$_0...S_{m-1}$_{m-1}
* ``block_sa``      -- ConstructSA, Alg.1 P:60 (suffixes of one block)
* ``block_bint``    -- B(S_jk, SA_int), Alg.1
* ``compute_ranks`` -- g by definition: # external suffixes smaller
* ``rank``          -- Eq.(2), literal scan
* ``insert``        -- Insert, Alg.1 P:72-73 / Sec.5, flat list insertion
* ``suffix_rank``   -- SA position of one suffix by counting (definition)
* ``count``         -- substring occurrences by literal comparison (what the
                       FM-index count answers)
* ``bwt_bucketed``  -- ``bwt`` in bucketed low-memory mode: suffixes
                       partitioned by their first h symbols ($ first), each
                       bucket sorted with the same comparator and emitted in
                       key order, streamed to a callback (configs c3-c5)

Pins for each are in ``tests/test_oracle_pins.py``; see DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_EMIT = ctypes.CFUNCTYPE(None, _u8p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile oracle.cpp into liboracle.so (g++, OpenMP for the library sort)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-shared", "-fPIC",
                               _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_bwt.argtypes = [ctypes.c_char_p, _u8p, _u64p, ctypes.c_uint64, _u8p,
                                   ctypes.c_int, _u64p]
        lib.oracle_block_sa.argtypes = [ctypes.c_char_p, _u8p, _u64p, ctypes.c_uint64, _u64p,
                                        ctypes.c_int, _u64p]
        lib.oracle_block_bint.argtypes = [ctypes.c_char_p, _u8p, _u64p, ctypes.c_uint64, _u64p,
                                          _u8p, _u64p]
        lib.oracle_compute_ranks.argtypes = [ctypes.c_char_p, _u8p, _u64p, ctypes.c_uint64,
                                             ctypes.c_uint64, _u64p, ctypes.c_int, _u64p]
        lib.oracle_rank.argtypes = [_u8p, ctypes.c_uint64, ctypes.c_uint8, ctypes.c_uint64]
        lib.oracle_rank.restype = ctypes.c_uint64
        lib.oracle_insert.argtypes = [_u8p, ctypes.c_uint64, _u8p, _u64p, ctypes.c_uint64, _u8p]
        lib.oracle_count.argtypes = [ctypes.c_char_p, _u8p, _u64p, ctypes.c_uint64, _u8p, _u64p,
                                     ctypes.c_uint64, _u64p, ctypes.c_int]
        lib.oracle_suffix_rank.argtypes = [ctypes.c_char_p, _u8p, _u64p, ctypes.c_uint64,
                                           ctypes.c_uint64, ctypes.c_uint64, _u64p, ctypes.c_int,
                                           _u64p]
        lib.oracle_bwt_bucketed.argtypes = [ctypes.c_char_p, _u8p, _u64p, ctypes.c_uint64,
                                            ctypes.c_int, ctypes.c_uint64, _EMIT,
                                            ctypes.c_void_p, ctypes.c_int, _u64p]
        _lib = lib
    return _lib


def _u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, a.ctypes.data_as(_u8p)


def _u64(a):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    return a, a.ctypes.data_as(_u64p)


def _check(rc, bad):
    if rc == -2:
        raise OracleError("invalid character at byte %d" % bad.value)
    if rc != 0:
        raise OracleError("oracle error %d" % rc)


def _threads(threads):
    if threads is None:
        return os.cpu_count() or 1
    return int(threads)


def bwt(alphabet: str, data, offsets, threads: int | None = 1) -> bytes:
    """One-shot string-set BWT (Eq.(1)), terminators written as '$'."""
    data, dp = _u8(data)
    offsets, op = _u64(offsets)
    m = len(offsets) - 1
    n = int(offsets[-1]) + m
    out = np.zeros(max(n, 1), dtype=np.uint8)
    bad = ctypes.c_uint64(0)
    rc = _load().oracle_bwt(alphabet.encode(), dp, op, m, out.ctypes.data_as(_u8p),
                            _threads(threads), ctypes.byref(bad))
    _check(rc, bad)
    return out[:n].tobytes()


def block_sa(alphabet: str, data, offsets, threads: int | None = 1) -> np.ndarray:
    """SA_int of one block as string-major slot ids (u64)."""
    data, dp = _u8(data)
    offsets, op = _u64(offsets)
    m = len(offsets) - 1
    n = int(offsets[-1]) + m
    out = np.zeros(max(n, 1), dtype=np.uint64)
    bad = ctypes.c_uint64(0)
    rc = _load().oracle_block_sa(alphabet.encode(), dp, op, m, out.ctypes.data_as(_u64p),
                                 _threads(threads), ctypes.byref(bad))
    _check(rc, bad)
    return out[:n]


def block_bint(alphabet: str, data, offsets, sa) -> bytes:
    data, dp = _u8(data)
    offsets, op = _u64(offsets)
    sa, sp = _u64(sa)
    m = len(offsets) - 1
    n = int(offsets[-1]) + m
    out = np.zeros(max(n, 1), dtype=np.uint8)
    bad = ctypes.c_uint64(0)
    rc = _load().oracle_block_bint(alphabet.encode(), dp, op, m, sp, out.ctypes.data_as(_u8p),
                                   ctypes.byref(bad))
    _check(rc, bad)
    return out[:n].tobytes()


def compute_ranks(alphabet: str, data, offsets, m_ext: int, threads: int | None = 1) -> np.ndarray:
    """g for the block made of strings m_ext.. of the set, against strings 0..m_ext-1."""
    data, dp = _u8(data)
    offsets, op = _u64(offsets)
    m = len(offsets) - 1
    m_blk = m - m_ext
    n_blk = int(offsets[m] - offsets[m_ext]) + m_blk
    out = np.zeros(max(n_blk, 1), dtype=np.uint64)
    bad = ctypes.c_uint64(0)
    rc = _load().oracle_compute_ranks(alphabet.encode(), dp, op, m_ext, m_blk,
                                      out.ctypes.data_as(_u64p), _threads(threads),
                                      ctypes.byref(bad))
    _check(rc, bad)
    return out[:n_blk]


def rank(B: bytes, c: str, k: int) -> int:
    """Eq.(2): occurrences of byte c in B[0:k]."""
    arr, p = _u8(np.frombuffer(B, dtype=np.uint8) if len(B) else np.zeros(1, np.uint8))
    return int(_load().oracle_rank(p, len(B), ord(c), k))


def insert(b_ext: bytes, b_int: bytes, g_sa) -> bytes:
    g_sa, gp = _u64(g_sa)
    n = len(b_ext) + len(b_int)
    e, ep = _u8(np.frombuffer(b_ext, np.uint8) if b_ext else np.zeros(1, np.uint8))
    i, ip = _u8(np.frombuffer(b_int, np.uint8) if b_int else np.zeros(1, np.uint8))
    out = np.zeros(max(n, 1), dtype=np.uint8)
    rc = _load().oracle_insert(ep, len(b_ext), ip, gp, len(b_int), out.ctypes.data_as(_u8p))
    if rc:
        raise OracleError("insert position out of range")
    return out[:n].tobytes()


def suffix_rank(alphabet: str, data, offsets, j: int, k: int, threads: int | None = None) -> int:
    data, dp = _u8(data)
    offsets, op = _u64(offsets)
    m = len(offsets) - 1
    out = ctypes.c_uint64(0)
    bad = ctypes.c_uint64(0)
    rc = _load().oracle_suffix_rank(alphabet.encode(), dp, op, m, j, k, ctypes.byref(out),
                                    _threads(threads), ctypes.byref(bad))
    _check(rc, bad)
    return int(out.value)


def count(alphabet: str, data, offsets, patterns, threads: int | None = 1) -> np.ndarray:
    """Occurrences of each pattern (list of str/bytes) in the strings."""
    bs = [p.encode() if isinstance(p, str) else bytes(p) for p in patterns]
    poff = np.zeros(len(bs) + 1, dtype=np.uint64)
    if bs:
        poff[1:] = np.cumsum([len(b) for b in bs])
    data, dp = _u8(data)
    offsets, op = _u64(offsets)
    pat, pp = _u8(np.frombuffer(b"".join(bs), np.uint8) if sum(map(len, bs)) else np.zeros(1, np.uint8))
    poff, pop = _u64(poff)
    out = np.zeros(max(len(bs), 1), dtype=np.uint64)
    rc = _load().oracle_count(alphabet.encode(), dp, op, len(offsets) - 1, pp, pop, len(bs),
                              out.ctypes.data_as(_u64p), _threads(threads))
    if rc:
        raise OracleError("oracle error %d" % rc)
    return out[:len(bs)]


def bwt_bucketed(alphabet: str, data, offsets, sink, h: int = 3,
                 batch_cap: int = 1 << 29, threads: int | None = None) -> int:
    """The one-shot BWT (Eq.(1)) in bucketed mode: ``sink(chunk: bytes, bucket: int)``
    receives the BWT bucket by bucket, in order (their concatenation is
    ``bwt(...)``).  Memory: the text codes plus ~9 B x ``batch_cap``.
    Returns n."""
    data, dp = _u8(data)
    offsets, op = _u64(offsets)
    m = len(offsets) - 1
    err = []

    def _emit(ptr, ln, bucket, _ctx):
        try:
            sink(ctypes.string_at(ptr, ln), int(bucket))
        except BaseException as e:  # pragma: no cover - surfaced below
            err.append(e)

    cb = _EMIT(_emit)
    bad = ctypes.c_uint64(0)
    rc = _load().oracle_bwt_bucketed(alphabet.encode(), dp, op, m, int(h), int(batch_cap), cb,
                                     None, _threads(threads), ctypes.byref(bad))
    if err:
        raise err[0]
    _check(rc, bad)
    return int(offsets[-1]) + m
