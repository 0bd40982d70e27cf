"""Seeded synthetic read sets -- shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws reads.  Both
the tests and bench.py feed the same (data, offsets) pair to the CUDA path and
to the oracle.  Layout: ``data`` is a u8 ASCII array of all bases concatenated
(no terminators), ``offsets`` a u64 CSR array of m+1 entries, string j =
data[offsets[j]:offsets[j+1]].

Recipes (shapes follow BASELINE.json configs):

* ``uniform(m, L)``        -- m reads of L bases, i.i.d. uniform over ACGT
                              (c1, c2, c3, c5: 100 bp short reads).
* ``uniform_var(m, lo, hi)`` -- lengths i.i.d. uniform integers in [lo, hi]
                              (c4 long reads, 1-10 kbp; "reads of
                              arbitrary length").
* ``genome_sampled(m, L, G)`` -- reads sampled from one random genome of G
                              bases: uniform start, 50 % reverse complement,
                              0.5 % substitutions -- overlapping reads give
                              deep LCPs like real sequencing sets.
* ``uniform_n(m, L, p_n)`` -- as ``uniform`` over ACGT, each base replaced by N
                              with probability p_n (sigma = 5).
* ``random_set(...)``      -- small random sets for property tests (m <= 64,
                              |P| <= 50, empty and duplicate strings).
* ``adversarial(kind)``    -- all-A, (AC)^k, many empty strings.
"""
from __future__ import annotations

import numpy as np

ACGT = np.frombuffer(b"ACGT", dtype=np.uint8)


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def from_strings(strings):
    """(data, offsets) from a list of str/bytes."""
    bs = [s.encode() if isinstance(s, str) else bytes(s) for s in strings]
    offsets = np.zeros(len(bs) + 1, dtype=np.uint64)
    if bs:
        offsets[1:] = np.cumsum([len(b) for b in bs], dtype=np.uint64)
    data = np.frombuffer(b"".join(bs), dtype=np.uint8).copy() if bs else np.zeros(0, np.uint8)
    return data, offsets


def to_strings(data, offsets):
    d = bytes(np.asarray(data, dtype=np.uint8))
    o = [int(x) for x in offsets]
    return [d[o[j]:o[j + 1]].decode() for j in range(len(o) - 1)]


def uniform(m: int, L: int, seed: int = 1):
    rng = _rng(seed)
    data = ACGT[rng.integers(0, 4, size=m * L, dtype=np.uint8)]
    offsets = np.arange(m + 1, dtype=np.uint64) * np.uint64(L)
    return data, offsets


def uniform_n(m: int, L: int, p_n: float = 0.01, seed: int = 1):
    rng = _rng(seed)
    data = ACGT[rng.integers(0, 4, size=m * L, dtype=np.uint8)]
    data[rng.random(m * L) < p_n] = ord("N")
    offsets = np.arange(m + 1, dtype=np.uint64) * np.uint64(L)
    return data, offsets


def uniform_var(m: int, lo: int, hi: int, seed: int = 1):
    rng = _rng(seed)
    lens = rng.integers(lo, hi + 1, size=m, dtype=np.int64)
    offsets = np.zeros(m + 1, dtype=np.uint64)
    offsets[1:] = np.cumsum(lens, dtype=np.uint64)
    data = ACGT[rng.integers(0, 4, size=int(offsets[-1]), dtype=np.uint8)]
    return data, offsets


def genome_sampled(m: int, L: int, G: int, seed: int = 1, sub_rate: float = 0.005):
    rng = _rng(seed)
    genome = rng.integers(0, 4, size=G, dtype=np.uint8)
    starts = rng.integers(0, G - L + 1, size=m, dtype=np.int64)
    idx = starts[:, None] + np.arange(L, dtype=np.int64)[None, :]
    reads = genome[idx]
    rc = rng.random(m) < 0.5
    reads[rc] = 3 - reads[rc][:, ::-1]          # reverse complement (A<->T, C<->G)
    subs = rng.random(reads.shape) < sub_rate
    reads[subs] = (reads[subs] + rng.integers(1, 4, size=int(subs.sum()), dtype=np.uint8)) & 3
    data = ACGT[reads.reshape(-1)]
    offsets = np.arange(m + 1, dtype=np.uint64) * np.uint64(L)
    return data, offsets


def random_set(seed: int, max_m: int = 64, max_len: int = 50, alphabet: str = "ACGT",
               p_empty: float = 0.05, p_dup: float = 0.1):
    """A small random string set drawn over ``alphabet`` (upper case)."""
    rng = _rng(seed)
    m = int(rng.integers(1, max_m + 1))
    alpha = np.frombuffer(alphabet.encode(), dtype=np.uint8)
    strings = []
    for _ in range(m):
        r = rng.random()
        if r < p_empty:
            strings.append(b"")
        elif r < p_empty + p_dup and strings:
            strings.append(strings[int(rng.integers(0, len(strings)))])
        else:
            L = int(rng.integers(0, max_len + 1))
            strings.append(alpha[rng.integers(0, len(alpha), size=L)].tobytes())
    return from_strings(strings)


def adversarial(kind: str, m: int = 100, L: int = 100):
    if kind == "all_A":
        return from_strings([b"A" * L] * m)
    if kind == "AC_repeat":
        return from_strings([b"AC" * (L // 2)] * m)
    if kind == "many_empty":
        return from_strings([b"" if j % 3 else b"ACG" for j in range(m)])
    if kind == "staircase":
        return from_strings([b"A" * j for j in range(m)])
    raise ValueError(kind)
