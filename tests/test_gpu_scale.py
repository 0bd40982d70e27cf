"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times.  c3, c4 and c5: the WHOLE BWT against the oracle's, through the
oracle-written digests of tests/golden/<cfg>_bwt_digest.json
(tools/make_golden_digests.py: the bucketed one-shot oracle, BLAKE2b-128 of
the full ASCII BWT, per-bucket digests and exact 4 KB windows) -- a byte
compare in all but name.  Also sampled outputs the oracle computes one by one
(the SA position of a suffix, gives B at that position by Eq.(1)) and
properties that hold at any size (B[0..m) = last symbols, m terminators, LF
inversion recovers reads)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
A = "ACGT"


GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _digest_checks(B: bytes, cfg: str):
    """The whole BWT against the oracle's digest, windows and bucket digests."""
    gd = json.load(open(os.path.join(GOLD, "%s_bwt_digest.json" % cfg)))
    assert len(B) == gd["n"]
    mv = memoryview(B)
    for w in gd["windows"]:
        s = w["start"]
        assert bytes(mv[s:s + len(w["bytes"])]) == w["bytes"].encode(), ("window", s)
    bad = [b["bucket"] for b in gd["buckets"]
           if hashlib.blake2b(mv[b["start"]:b["start"] + b["len"]], digest_size=16).hexdigest()
           != b["blake2b_128"]]
    assert not bad, ("buckets differ", bad[:10])
    h = hashlib.blake2b(digest_size=16)
    h.update(mv)
    assert h.hexdigest() == gd["digest"]["hex"]


def _sampled_checks(idx, data, offsets, n_samples, seed):
    from paper_1410_0562_b200 import SetBWTE  # noqa: F401
    m = len(offsets) - 1
    n, mm = idx.size()
    assert mm == m and n == int(offsets[-1]) + m
    B = np.frombuffer(idx.bwt(), dtype=np.uint8)
    # B[0..m) = the last symbol of each string (rows 0..m-1 are $_0..$_{m-1})
    last = data[(offsets[1:] - 1).astype(np.int64)]
    assert np.array_equal(B[:m], last)
    # exactly m terminators; symbol multiset = input multiset
    assert int((B == ord("$")).sum()) == m
    for c in A:
        assert int((B == ord(c)).sum()) == int((data == ord(c)).sum())
    rng = np.random.default_rng(seed)
    # sampled SA positions by the oracle's counting definition
    for _ in range(n_samples):
        j = int(rng.integers(0, m))
        L = int(offsets[j + 1] - offsets[j])
        k = int(rng.integers(0, L + 1))
        r = oracle.suffix_rank(A, data, offsets, j, k, threads=None)
        want = ord("$") if k == 0 else int(data[int(offsets[j]) + k - 1])
        assert int(B[r]) == want, (j, k, r)
    # LF inversion (FM-index backward steps through setbwte_rank) recovers reads
    C = {}
    acc = m
    for c in A:
        C[c] = acc
        acc += int((B == ord(c)).sum())
    for j in rng.integers(0, m, size=3):
        i = int(j)
        out = []
        while B[i] != ord("$"):
            c = chr(B[i])
            out.append(c)
            i = C[c] + idx.rank(c, i)
        s = "".join(reversed(out))
        assert s == bytes(data[int(offsets[j]):int(offsets[j + 1])]).decode()


@pytest.mark.slow
def test_c3_full_sampled():
    """configs[2]: 20M x 100 bp, M = 2^27 (16 blocks)."""
    from paper_1410_0562_b200 import SetBWTE
    d, o = synth.uniform(20_000_000, 100, seed=1)
    idx = SetBWTE(A, block_suffixes=1 << 27)
    idx.append(d, o)
    assert idx.stats()["blocks"] == 16
    _digest_checks(idx.bwt(), "c3")
    _sampled_checks(idx, d, o, n_samples=4, seed=3)


@pytest.mark.slow
def test_c4_scaled_sampled():
    """configs[3]-shaped: long reads of U[1000, 10000] bp (100k reads, 550 Mbp),
    M = 2^28; arbitrary-length suffix keys."""
    from paper_1410_0562_b200 import SetBWTE
    d, o = synth.uniform_var(100_000, 1000, 10000, seed=1)
    idx = SetBWTE(A, block_suffixes=1 << 28)
    idx.append(d, o)
    _sampled_checks(idx, d, o, n_samples=4, seed=4)


def test_genome_sampled_deep_lcp():
    """Reads sampled from a 4 Mbp genome at ~25x coverage: deep LCPs, many
    key words per suffix; whole BWT vs the oracle."""
    from paper_1410_0562_b200 import SetBWTE
    d, o = synth.genome_sampled(1_000_000, 100, 4_000_000, seed=2)
    want = oracle.bwt(A, d, o, threads=None)
    idx = SetBWTE(A, block_suffixes=1 << 24)
    idx.append(d, o)
    assert idx.bwt() == want


@pytest.mark.slow
def test_c4_full_sampled():
    """configs[3] at full size: 1M reads of U[1000, 10000] bp (~5.5 Gbp),
    M = 2^30, u64 ranks -- the launch configuration of bench.py --workload c4."""
    from paper_1410_0562_b200 import SetBWTE
    d, o = synth.uniform_var(1_000_000, 1000, 10000, seed=1)
    idx = SetBWTE(A, block_suffixes=1 << 30)
    idx.append(d, o)
    assert idx.stats()["blocks"] >= 5
    _digest_checks(idx.bwt(), "c4")
    _sampled_checks(idx, d, o, n_samples=2, seed=5)


@pytest.mark.slow
def test_c5_full_sampled():
    """configs[4] at full size: 10M reads appended into a 50M-read index whose
    B_ext is host-tiered (pinned host memory), M = 2^27 -- as bench.py
    --workload c5 runs it."""
    from paper_1410_0562_b200 import SetBWTE
    bd, bo = synth.uniform(50_000_000, 100, seed=1)
    ad, ao = synth.uniform(10_000_000, 100, seed=2)
    idx = SetBWTE(A, block_suffixes=1 << 27)
    idx.append(bd, bo)
    idx.set_option("host_tier", 1)
    idx.append(ad, ao)
    assert idx.stats()["host_tier"]
    d = np.concatenate([bd, ad])
    o = np.concatenate([np.asarray(bo, dtype=np.uint64),
                        np.asarray(ao[1:], dtype=np.uint64) + np.uint64(bo[-1])])
    del bd, ad
    _digest_checks(idx.bwt(), "c5")
    _sampled_checks(idx, d, o, n_samples=2, seed=6)
