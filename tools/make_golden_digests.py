"""Write tests/golden/<cfg>_bwt_digest.json for the full-size configs c3, c4, c5.

Calls ONLY ``oracle/`` (the bucketed one-shot BWT, Eq.(1) P:33-35 on T of
P:36-37) and ``synth/`` (the seeded inputs).  Nothing here touches the CUDA
path.  For each config it records:

* n, m and the symbol multiset of the BWT;
* a 128-bit streaming digest of the whole ASCII BWT (BLAKE2b, digest_size=16);
* the digest, start and length of every bucket (suffixes grouped by their
  first 3 symbols, $ first) so a mismatch can be located;
* ``WINDOWS`` exact windows of ``WLEN`` bytes at seeded positions, plus the
  first and the last window.

Usage: python tools/make_golden_digests.py c3 [c4 c5] [--threads T]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

WINDOWS = 64
WLEN = 4096
A = "ACGT"


def inputs(cfg):
    """The exact inputs bench.py / tests/test_gpu_scale.py feed the GPU path."""
    if cfg == "c3":
        return synth.uniform(20_000_000, 100, seed=1), "synth.uniform(20_000_000, 100, seed=1)"
    if cfg == "c4":
        return (synth.uniform_var(1_000_000, 1000, 10000, seed=1),
                "synth.uniform_var(1_000_000, 1000, 10000, seed=1)")
    if cfg == "c5":
        bd, bo = synth.uniform(50_000_000, 100, seed=1)
        ad, ao = synth.uniform(10_000_000, 100, seed=2)
        d = np.concatenate([bd, ad])
        del bd, ad
        o = np.concatenate([np.asarray(bo, np.uint64),
                            np.asarray(ao[1:], np.uint64) + np.uint64(bo[-1])])
        return (d, o), ("synth.uniform(50_000_000, 100, seed=1) then "
                        "synth.uniform(10_000_000, 100, seed=2), one string set in that order")
    raise ValueError(cfg)


def window_starts(n, seed=12345):
    rng = np.random.default_rng(seed)
    hi = max(n - WLEN, 0)
    starts = set(int(x) for x in rng.integers(0, hi + 1, size=WINDOWS))
    starts.update({0, hi})
    return sorted(starts)


def digest(cfg, threads):
    (d, o), recipe = inputs(cfg)
    m = len(o) - 1
    n = int(o[-1]) + m
    starts = window_starts(n)
    wins = {s: bytearray() for s in starts}
    h = hashlib.blake2b(digest_size=16)
    counts = {c: 0 for c in "$" + A}
    buckets = []
    pos = [0]

    def sink(chunk, bucket):
        p0 = pos[0]
        p1 = p0 + len(chunk)
        h.update(chunk)
        arr = np.frombuffer(chunk, np.uint8)
        for c in counts:
            counts[c] += int(np.count_nonzero(arr == ord(c)))
        buckets.append({"bucket": bucket, "start": p0, "len": len(chunk),
                        "blake2b_128": hashlib.blake2b(chunk, digest_size=16).hexdigest()})
        for s in starts:
            e = s + WLEN
            if e > p0 and s < p1:
                a, b = max(s, p0), min(e, p1)
                wins[s] += chunk[a - p0:b - p0]
        pos[0] = p1

    t0 = time.time()
    got = oracle.bwt_bucketed(A, d, o, sink, h=3, batch_cap=1 << 29, threads=threads)
    dt = time.time() - t0
    assert got == n == pos[0]
    return {
        "config": cfg,
        "inputs": recipe,
        "alphabet": A,
        "definition": "one-shot BWT of the string set, Eq.(1) P:33-35 on T of P:36-37, "
                      "every $_j written '$' (DESIGN.md R5)",
        "written_by": "tools/make_golden_digests.py (oracle.bwt_bucketed, h=3)",
        "n": n,
        "m": m,
        "symbol_counts": counts,
        "digest": {"algo": "blake2b", "digest_size": 16, "hex": h.hexdigest()},
        "buckets_h": 3,
        "buckets": buckets,
        "window_len": WLEN,
        "windows": [{"start": s, "bytes": bytes(wins[s]).decode()} for s in starts],
        "oracle_seconds": round(dt, 1),
        "oracle_threads": threads,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    for cfg in a.configs:
        r = digest(cfg, a.threads)
        path = os.path.join(ROOT, "tests", "golden", "%s_bwt_digest.json" % cfg)
        with open(path, "w") as f:
            json.dump(r, f, indent=0)
        print(cfg, r["n"], r["digest"]["hex"], "%.1fs" % r["oracle_seconds"], flush=True)


if __name__ == "__main__":
    main()
