"""Host logic of bench.py (no GPU): the oracle's bounded samples and the
stage map."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_sample_reads_bounds():
    o = np.arange(0, 101 * 100, 100, dtype=np.uint64)          # 100 reads of 100 bases
    assert bench.sample_reads(o, 1000, 1000) == 10             # bases bound
    assert bench.sample_reads(o, 5, 10 ** 9) == 5               # reads bound
    assert bench.sample_reads(o, 1000, 10 ** 9) == 100          # whole workload
    assert bench.sample_reads(o, 1000, 50) == 1                 # at least one read
    o2 = np.array([0, 1000, 5000, 6000], dtype=np.uint64)
    assert bench.sample_reads(o2, 10, 5500) == 2
    assert bench.sample_reads(o2, 10, 5000) == 2
    assert bench.sample_reads(o2, 10, 4999) == 1


def test_default_samples_of_the_configs():
    """c2 / c3: the oracle sample is 1M reads = 100 Mbases (c2 whole, so its
    bench parity is a full byte compare); c4: bounded by bases, not reads."""
    o = np.arange(1_000_001, dtype=np.uint64) * 100            # c2's layout (c3's prefix)
    assert bench.sample_reads(o, 1_000_000, 100_000_000) == 1_000_000
    rng = np.random.default_rng(0)
    lens = rng.integers(1000, 10001, size=50_000)
    o = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    k = bench.sample_reads(o, 1_000_000, 100_000_000)
    assert o[k] <= 100_000_000 < o[k + 1]


def test_stage_map():
    """Every stage of Table 2's taxonomy has kernels mapped to it."""
    assert set(bench.STAGE_OF.values()) == {"pack", "sort", "rank", "gather", "insert"}
    for k in ("pack", "digit_scatter", "compute_ranks", "gather", "insert"):
        assert k in bench.STAGE_OF
