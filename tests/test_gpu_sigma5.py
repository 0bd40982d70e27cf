"""sigma = 5 (NEXT-4; SPEC S:31 default alphabet {A,C,G,T,N}, Sec.2
"ordered alphabet c_1 < ... < c_sigma"): the CUDA path with the fifth symbol
against the alphabet-generic CPU oracle (itself pinned for sigma = 5 against
brute force in tests/test_oracle_pins.py), element by element.  Integer work:
bit-exact."""
import numpy as np
import pytest

import oracle
import synth
from tests import brute

pytestmark = pytest.mark.gpu
A5 = "ACGTN"


@pytest.fixture(scope="module")
def SetBWTE():
    from paper_1410_0562_b200 import SetBWTE
    return SetBWTE


def build(SetBWTE, data, offsets, M=None, splits=None, alphabet=A5, **opts):
    idx = SetBWTE(alphabet, block_suffixes=M)
    for k, v in opts.items():
        idx.set_option(k, v)
    m = len(offsets) - 1
    cuts = [0] + list(splits or []) + [m]
    for a, b in zip(cuts[:-1], cuts[1:]):
        o = np.asarray(offsets[a:b + 1], dtype=np.uint64)
        d = data[int(o[0]):int(o[-1])]
        idx.append(d, o - o[0])
    return idx


def test_worked_examples(SetBWTE):
    """Textbook single-string BWTs (m = 1 reduces to the rotation BWT of S$)
    and a two-string set by brute force over the integer text."""
    for s in ["NNNN", "GATNACA", "N", "ANTN", "NACGTN"]:
        idx = SetBWTE(A5)
        idx.append_strings([s])
        assert idx.bwt().decode() == brute.rotation_bwt(s, A5), s
    strings = ["ACN", "N", "", "GNT"]
    idx = SetBWTE(A5)
    idx.append_strings(strings)
    assert idx.bwt().decode() == brute.brute_bwt(strings, A5)


@pytest.mark.parametrize("seed", range(24))
def test_random_sets_vs_oracle(SetBWTE, seed):
    alpha = ["ACGTN", "NA", "TN", "N", "ACN"][seed % 5]
    d, o = synth.random_set(23000 + seed, max_m=64, max_len=60, alphabet=alpha)
    want = oracle.bwt(A5, d, o)
    m = len(o) - 1
    rng = np.random.default_rng(seed)
    splits = sorted(set(rng.integers(0, m + 1, size=3).tolist()))
    idx = build(SetBWTE, d, o, M=int(rng.integers(1, 300)), splits=splits)
    assert idx.bwt() == want


@pytest.mark.parametrize("seed", range(10))
def test_block_sa_and_ranks(SetBWTE, seed):
    d, o = synth.random_set(23100 + seed, max_m=64, max_len=50,
                            alphabet=["ACGTN", "NA"][seed % 2])
    strings = synth.to_strings(d, o)
    idx = SetBWTE(A5)
    sa, bint = idx.construct_sa(d, o)
    want_sa = oracle.block_sa(A5, d, o)
    assert np.array_equal(sa.astype(np.uint64), want_sa)
    assert bint == oracle.block_bint(A5, d, o, want_sa)
    cut = len(strings) // 2
    ed, eo = synth.from_strings(strings[:cut])
    bd, bo = synth.from_strings(strings[cut:])
    idx.append(ed, eo)
    g = idx.compute_ranks(bd, bo)
    assert np.array_equal(g, oracle.compute_ranks(A5, d, o, m_ext=cut))


@pytest.fixture(scope="module")
def c1n():
    d, o = synth.uniform_n(1000, 100, p_n=0.02, seed=1)
    return d, o, oracle.bwt(A5, d, o, threads=None)


@pytest.mark.parametrize("M", [25250, 997, 1 << 20])
def test_c1_with_n(SetBWTE, c1n, M):
    """c1 shape (1000 x 100 bp) with 2 % N, K = 4 and other block sizes."""
    d, o, want = c1n
    assert build(SetBWTE, d, o, M=M).bwt() == want


@pytest.mark.parametrize("opts", [dict(sa_payload=0), dict(g_width=8),
                                  dict(sa_payload=0, g_width=8), dict(sort_lanes=0)])
def test_c1_with_n_forced_paths(SetBWTE, c1n, opts):
    """Without the SA payload (B_int recorded per slot by ComputeRanks, or in
    g's top byte with u64 g), u64 ranks, and the unpipelined order."""
    d, o, want = c1n
    assert build(SetBWTE, d, o, M=25250, splits=[500], **opts).bwt() == want


def test_rank_and_count_every_symbol(SetBWTE, c1n):
    d, o, want = c1n
    idx = build(SetBWTE, d, o, M=25250)
    rng = np.random.default_rng(3)
    for k in list(rng.integers(0, len(want) + 1, size=20)) + [0, len(want)]:
        for c in "$ACGTN":
            assert idx.rank(c, int(k)) == oracle.rank(want, c, int(k)), (c, k)
    strings = synth.to_strings(d, o)
    pats = ["N", "NN", "AN", "NA", "ACGTN", "GNT", "n", "A", ""]
    pats += ["".join(rng.choice(list("ACGTN"), size=int(rng.integers(1, 6)))) for _ in range(100)]
    got = idx.count(pats)
    assert list(got) == list(oracle.count(A5, d, o, pats))
    assert [int(x) for x in got[:6]] == [brute.naive_count(p, strings) for p in pats[:6]]


def test_prepend_with_n(SetBWTE):
    d, o = synth.random_set(23200, max_m=60, max_len=40, alphabet="ACGTN")
    strings = synth.to_strings(d, o)
    cut = len(strings) // 2
    a = synth.from_strings(strings[:cut])
    b = synth.from_strings(strings[cut:])
    idx = SetBWTE(A5, block_suffixes=200)
    idx.append(*b)
    idx.prepend(*a)
    assert idx.bwt() == oracle.bwt(A5, d, o)


def test_scaled_reads_with_n(SetBWTE):
    """200k reads x 100 bp with 1 % N, blocks of 2^22 suffixes: multi-pass
    digit sorts on 3-bit keys, every kernel class."""
    d, o = synth.uniform_n(200_000, 100, p_n=0.01, seed=7)
    want = oracle.bwt(A5, d, o, threads=None)
    assert build(SetBWTE, d, o, M=1 << 22).bwt() == want


def test_genome_sampled_with_n(SetBWTE):
    """Deep LCPs (reads from a 1 Mbp genome at ~10x) with N runs."""
    d, o = synth.genome_sampled(100_000, 100, 1_000_000, seed=5)
    d = d.copy()
    d[::97] = ord("N")
    want = oracle.bwt(A5, d, o, threads=None)
    assert build(SetBWTE, d, o, M=1 << 21).bwt() == want


def test_lowercase_and_invalid(SetBWTE):
    idx = SetBWTE(A5)
    idx.append_strings(["acgtn", "nN"])
    assert idx.bwt() == oracle.bwt(A5, *synth.from_strings(["ACGTN", "NN"]))
    from paper_1410_0562_b200 import SetBWTEError
    with pytest.raises(SetBWTEError) as e:
        idx.append_strings(["ACX"])
    assert e.value.name == "E_INVALID_CHAR"


def test_unsupported_combinations(SetBWTE):
    from paper_1410_0562_b200 import SetBWTEError
    idx = SetBWTE(A5)
    idx.append_strings(["ACN"])
    for key in ("host_tier",):
        with pytest.raises(SetBWTEError) as e:
            idx.set_option(key, 1)
        assert e.value.name == "E_UNSUPPORTED"
    other = SetBWTE(A5)
    other.append_strings(["N"])
    with pytest.raises(SetBWTEError) as e:
        idx.merge(other)
    assert e.value.name == "E_UNSUPPORTED"


@pytest.mark.slow
def test_c2_size_with_n(SetBWTE):
    """c2's shape (1M x 100 bp, M = 2^24, K = 7) with 1 % N: every pass of
    the sort on 3-bit key words at full block size, whole BWT vs the oracle."""
    d, o = synth.uniform_n(1_000_000, 100, p_n=0.01, seed=3)
    want = oracle.bwt(A5, d, o, threads=None)
    idx = build(SetBWTE, d, o, M=1 << 24)
    assert idx.stats()["blocks"] == 7
    assert idx.bwt() == want


def test_large_block_with_n(SetBWTE):
    """A 35 M-suffix block with N ranked into a 25 M-symbol index (blocks of
    >= 2^25 suffixes take the one-CTA digit pass for their ~500-member third
    level)."""
    d, o = synth.uniform_n(600_000, 100, p_n=0.02, seed=4)
    want = oracle.bwt(A5, d, o, threads=None)
    # the second append (350k reads, 35 M suffixes) is one large block
    assert build(SetBWTE, d, o, M=1 << 26, splits=[250_000]).bwt() == want
