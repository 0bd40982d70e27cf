"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle,
element by element, on seeded synthetic inputs.  Integer work => bit-exact."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests import brute

pytestmark = pytest.mark.gpu

A = "ACGT"
GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))
TWO = json.load(open(os.path.join(GOLD, "two_block_example.json")))


@pytest.fixture(scope="module")
def SetBWTE():
    from paper_1410_0562_b200 import SetBWTE
    return SetBWTE


def build(SetBWTE, data, offsets, M=None, splits=None, alphabet=A):
    idx = SetBWTE(alphabet, block_suffixes=M)
    m = len(offsets) - 1
    cuts = [0] + list(splits or []) + [m]
    for a, b in zip(cuts[:-1], cuts[1:]):
        o = np.asarray(offsets[a:b + 1], dtype=np.uint64)
        d = data[int(o[0]):int(o[-1])]
        idx.append(d, o - o[0])
    return idx


# --- worked examples ----------------------------------------------------------

def test_golden_bwt(SetBWTE):
    for case in SPEC["bwt"]:
        idx = SetBWTE(A)
        for blk in case.get("blocks", [case["strings"]]):
            idx.append_strings(blk)
        assert idx.bwt().decode() == case["bwt"], case["cite"]


def test_golden_two_block(SetBWTE):
    idx = SetBWTE(A)
    for blk in TWO["blocks"]:
        d, o = synth.from_strings(blk["strings"])
        sa, bint = idx.construct_sa(d, o)
        assert list(sa) == blk["sa_slots"]
        assert bint.decode() == blk["bint"]
        assert list(idx.compute_ranks(d, o)) == blk["g"]
        idx.append(d, o)
        assert idx.bwt().decode() == blk["b_ext_after"]
    B = idx.bwt()
    assert B.decode() == TWO["one_shot_bwt"]


def test_golden_stage_examples(SetBWTE):
    idx = SetBWTE(A)
    for case in SPEC["block_sa"]:
        d, o = synth.from_strings(case["strings"])
        sa, _ = idx.construct_sa(d, o)
        slot = {p: s for s, p in enumerate(brute.slot_jk(case["strings"]))}
        assert list(sa) == [slot[tuple(p)] for p in case["sa_jk"]], case["cite"]
    for case in SPEC["compute_ranks"]:
        idx2 = SetBWTE(A)
        if case["ext"]:
            idx2.append_strings(case["ext"])
        d, o = synth.from_strings(case["block"])
        assert list(idx2.compute_ranks(d, o)) == case["g"], case["cite"]
    for case in SPEC["rank"]:
        idx3 = SetBWTE(A)
        # B of the worked example is the BWT of a set; rebuild it from its strings
        strings = {"C$A": ["AC"], "CG$A$": ["AC", "G"]}[case["B"]]
        idx3.append_strings(strings)
        assert idx3.bwt().decode() == case["B"]
        assert idx3.rank(case["c"], case["k"]) == case["rank"], case["cite"]


# --- random small sets: every block size, every append split ------------------

@pytest.mark.parametrize("seed", range(120))
def test_random_sets_vs_oracle(SetBWTE, seed):
    alpha = ["ACGT", "AC", "A", "ACG", "GT"][seed % 5]
    d, o = synth.random_set(seed, max_m=64, max_len=50, alphabet=alpha)
    want = oracle.bwt(A, d, o)
    n = len(want)
    m = len(o) - 1
    for M in (1, 40, 400, n + 1):
        assert build(SetBWTE, d, o, M=M).bwt() == want, ("M", M)
    rng = np.random.default_rng(seed)
    splits = sorted(set(rng.integers(0, m + 1, size=3).tolist()))
    assert build(SetBWTE, d, o, M=int(rng.integers(1, 200)), splits=splits).bwt() == want


@pytest.mark.parametrize("seed", range(20))
def test_random_block_sa_and_ranks(SetBWTE, seed):
    d, o = synth.random_set(100 + seed, max_m=64, max_len=50,
                            alphabet=["ACGT", "AC"][seed % 2])
    strings = synth.to_strings(d, o)
    idx = SetBWTE(A)
    sa, bint = idx.construct_sa(d, o)
    want_sa = oracle.block_sa(A, d, o)
    assert np.array_equal(sa.astype(np.uint64), want_sa)
    assert bint == oracle.block_bint(A, d, o, want_sa)
    cut = len(strings) // 2
    ed, eo = synth.from_strings(strings[:cut])
    bd, bo = synth.from_strings(strings[cut:])
    idx.append(ed, eo)
    g = idx.compute_ranks(bd, bo)
    assert np.array_equal(g, oracle.compute_ranks(A, d, o, m_ext=cut))


# --- c1 (BASELINE configs[0]): 1000 x 100 bp, K = 4, and sweeps ----------------

@pytest.fixture(scope="module")
def c1():
    d, o = synth.uniform(1000, 100, seed=1)
    return d, o, oracle.bwt(A, d, o, threads=None)


@pytest.mark.parametrize("M", [25250, 101000, 50500, 101])
def test_c1_block_sizes(SetBWTE, c1, M):
    d, o, want = c1
    idx = build(SetBWTE, d, o, M=M)
    assert idx.bwt() == want
    assert idx.stats()["blocks"] == -(-101000 // M)


@pytest.mark.parametrize("seed", range(4))
def test_c1_random_append_splits(SetBWTE, c1, seed):
    d, o, want = c1
    rng = np.random.default_rng(seed)
    splits = sorted(set(rng.integers(1, 1000, size=5).tolist()))
    assert build(SetBWTE, d, o, M=int(rng.integers(2000, 40000)), splits=splits).bwt() == want


def test_c1_rank_every_symbol(SetBWTE, c1):
    d, o, want = c1
    idx = build(SetBWTE, d, o, M=25250)
    n = len(want)
    arr = np.frombuffer(want, dtype=np.uint8)
    ks = [0, 1, 63, 64, 65, 4095, 65535, 65536, 65537, n - 1, n] + \
        list(np.random.default_rng(3).integers(0, n + 1, size=40))
    for c in "$ACGT":
        cum = np.concatenate([[0], np.cumsum(arr == ord(c))])
        for k in ks:
            assert idx.rank(c, int(k)) == int(cum[k]), (c, k)
    # batched on the device
    import torch
    cq = torch.tensor([ord(c) for c in "$ACGT" for _ in ks], dtype=torch.uint8, device="cuda")
    kq = torch.tensor([int(k) for _ in "$ACGT" for k in ks], dtype=torch.int64, device="cuda")
    out = torch.empty_like(kq)
    idx.rank_batch(cq, kq, out)
    ref = [oracle.rank(want, c, int(k)) for c in "$ACGT" for k in ks]
    assert out.cpu().tolist() == ref


# --- sorts that exercise the digit passes and deep LCPs ------------------------

@pytest.mark.parametrize("kind", ["uniform", "genome", "all_A", "AC_repeat", "staircase",
                                  "many_empty", "long"])
def test_block_sa_structured(SetBWTE, kind):
    if kind == "uniform":
        d, o = synth.uniform(3000, 100, seed=5)
    elif kind == "genome":
        d, o = synth.genome_sampled(4000, 100, 20000, seed=5)   # ~20x coverage: deep LCPs
    elif kind == "long":
        d, o = synth.uniform_var(30, 1000, 10000, seed=5)
    else:
        d, o = synth.adversarial(kind, m=150, L=100)
    idx = SetBWTE(A)
    sa, bint = idx.construct_sa(d, o)
    want = oracle.block_sa(A, d, o, threads=None)
    assert np.array_equal(sa.astype(np.uint64), want)
    assert bint == oracle.block_bint(A, d, o, want)


@pytest.mark.parametrize("kind", ["genome", "all_A", "long", "mixed_empty"])
def test_build_structured(SetBWTE, kind):
    if kind == "genome":
        d, o = synth.genome_sampled(5000, 100, 30000, seed=9)
        M = 100000
    elif kind == "all_A":
        d, o = synth.adversarial("all_A", m=400, L=100)
        M = 10000
    elif kind == "long":
        d, o = synth.uniform_var(60, 1000, 10000, seed=9)
        M = 50000
    else:
        d, o = synth.adversarial("many_empty", m=3000)
        M = 777
    want = oracle.bwt(A, d, o, threads=None)
    assert build(SetBWTE, d, o, M=M).bwt() == want


# --- edge cases ----------------------------------------------------------------

def test_edge_cases(SetBWTE):
    from paper_1410_0562_b200 import SetBWTEError
    idx = SetBWTE(A)
    assert idx.size() == (0, 0) and idx.bwt() == b""
    assert idx.rank("A", 0) == 0
    with pytest.raises(SetBWTEError) as e:
        idx.rank("A", 1)
    assert e.value.name == "E_OUT_OF_RANGE"
    idx.append_strings([""])
    assert idx.bwt() == b"$"
    idx.append_strings([])                      # no-op
    assert idx.size() == (1, 1)
    # invalid character: error with position, index unchanged
    with pytest.raises(SetBWTEError) as e:
        idx.append_strings(["ACGT", "ACXGT"])
    assert e.value.name == "E_INVALID_CHAR"
    assert idx.last_error() == (6, ord("X"))
    assert idx.bwt() == b"$"
    # lowercase accepted (reading R10)
    idx.append_strings(["acgt"])
    assert idx.bwt() == oracle.bwt(A, *synth.from_strings(["", "ACGT"]))
    with pytest.raises(SetBWTEError):
        idx.rank("N", 1)
    # bad offsets
    with pytest.raises(SetBWTEError) as e:
        idx.append(np.frombuffer(b"ACGT", np.uint8), np.array([0, 3, 2, 4], np.uint64))
    assert e.value.name == "E_INVALID_ARG"
    # clear
    idx.clear()
    assert idx.size() == (0, 0)
    idx.append_strings(["AC", "G"])
    assert idx.bwt() == b"CG$A$"


def test_small_alphabets(SetBWTE):
    for alpha in ["AC", "A", "GT", "ACG"]:
        d, o = synth.random_set(77, max_m=40, max_len=40, alphabet=alpha)
        idx = SetBWTE(alpha, block_suffixes=200)
        idx.append(d, o)
        # oracle in the same alphabet
        assert idx.bwt() == oracle.bwt(alpha, d, o)


def test_append_device_matches_host(SetBWTE):
    import torch
    d, o = synth.uniform(5000, 100, seed=11)
    a = SetBWTE(A, block_suffixes=1 << 17)
    a.append(d, o)
    b = SetBWTE(A, block_suffixes=1 << 17)
    b.append_device(torch.from_numpy(d).cuda(), torch.from_numpy(o.astype(np.int64)).cuda())
    assert a.bwt() == b.bwt()
    out = torch.empty(a.size()[0], dtype=torch.uint8, device="cuda")
    a.bwt_device(out)
    assert bytes(out.cpu().numpy()) == a.bwt()


# --- scale: c2-shaped sets (many tiles, ragged tails) ---------------------------

def test_scaled_c2_vs_oracle(SetBWTE):
    d, o = synth.uniform(100_000, 100, seed=1)
    want = oracle.bwt(A, d, o, threads=None)
    idx = build(SetBWTE, d, o, M=1 << 20)
    assert idx.bwt() == want


def test_long_reads_vs_oracle(SetBWTE):
    d, o = synth.uniform_var(2000, 1000, 10000, seed=4)     # c4-shaped lengths
    want = oracle.bwt(A, d, o, threads=None)
    assert build(SetBWTE, d, o, M=1 << 21).bwt() == want


@pytest.mark.slow
def test_c2_full_vs_oracle(SetBWTE):
    """BASELINE configs[1] at full size, in the configuration bench.py times."""
    d, o = synth.uniform(1_000_000, 100, seed=1)
    want = oracle.bwt(A, d, o, threads=None)
    idx = build(SetBWTE, d, o, M=1 << 24)
    assert idx.stats()["blocks"] == 7
    assert idx.bwt() == want


# --- host-tiered B_ext (A6 variant, c5 path) -----------------------------------

@pytest.mark.parametrize("budget", [1, 20000, 1 << 40])
def test_host_tier_c1(SetBWTE, c1, budget):
    """B_ext in pinned host memory (hbm_budget_bytes=1: from the first block;
    20000: moves to the host mid-append), bit-exact vs the oracle."""
    d, o, want = c1
    idx = SetBWTE(A, block_suffixes=25250)
    idx.set_option("hbm_budget_bytes", budget)
    idx.append(d, o)
    assert idx.stats()["host_tier"] == (1 if budget < (1 << 40) else 0)
    assert idx.bwt() == want
    n = len(want)
    for c in "$ACGT":
        for k in (0, 1, 64, 65537, n):
            assert idx.rank(c, k) == oracle.rank(want, c, k)


@pytest.mark.parametrize("seed", range(10))
def test_host_tier_random_appends(SetBWTE, seed):
    d, o = synth.random_set(900 + seed, max_m=64, max_len=50)
    want = oracle.bwt(A, d, o)
    idx = SetBWTE(A, block_suffixes=int(np.random.default_rng(seed).integers(20, 400)))
    idx.set_option("hbm_budget_bytes", 1)
    m = len(o) - 1
    cuts = sorted(set(np.random.default_rng(seed).integers(0, m + 1, size=3).tolist()))
    prev = 0
    for c in cuts + [m]:
        if c > prev:
            oo = np.asarray(o[prev:c + 1], dtype=np.uint64)
            idx.append(d[int(oo[0]):int(oo[-1])], oo - oo[0])
            prev = c
    assert idx.bwt() == want


def test_host_tier_multichunk(SetBWTE):
    """More than one 2^26-symbol staging chunk: 1M x 100 bp (101 M symbols)."""
    d, o = synth.uniform(700_000, 100, seed=21)
    want = oracle.bwt(A, d, o, threads=None)
    idx = SetBWTE(A, block_suffixes=1 << 24)
    idx.set_option("hbm_budget_bytes", 1 << 20)
    idx.append(d, o)
    st = idx.stats()
    assert st["host_tier"] == 1
    assert idx.bwt() == want
    # <= 3 n log(sigma) bits of system memory = 0.75 B/symbol for
    # sigma = 4 (1.5x growth of 4 bits/symbol), +2 MB mapping granularity
    assert st["host_dict_bytes"] <= 0.75 * st["n"] + (4 << 20)


def test_host_tier_growth_keeps_content_and_bound(SetBWTE):
    """Many appends into a host-tier index: the pinned dictionary grows in
    place (mremap) several times, pipelined multi-chunk Inserts each time."""
    d, o = synth.uniform(900_000, 100, seed=22)
    want = oracle.bwt(A, d, o, threads=None)
    idx = SetBWTE(A, block_suffixes=1 << 22)
    idx.set_option("host_tier", 1)
    m = len(o) - 1
    oo = np.asarray(o, dtype=np.uint64)
    cuts = [0, 1000, 20_000, 100_000, 300_000, m]
    for a, b in zip(cuts[:-1], cuts[1:]):
        idx.append(d[int(oo[a]):int(oo[b])], oo[a:b + 1] - oo[a])
        st = idx.stats()
        assert st["host_dict_bytes"] <= 0.75 * st["n"] + (4 << 20)
    assert idx.bwt() == want


# --- FM-index count (NEXT-2) ----------------------------------------------------

def test_fm_count_examples(SetBWTE):
    for case in SPEC["fm_count"]:
        idx = SetBWTE(A)
        idx.append_strings(case["strings"])
        assert list(idx.count([case["pattern"]])) == [case["count"]], case["cite"]


@pytest.mark.parametrize("seed", range(6))
def test_fm_count_vs_oracle(SetBWTE, seed):
    d, o = synth.random_set(8000 + seed, max_m=64, max_len=50, alphabet=["ACGT", "AC", "GT"][seed % 3])
    rng = np.random.default_rng(seed)
    pats = ["".join(rng.choice(list("ACGT"), size=int(rng.integers(1, 13)))) for _ in range(300)]
    pats += ["", "ACGTN", "a"]
    idx = SetBWTE(A, block_suffixes=int(rng.integers(50, 500)))
    idx.append(d, o)
    want = oracle.count(A, d, o, pats)
    want[-2] = 0  # 'N' is outside the alphabet
    assert np.array_equal(idx.count(pats), want)


def test_fm_count_c1_and_host_tier(SetBWTE, c1):
    d, o, _ = c1
    rng = np.random.default_rng(5)
    starts = rng.integers(0, len(d) - 20, size=200)
    pats = [bytes(d[a:a + int(rng.integers(1, 16))]).decode() for a in starts]
    want = oracle.count(A, d, o, pats, threads=None)
    for budget in (1 << 40, 1):
        idx = SetBWTE(A, block_suffixes=25250)
        idx.set_option("hbm_budget_bytes", budget)
        idx.append(d, o)
        assert np.array_equal(idx.count(pats), want)


# --- reverse orientation and BWT merge (NEXT-4) ------------------------

def _split(d, o, cut):
    o = np.asarray(o, dtype=np.uint64)
    a_d, a_o = d[: int(o[cut])], o[: cut + 1]
    b_d, b_o = d[int(o[cut]):], o[cut:] - o[cut]
    return (a_d, a_o), (b_d, b_o)


def test_prepend_golden(SetBWTE):
    idx = SetBWTE(A)
    idx.append_strings(["GG", "", "AC"])
    idx.prepend_strings(["ACGT", "CA"])
    assert idx.bwt().decode() == TWO["one_shot_bwt"]
    idx = SetBWTE(A)
    idx.prepend_strings(["G"])
    idx.prepend_strings(["AC"])
    assert idx.bwt().decode() == "CG$A$"


@pytest.mark.parametrize("seed", range(12))
def test_prepend_random_vs_oracle(SetBWTE, seed):
    d, o = synth.random_set(9000 + seed, max_m=48, max_len=40, alphabet=["ACGT", "AC"][seed % 2])
    m = len(o) - 1
    rng = np.random.default_rng(seed)
    c1, c2 = sorted(rng.integers(0, m + 1, size=2).tolist())
    (x_d, x_o), (yz_d, yz_o) = _split(d, o, c1)
    (y_d, y_o), (z_d, z_o) = _split(yz_d, yz_o, c2 - c1)
    idx = SetBWTE(A, block_suffixes=int(rng.integers(20, 300)))
    idx.append(y_d, y_o)      # Y
    idx.prepend(x_d, x_o)     # X Y
    idx.append(z_d, z_o)      # X Y Z
    assert idx.bwt() == oracle.bwt(A, d, o)


def test_prepend_device_c1(SetBWTE, c1):
    import torch
    d, o, want = c1
    (a_d, a_o), (b_d, b_o) = _split(d, o, 400)
    idx = SetBWTE(A, block_suffixes=25250)
    idx.append(b_d, b_o)
    idx.prepend_device(torch.from_numpy(np.ascontiguousarray(a_d)).cuda(),
                       torch.from_numpy(np.ascontiguousarray(a_o).view(np.int64)).cuda())
    assert idx.bwt() == want


@pytest.mark.parametrize("seed", range(12))
def test_merge_random_vs_oracle(SetBWTE, seed):
    d, o = synth.random_set(9500 + seed, max_m=48, max_len=40, alphabet=["ACGT", "GT"][seed % 2])
    m = len(o) - 1
    rng = np.random.default_rng(seed)
    cut = int(rng.integers(0, m + 1))
    (a_d, a_o), (b_d, b_o) = _split(d, o, cut)
    h = SetBWTE(A, block_suffixes=int(rng.integers(20, 300)))
    h.append(a_d, a_o)
    other = SetBWTE(A, block_suffixes=int(rng.integers(20, 300)))
    other.append(b_d, b_o)
    before = other.bwt()
    h.merge(other)
    assert h.bwt() == oracle.bwt(A, d, o)
    assert other.bwt() == before == oracle.bwt(A, b_d, b_o)
    assert h.size() == (int(o[-1]) + m, m)


@pytest.mark.parametrize("budget", [1 << 40, 1])
def test_merge_c1_and_host_tier(SetBWTE, c1, budget):
    d, o, want = c1
    (a_d, a_o), (b_d, b_o) = _split(d, o, 600)
    h = SetBWTE(A, block_suffixes=25250)
    h.set_option("hbm_budget_bytes", budget)
    h.append(a_d, a_o)
    other = SetBWTE(A, block_suffixes=10000)
    other.set_option("hbm_budget_bytes", budget)
    other.append(b_d, b_o)
    h.merge(other)
    assert h.bwt() == want
    # queries on the merged index
    rng = np.random.default_rng(1)
    starts = rng.integers(0, len(d) - 12, size=50)
    pats = [bytes(d[a:a + 6]).decode() for a in starts]
    assert np.array_equal(h.count(pats), oracle.count(A, d, o, pats))


def test_merge_edge_cases(SetBWTE):
    empty = SetBWTE(A)
    h = SetBWTE(A)
    h.append_strings(["AC", "G"])
    h.merge(empty)
    assert h.bwt().decode() == "CG$A$"
    e2 = SetBWTE(A)
    e2.merge(h)
    assert e2.bwt().decode() == "CG$A$"
    e3 = SetBWTE(A)
    e3.append_strings(["", ""])
    e3.merge(h)   # {"","","AC","G"}
    d, o = synth.from_strings(["", "", "AC", "G"])
    assert e3.bwt() == oracle.bwt(A, d, o)
    with pytest.raises(Exception):
        h.merge(h)
    other = SetBWTE("AC")
    other.append_strings(["AC"])
    with pytest.raises(Exception):
        h.merge(other)


# --- blocks without the SA payload (the > 2^29-suffix path, forced small) ---------

@pytest.mark.parametrize("seed", range(16))
def test_random_sets_without_payload(SetBWTE, seed):
    d, o = synth.random_set(13000 + seed, max_m=48, max_len=60, alphabet=["ACGT", "AC"][seed % 2])
    rng = np.random.default_rng(seed)
    idx = SetBWTE(A, block_suffixes=int(rng.integers(30, 400)))
    idx.set_option("sa_payload", 0)
    m = len(o) - 1
    cut = int(rng.integers(0, m + 1))
    o = np.asarray(o, dtype=np.uint64)
    idx.append(d[: int(o[cut])], o[: cut + 1])
    idx.append(d[int(o[cut]):], o[cut:] - o[cut])
    assert idx.bwt() == oracle.bwt(A, d, o)


@pytest.mark.parametrize("M", [25250, 50500])
def test_c1_without_payload(SetBWTE, c1, M):
    d, o, want = c1
    idx = SetBWTE(A, block_suffixes=M)
    idx.set_option("sa_payload", 0)
    idx.append(d, o)
    assert idx.bwt() == want
    # stage view: ConstructSA + B_int of one block, SA entries without payload
    sa, bint = idx.construct_sa(d[: int(o[50])], o[:51])
    assert list(sa) == list(oracle.block_sa(A, d[: int(o[50])], o[:51]))


def test_genome_without_payload(SetBWTE):
    d, o = synth.genome_sampled(3000, 120, 60000, seed=4)
    idx = SetBWTE(A, block_suffixes=60000)
    idx.set_option("sa_payload", 0)
    idx.append(d, o)
    assert idx.bwt() == oracle.bwt(A, d, o, threads=None)


@pytest.mark.parametrize("payload", [0, 1])
@pytest.mark.parametrize("seed", range(6))
def test_random_sets_u64_g(SetBWTE, seed, payload):
    """u64 g / pos (forced), with and without the SA payload (without it,
    ComputeRanks stores B_int in g's top byte)."""
    d, o = synth.random_set(14000 + seed, max_m=48, max_len=60)
    rng = np.random.default_rng(seed)
    idx = SetBWTE(A, block_suffixes=int(rng.integers(30, 400)))
    idx.set_option("g_width", 8)
    idx.set_option("sa_payload", payload)
    idx.append(d, o)
    assert idx.bwt() == oracle.bwt(A, d, o)


def test_c1_u64_g_without_payload(SetBWTE, c1):
    d, o, want = c1
    idx = SetBWTE(A, block_suffixes=25250)
    idx.set_option("g_width", 8)
    idx.set_option("sa_payload", 0)
    idx.append(d, o)
    assert idx.bwt() == want


@pytest.mark.parametrize("payload", [0, 1])
@pytest.mark.parametrize("kind", ["all_A", "AC_repeat", "staircase", "uniform"])
def test_tie_heavy_small_blocks(SetBWTE, kind, payload):
    """Tie-heavy inputs in small blocks (many key words per suffix), with and
    without the SA payload."""
    if kind == "uniform":
        d, o = synth.random_set(15000, max_m=64, max_len=80)
    else:
        d, o = synth.adversarial(kind, 40, 70)
    idx = SetBWTE(A, block_suffixes=500)
    idx.set_option("sa_payload", payload)
    idx.append(d, o)
    assert idx.bwt() == oracle.bwt(A, d, o)


def test_genome_one_block(SetBWTE):
    d, o = synth.genome_sampled(3000, 120, 60000, seed=5)
    idx = SetBWTE(A, block_suffixes=90000)
    idx.append(d, o)
    assert idx.bwt() == oracle.bwt(A, d, o, threads=None)


@pytest.mark.parametrize("seed", range(12))
def test_random_sets_small_blocks(SetBWTE, seed):
    """Random sets with small blocks, both SA layouts and g widths."""
    d, o = synth.random_set(16000 + seed, max_m=64, max_len=90, alphabet=["ACGT", "AC", "A"][seed % 3])
    rng = np.random.default_rng(seed)
    idx = SetBWTE(A, block_suffixes=int(rng.integers(40, 3000)))
    idx.set_option("sa_payload", seed % 2)
    if seed % 4 == 3:
        idx.set_option("g_width", 8)
    idx.append(d, o)
    assert idx.bwt() == oracle.bwt(A, d, o)


def test_c1_one_and_four_blocks(SetBWTE, c1):
    d, o, want = c1
    for M in (25250, 101000):
        idx = SetBWTE(A, block_suffixes=M)
        idx.append(d, o)
        assert idx.bwt() == want


@pytest.mark.parametrize("budget", [1 << 40, 1])
@pytest.mark.parametrize("seed", range(4))
def test_random_sets_hbm_and_host_tier(SetBWTE, seed, budget):
    """Random sets, HBM and host-tier dictionaries (options rank_ilp / kw1_min
    are retired: they must be rejected)."""
    d, o = synth.random_set(17000 + seed, max_m=64, max_len=70)
    rng = np.random.default_rng(seed)
    idx = SetBWTE(A, block_suffixes=int(rng.integers(30, 600)))
    from paper_1410_0562_b200 import SetBWTEError
    for key in ("rank_ilp", "kw1_min"):
        with pytest.raises(SetBWTEError):
            idx.set_option(key, 4)
    idx.set_option("hbm_budget_bytes", budget)
    if seed % 2:
        idx.set_option("g_width", 8)
    idx.append(d, o)
    assert idx.bwt() == oracle.bwt(A, d, o)


@pytest.mark.parametrize("lanes", [0, 1, 2])
def test_pipeline_depth_does_not_change_the_result(SetBWTE, c1, lanes):
    """SPEC acceptance 8 (determinism across pipeline depth): the sort lanes
    only reorder work, never the result."""
    d, o, want = c1
    idx = SetBWTE(A, block_suffixes=7000)
    idx.set_option("sort_lanes", lanes)
    idx.append(d, o)
    assert idx.bwt() == want


def test_option_validation(SetBWTE):
    idx = SetBWTE(A)
    for key, bad in [("block_suffixes", 0), ("rank_ilp", 9), ("g_width", 5), ("sa_payload", 2),
                     ("insert_split", 3), ("kw1_min", 0), ("no_such_option", 1)]:
        with pytest.raises(Exception):
            idx.set_option(key, bad)
    idx.append_strings(["ACGT"])
    assert idx.bwt().decode() == "T$ACG"


@pytest.mark.parametrize("kind", ["uniform", "genome"])
def test_replayed_sort_pattern(SetBWTE, kind):
    """Blocks of >= 2^20 suffixes replay the launch pattern recorded on an
    earlier block (no count read-backs between rounds).  Segments of a class
    the pattern skips carry over to a later round; the genome-sampled reads
    (deep, uneven LCPs) make the replayed pattern miss rounds."""
    if kind == "uniform":
        d, o = synth.uniform(40000, 100, seed=21)
    else:
        d, o = synth.genome_sampled(40000, 100, 1_500_000, seed=22)
    want = oracle.bwt(A, d, o, threads=None)
    idx = SetBWTE(A, block_suffixes=1 << 20)
    idx.append(d, o)          # the first block records, later full blocks replay
    assert idx.bwt() == want
    idx.clear()
    idx.append(d, o)          # every full block replays
    assert idx.bwt() == want
    st = idx.stats()["sort"]
    assert st["replayed_blocks"] >= 3, st


def test_replayed_pattern_that_does_not_fit(SetBWTE):
    """A pattern recorded on uniform reads replayed on genome-sampled and
    all-A blocks of the same size: the replay misses classes and rounds, the
    skipped segments carry over and host-driven rounds finish the sort."""
    du, ou = synth.uniform(20000, 100, seed=23)
    dg, og = synth.genome_sampled(20000, 100, 300_000, seed=24)
    da, oa = synth.adversarial("all_A", 12000, 100)
    parts = [(du, ou), (dg, og), (da, oa)]
    d = np.concatenate([p[0] for p in parts])
    offs = [np.asarray(ou, dtype=np.uint64)]
    for p in parts[1:]:
        offs.append(np.asarray(p[1][1:], dtype=np.uint64) + offs[-1][-1])
    o = np.concatenate(offs)
    want = oracle.bwt(A, d, o, threads=None)
    idx = SetBWTE(A, block_suffixes=1 << 20)
    for pd, po in parts:
        idx.append(pd, po)
    assert idx.bwt() == want
    st = idx.stats()["sort"]
    assert st["replayed_blocks"] >= 1 and st["rounds_after_replay"] >= 1, st


# --- caller allocator (setbwte_set_allocator) --------------------

def test_torch_caching_allocator(SetBWTE, c1):
    """Every handle allocation comes from torch's caching allocator (also from
    the sort-lane threads) and is handed back at destroy; results unchanged."""
    import torch
    d, o, want = c1
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    idx = SetBWTE(A, block_suffixes=20000)
    idx.use_torch_allocator()
    (a_d, a_o), (b_d, b_o) = _split(d, o, 300)
    idx.append(a_d, a_o)
    idx.append(b_d, b_o)  # larger: buffers regrow through the allocator
    assert idx.bwt() == want
    assert torch.cuda.memory_allocated() - base > 4 * len(d)
    idx.close()
    assert torch.cuda.memory_allocated() == base


def test_counting_allocator_and_restore(SetBWTE):
    import torch
    live = {}

    def alloc(n):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        live[t.data_ptr()] = t
        return t.data_ptr()

    def free(p):
        del live[p]
    d, o = synth.uniform(40, 60, seed=77)
    idx = SetBWTE(A, block_suffixes=100)
    idx.append(d[: int(o[10])], o[:11])   # cudaMalloc'd buffers
    idx.set_allocator(alloc, free)
    idx.append(d[int(o[10]):], o[10:] - o[10])
    assert idx.bwt() == oracle.bwt(A, d, o)
    assert live
    idx.set_allocator(None, None)
    idx.close()
    assert not live
    # an allocator that fails: E_NOMEM, handle reports it
    idx = SetBWTE(A)
    idx.set_allocator(lambda n: 0, lambda p: None)
    from paper_1410_0562_b200.binding import SetBWTEError
    with pytest.raises(SetBWTEError, match="E_NOMEM"):
        idx.append(d, o)


# --- invalid input into an EMPTY index: validation deferred to the end ----------

@pytest.mark.parametrize("lanes", [0, 3])
@pytest.mark.parametrize("device", [False, True])
def test_invalid_char_into_empty_index(SetBWTE, lanes, device):
    """An empty index validates host input only after the blocks were inserted
    (nothing to roll back); a bad byte in a late block empties it again and
    reports the same position as the eager check."""
    import torch
    from paper_1410_0562_b200 import SetBWTEError
    d, o = synth.uniform(3000, 50, seed=5)
    bad = d.copy()
    bad_pos = int(o[2900]) + 7
    bad[bad_pos] = ord("X")
    idx = SetBWTE(A, block_suffixes=5000)
    idx.set_option("sort_lanes", lanes)
    with pytest.raises(SetBWTEError) as e:
        if device:
            idx.append_device(torch.from_numpy(bad).cuda(), torch.from_numpy(o.view(np.int64)).cuda())
        else:
            idx.append(bad, o)
    assert e.value.name == "E_INVALID_CHAR"
    assert idx.last_error() == (bad_pos, ord("X"))
    assert idx.size() == (0, 0) and idx.bwt() == b""
    idx.append(d, o)
    assert idx.bwt() == oracle.bwt(A, d, o)
    # a non-empty index still rejects before its first Insert (unchanged)
    with pytest.raises(SetBWTEError):
        idx.append(bad, o)
    assert idx.bwt() == oracle.bwt(A, d, o)


# --- bucketed gather (gather.cu): forced at small sizes, every B_int source ----

@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("opts", [dict(), dict(g_width=8), dict(sa_payload=0),
                                  dict(sa_payload=0, g_width=8)])
def test_bucketed_gather_random_sets(SetBWTE, seed, opts):
    d, o = synth.random_set(24000 + seed, max_m=64, max_len=60)
    want = oracle.bwt(A, d, o)
    idx = SetBWTE(A, block_suffixes=int(np.random.default_rng(seed).integers(50, 3000)))
    idx.set_option("gather_buckets", 2)
    for k, v in opts.items():
        idx.set_option(k, v)
    m = len(o) - 1
    oo = np.asarray(o, dtype=np.uint64)
    idx.append(d[: int(oo[m // 2])], oo[: m // 2 + 1])
    idx.append(d[int(oo[m // 2]):], oo[m // 2:] - oo[m // 2])
    assert idx.bwt() == want


@pytest.mark.parametrize("M", [25250, 1 << 20])
def test_bucketed_gather_c1_and_scaled(SetBWTE, c1, M):
    d, o, want = c1
    idx = build(SetBWTE, d, o, M=M)
    ref = idx.bwt()
    idx2 = SetBWTE(A, block_suffixes=M)
    idx2.set_option("gather_buckets", 2)
    idx2.append(d, o)
    assert idx2.bwt() == want == ref


def test_bucketed_gather_multi_tile_blocks(SetBWTE):
    """300k reads, blocks of 2^23 suffixes: thousands of 4096-position tiles
    and 8+ buckets per block, forced."""
    d, o = synth.uniform(300_000, 100, seed=11)
    want = oracle.bwt(A, d, o, threads=None)
    for gw in (0, 8):
        idx = SetBWTE(A, block_suffixes=1 << 23)
        idx.set_option("gather_buckets", 2)
        if gw:
            idx.set_option("g_width", 8)
        idx.append(d, o)
        assert idx.bwt() == want


def test_third_level_counting_path(SetBWTE):
    """One block of 40 M suffixes (400k x 100 bp, M = 2^26): after two 8-bit
    digit passes the segments hold ~600 members with 16 key bits left -- the
    one-CTA pass's 11-bit counting placement (sort.cu FAST PATH), whose
    in-bucket order is restored by original position.  Whole BWT vs the
    oracle, plus a genome-sampled set whose deep ties take the stable path."""
    d, o = synth.uniform(400_000, 100, seed=31)
    want = oracle.bwt(A, d, o, threads=None)
    idx = SetBWTE(A, block_suffixes=1 << 26)
    idx.append(d, o)
    assert idx.bwt() == want
    d, o = synth.genome_sampled(400_000, 100, 8_000_000, seed=32)
    want = oracle.bwt(A, d, o, threads=None)
    idx = SetBWTE(A, block_suffixes=1 << 26)
    idx.append(d, o)
    assert idx.bwt() == want


# --- pack (pack.cu): string boundaries against 32-slot groups and 1024-slot
# warp windows, runs of empty / one-symbol strings, long strings -------------

def _pack_layout(kind, rng):
    if kind == "short":       # 0..2 symbols: up to 32 terminators per group
        lens = rng.integers(0, 3, size=3000)
    elif kind == "edges":     # lengths 31, 32, 33, 1023, 1024, 1025 (slot = len + 1)
        lens = rng.choice([30, 31, 32, 1022, 1023, 1024], size=300)
    elif kind == "long":      # few long strings: groups with no terminator
        lens = rng.integers(2000, 6000, size=12)
    else:                     # mixed
        lens = np.concatenate([rng.integers(0, 3, size=500), rng.integers(90, 110, size=300),
                               rng.integers(1000, 3000, size=5)])
        rng.shuffle(lens)
    return ["".join("ACGT"[c] for c in rng.integers(0, 4, size=int(n))) for n in lens]


@pytest.mark.parametrize("kind", ["short", "edges", "long", "mixed"])
@pytest.mark.parametrize("lanes", [0, 3])
def test_pack_layouts(SetBWTE, kind, lanes):
    rng = np.random.default_rng(["short", "edges", "long", "mixed"].index(kind))
    d, o = synth.from_strings(_pack_layout(kind, rng))
    # small blocks: several pack ranges, each starting mid-group
    M = max(64, int(o[-1] + len(o) - 1) // 5 + 1)
    idx = SetBWTE(A, block_suffixes=M)
    idx.set_option("sort_lanes", lanes)
    idx.append(d, o)
    assert idx.bwt() == oracle.bwt(A, d, o)


@pytest.mark.parametrize("where", ["first", "window_edge", "last", "two"])
def test_pack_invalid_byte_position(SetBWTE, where):
    """The first invalid byte is reported, wherever it falls against the
    pack's groups and warp windows (the index stays as it was)."""
    from paper_1410_0562_b200 import SetBWTEError
    rng = np.random.default_rng(7)
    d, o = synth.from_strings(_pack_layout("mixed", rng))
    n = int(o[-1])
    pos = {"first": [0], "window_edge": [1023 - 40, 2047 - 77], "last": [n - 1],
           "two": [n // 2, n // 3]}[where]
    bad = d.copy()
    for p in pos:
        bad[p] = ord("#")
    idx = SetBWTE(A, block_suffixes=max(64, (n + len(o)) // 4))
    idx.append_strings(["ACGT"])
    with pytest.raises(SetBWTEError) as e:
        idx.append(bad, o)
    assert e.value.name == "E_INVALID_CHAR"
    assert idx.last_error() == (min(pos), ord("#"))
    assert idx.bwt() == oracle.bwt(A, *synth.from_strings(["ACGT"]))


@pytest.mark.parametrize("kind", ["short", "edges", "mixed"])
def test_pack_layouts_sigma5(SetBWTE, kind):
    rng = np.random.default_rng(11 + len(kind))
    strs = _pack_layout(kind, rng)
    # an N in about every tenth string
    strs = [s[:len(s) // 2] + "N" + s[len(s) // 2 + 1:] if s and i % 10 == 0 else s
            for i, s in enumerate(strs)]
    d, o = synth.from_strings(strs)
    idx = SetBWTE("ACGTN", block_suffixes=max(64, int(o[-1] + len(o) - 1) // 3 + 1))
    idx.append(d, o)
    assert idx.bwt() == oracle.bwt("ACGTN", d, o)


def test_profile_timeline(SetBWTE, c1):
    """Profile mode 3: every launch of the last append with its stream and
    start / end (ms from the append's start); results unchanged."""
    d, o, want = c1
    idx = SetBWTE(A, block_suffixes=25250)
    idx.set_profile(3)
    idx.append(d, o)
    st = idx.stats()
    tl = st["timeline"]
    assert len(tl) == st["launches"] > 0
    names = {n for n, _, _, _ in tl}
    assert {"compute_ranks", "gather", "insert", "pack"} <= names
    assert all(t1 >= t0 >= -0.01 for _, _, t0, t1 in tl)
    assert sum(k["launches"] for k in st["kernels"].values()) == len(tl)
    assert idx.bwt() == want
    idx.set_profile(0)
    idx.clear()
    idx.append(d, o)
    assert "timeline" not in idx.stats()
