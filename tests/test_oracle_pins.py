"""Pins for the CPU oracle (no GPU).  Each test ties an oracle function to
something other than itself: worked examples (tests/golden, cited), brute
force over the materialised text, the textbook rotation BWT, closed forms,
invariants, and Algorithm 1/2 transcribed naively (tests/brute.py)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))
TWO = json.load(open(os.path.join(GOLD, "two_block_example.json")))
A = "ACGT"


def _fs(strings):
    return synth.from_strings(strings)


def _slots_from_jk(strings, jk):
    slot = {p: s for s, p in enumerate(brute.slot_jk(strings))}
    return [slot[tuple(p)] for p in jk]


# --- worked examples --------------------------------------------------------

@pytest.mark.parametrize("case", SPEC["bwt"], ids=lambda c: c["cite"][:12])
def test_golden_bwt(case):
    d, o = _fs(case["strings"])
    assert oracle.bwt(A, d, o).decode() == case["bwt"]


@pytest.mark.parametrize("case", SPEC["block_sa"], ids=lambda c: c["cite"][:6])
def test_golden_block_sa(case):
    d, o = _fs(case["strings"])
    want = _slots_from_jk(case["strings"], case["sa_jk"])
    assert list(oracle.block_sa(A, d, o)) == want


@pytest.mark.parametrize("case", SPEC["block_bint"], ids=lambda c: c["cite"][:6])
def test_golden_block_bint(case):
    d, o = _fs(case["strings"])
    sa = oracle.block_sa(A, d, o)
    assert oracle.block_bint(A, d, o, sa).decode() == case["bint"]


@pytest.mark.parametrize("case", SPEC["compute_ranks"], ids=lambda c: c["cite"][:6])
def test_golden_compute_ranks(case):
    d, o = _fs(case["ext"] + case["block"])
    g = oracle.compute_ranks(A, d, o, m_ext=len(case["ext"]))
    assert list(g) == case["g"]


@pytest.mark.parametrize("case", SPEC["rank"], ids=lambda c: c["cite"][:6])
def test_golden_rank(case):
    assert oracle.rank(case["B"].encode(), case["c"], case["k"]) == case["rank"]


@pytest.mark.parametrize("case", SPEC["insert"], ids=lambda c: c["cite"][:6])
def test_golden_insert(case):
    out = oracle.insert(case["b_ext"].encode(), case["b_int"].encode(), case["g_sa"])
    assert out.decode() == case["out"]


def test_golden_lf_and_C():
    for case in SPEC["C"]:
        B = case["B"].encode()
        for c, want in case["C"].items():
            got = sum(oracle.rank(B, x, len(B)) for x in ("$" + A)[: ("$" + A).index(c)])
            assert got == want, case["cite"]
    for case in SPEC["lf_step"]:
        B = case["B"].encode()
        C = {c: sum(oracle.rank(B, x, len(B)) for x in ("$" + A)[: ("$" + A).index(c)])
             for c in "$" + A}
        assert C[case["c"]] + oracle.rank(B, case["c"], case["i"]) == case["j"], case["cite"]


def test_golden_two_block_all_intermediates():
    strings = TWO["strings"]
    d, o = _fs(strings)
    assert oracle.bwt(A, d, o).decode() == TWO["one_shot_bwt"]
    m_ext = 0
    b_ext = b""
    for blk in TWO["blocks"]:
        bd, bo = _fs(blk["strings"])
        sa = oracle.block_sa(A, bd, bo)
        assert list(sa) == blk["sa_slots"]
        bint = oracle.block_bint(A, bd, bo, sa)
        assert bint.decode() == blk["bint"]
        sd, so = _fs(strings[: m_ext + len(blk["strings"])])
        g = oracle.compute_ranks(A, sd, so, m_ext=m_ext)
        assert list(g) == blk["g"]
        g_sa = g[sa.astype(np.int64)]
        assert list(g_sa) == blk["g_sa"]
        assert list(g_sa + np.arange(len(g_sa), dtype=np.uint64)) == blk["pos"]
        b_ext = oracle.insert(b_ext, bint, g_sa)
        assert b_ext.decode() == blk["b_ext_after"]
        m_ext += len(blk["strings"])


# --- brute force on tiny inputs ---------------------------------------------

@pytest.mark.parametrize("seed", range(60))
def test_bwt_equals_brute_force(seed):
    alpha = ["ACGT", "AC", "A", "ACG"][seed % 4]
    d, o = synth.random_set(seed, max_m=16, max_len=20, alphabet=alpha)
    strings = synth.to_strings(d, o)
    assert oracle.bwt(A, d, o).decode() == brute.brute_bwt(strings)


@pytest.mark.parametrize("seed", range(30))
def test_block_sa_equals_brute_force(seed):
    d, o = synth.random_set(1000 + seed, max_m=12, max_len=15, alphabet=["ACGT", "AC"][seed % 2])
    strings = synth.to_strings(d, o)
    want = _slots_from_jk(strings, brute.brute_sa_jk(strings))
    assert list(oracle.block_sa(A, d, o)) == want


@pytest.mark.parametrize("seed", range(30))
def test_compute_ranks_equals_brute_force_and_alg2(seed):
    d, o = synth.random_set(2000 + seed, max_m=14, max_len=12, alphabet=["ACGT", "AG"][seed % 2])
    strings = synth.to_strings(d, o)
    cut = len(strings) // 2
    ext, blk = strings[:cut], strings[cut:]
    g = list(oracle.compute_ranks(A, d, o, m_ext=cut))
    assert g == brute.brute_g(ext, blk)
    # Lemma 1 / Alg.2 with m_ext initialisation (reading R1) gives the same g
    B_ext = brute.brute_bwt(ext) if ext else ""
    assert g == brute.alg2_compute_ranks(blk, B_ext, len(ext))


def test_alg2_with_n_ext_init_disagrees():
    """Reading R1: the literal 'i := n_ext' contradicts Lemma 1 under
    the order of P:37.  {"AC"} then {"G"}: m_ext init reproduces Eq.(1)."""
    B_ext = brute.brute_bwt(["AC"])
    g_m = brute.alg2_compute_ranks(["G"], B_ext, m_ext=1)
    g_n = brute.alg2_compute_ranks(["G"], B_ext, m_ext=len(B_ext))
    assert g_m == [3, 1] and g_n != g_m


@pytest.mark.parametrize("seed", range(10))
def test_suffix_rank_equals_brute_sa(seed):
    d, o = synth.random_set(3000 + seed, max_m=8, max_len=10)
    strings = synth.to_strings(d, o)
    sa = brute.brute_sa_jk(strings)
    for r, (j, k) in enumerate(sa):
        assert oracle.suffix_rank(A, d, o, j, k, threads=1) == r


# --- textbook special case, closed forms, invariants -------------------------

@pytest.mark.parametrize("s", ["ACGT", "GATTACA", "A", "AAAA", "TTTTGA", "ACACACAG", ""])
def test_single_string_is_textbook_bwt(s):
    d, o = _fs([s])
    assert oracle.bwt(A, d, o).decode() == brute.rotation_bwt(s)


@pytest.mark.parametrize("m,L", [(1, 1), (3, 5), (7, 2), (20, 13)])
def test_closed_form_identical_A_reads(m, L):
    d, o = _fs(["A" * L] * m)
    assert oracle.bwt(A, d, o).decode() == "A" * (m * L) + "$" * m


@pytest.mark.parametrize("seed", range(20))
def test_invariants(seed):
    d, o = synth.random_set(4000 + seed, max_m=20, max_len=30)
    strings = synth.to_strings(d, o)
    m = len(strings)
    B = oracle.bwt(A, d, o).decode()
    # |B| = sum(|S|+1); exactly m '$'; permutation of the input plus m '$'
    assert len(B) == sum(len(s) + 1 for s in strings)
    assert sorted(B) == sorted("".join(strings) + "$" * m)
    # B[0..m) = the last symbol of each string, '$' for an empty one
    assert B[:m] == "".join(s[-1] if s else "$" for s in strings)
    # LF inversion recovers every string (FM-index)
    assert brute.lf_invert(B, m) == strings
    # rank identities (Eq.(2)): sum_c rank(c,i) = i
    Bb = B.encode()
    for i in range(0, len(B) + 1, max(1, len(B) // 7)):
        assert sum(oracle.rank(Bb, c, i) for c in "$" + A) == i


def test_lowercase_and_invalid():
    d, o = _fs(["acgt", "Gg"])
    assert oracle.bwt(A, d, o) == oracle.bwt(A, *_fs(["ACGT", "GG"]))
    d, o = _fs(["ACGT", "AXG"])
    with pytest.raises(oracle.OracleError, match="byte 5"):
        oracle.bwt(A, d, o)


# --- incremental construction == one-shot (north_star requirement) -----------

@pytest.mark.parametrize("seed", range(40))
def test_incremental_model_equals_oracle(seed):
    d, o = synth.random_set(5000 + seed, max_m=16, max_len=12)
    strings = synth.to_strings(d, o)
    rng = np.random.default_rng(seed)
    cuts = sorted(set(rng.integers(0, len(strings) + 1, size=3).tolist()))
    blocks, prev = [], 0
    for c in cuts + [len(strings)]:
        if c > prev:
            blocks.append(strings[prev:c])
            prev = c
    assert brute.alg1_incremental(blocks) == oracle.bwt(A, d, o).decode()


@pytest.mark.parametrize("seed", range(20))
def test_oracle_pieces_compose_to_oracle_bwt(seed):
    """The oracle's stage functions, chained as Algorithm 1, give its one-shot BWT."""
    d, o = synth.random_set(6000 + seed, max_m=20, max_len=15)
    strings = synth.to_strings(d, o)
    K = 1 + seed % 4
    bounds = np.linspace(0, len(strings), K + 1).astype(int)
    b_ext = b""
    for a, b in zip(bounds[:-1], bounds[1:]):
        if b == a:
            continue
        bd, bo = _fs(strings[a:b])
        sa = oracle.block_sa(A, bd, bo)
        bint = oracle.block_bint(A, bd, bo, sa)
        sd, so = _fs(strings[:b])
        g = oracle.compute_ranks(A, sd, so, m_ext=int(a))
        b_ext = oracle.insert(b_ext, bint, g[sa.astype(np.int64)])
    assert b_ext == oracle.bwt(A, d, o)


def test_parallel_sort_matches_serial():
    d, o = synth.uniform(2000, 50, seed=7)
    assert oracle.bwt(A, d, o, threads=4) == oracle.bwt(A, d, o, threads=1)


def test_fm_count_examples_via_oracle_bwt():
    """Backward search on the oracle BWT (C + rank) reproduces
    the SPEC fm_count examples and the naive substring count."""
    for case in SPEC["fm_count"]:
        d, o = _fs(case["strings"])
        B = oracle.bwt(A, d, o)
        C = {c: sum(oracle.rank(B, x, len(B)) for x in ("$" + A)[: ("$" + A).index(c)])
             for c in A}
        lo, hi = 0, len(B)
        for c in reversed(case["pattern"]):
            lo = C[c] + oracle.rank(B, c, lo)
            hi = C[c] + oracle.rank(B, c, hi)
        assert hi - lo == case["count"] == brute.naive_count(case["pattern"], case["strings"])


def test_oracle_count_pins():
    """oracle.count against SPEC's fm_count examples and a Python
    brute force (different code: str slicing)."""
    for case in SPEC["fm_count"]:
        d, o = _fs(case["strings"])
        assert list(oracle.count(A, d, o, [case["pattern"]])) == [case["count"]]
    for seed in range(10):
        d, o = synth.random_set(7000 + seed, max_m=12, max_len=20, alphabet=["ACGT", "AC"][seed % 2])
        strings = synth.to_strings(d, o)
        rng = np.random.default_rng(seed)
        pats = ["".join(rng.choice(list("ACGT"), size=int(rng.integers(1, 5)))) for _ in range(20)]
        got = oracle.count(A, d, o, pats)
        assert list(got) == [brute.naive_count(p, strings) for p in pats]


# --- sigma = 5 (N; NEXT-4 groundwork): the oracle is alphabet-generic

A5 = "ACGTN"  # code order A < C < G < T < N (SPEC's default alphabet)


@pytest.mark.parametrize("seed", range(12))
def test_sigma5_bwt_and_ranks_equal_brute_force(seed):
    d, o = synth.random_set(8000 + seed, max_m=12, max_len=14, alphabet=["ACGTN", "NA", "TN"][seed % 3])
    strings = synth.to_strings(d, o)
    assert oracle.bwt(A5, d, o).decode() == brute.brute_bwt(strings, A5)
    cut = len(strings) // 2
    g = list(oracle.compute_ranks(A5, d, o, m_ext=cut))
    assert g == brute.brute_g(strings[:cut], strings[cut:], A5)
    pats = ["N", "AN", "NN", "TNA", "GT"]
    assert list(oracle.count(A5, d, o, pats)) == [brute.naive_count(p, strings) for p in pats]


@pytest.mark.parametrize("s", ["NNNN", "GATNACA", "N", "ANTN"])
def test_sigma5_single_string_is_textbook_bwt(s):
    d, o = _fs([s])
    assert oracle.bwt(A5, d, o).decode() == brute.rotation_bwt(s, A5)


# --- bucketed low-memory mode (used for the c3-c5 golden digests)

def _bucketed(alpha, d, o, h, cap, threads=2):
    parts, keys = [], []
    oracle.bwt_bucketed(alpha, d, o, lambda c, b: (parts.append(c), keys.append(b)),
                        h=h, batch_cap=cap, threads=threads)
    return b"".join(parts), keys, parts


@pytest.mark.parametrize("seed", range(16))
def test_bucketed_bwt_equals_brute_force(seed):
    """Bucketed mode against the brute force over the materialised integer
    text (tests/brute.py, different code), for h = 1..4 and batch caps that
    force one bucket per batch, a few buckets per batch, and one batch."""
    alpha = ["ACGT", "AC", "A", "ACGTN"][seed % 4]
    d, o = synth.random_set(9100 + seed, max_m=20, max_len=16,
                            alphabet=alpha if alpha != "ACGTN" else "ACGTN")
    strings = synth.to_strings(d, o)
    want = brute.brute_bwt(strings, alpha).encode()
    for h in (1, 2, 3, 4):
        for cap in (1, 5, 1 << 20):
            got, _, _ = _bucketed(alpha, d, o, h, cap)
            assert got == want, (h, cap)


def test_bucketed_bucket_sizes_and_order():
    """Each emitted chunk is exactly the bucket of suffixes sharing that
    h-symbol prefix ($ and after as digit 0), emitted in increasing key order:
    counted here by slicing the strings in Python."""
    d, o = synth.random_set(9301, max_m=30, max_len=12)
    strings = synth.to_strings(d, o)
    h, base = 2, 5
    want = {}
    for s in strings:
        for k in range(len(s) + 1):
            key = 0
            for p in range(k, k + h):
                key = key * base + ("ACGT".index(s[p]) + 1 if p < len(s) else 0)
            want[key] = want.get(key, 0) + 1
    _, keys, parts = _bucketed(A, d, o, h, 3)
    assert keys == sorted(want)
    assert [len(p) for p in parts] == [want[k] for k in keys]


@pytest.mark.parametrize("m,L", [(7, 5), (40, 1), (3, 30)])
def test_bucketed_closed_form_identical_A_reads(m, L):
    d, o = _fs(["A" * L] * m)
    got, _, _ = _bucketed(A, d, o, 3, 2)
    assert got == b"A" * (m * L) + b"$" * m


def test_bucketed_matches_oracle_on_reads():
    d, o = synth.uniform(3000, 100, seed=5)
    got, _, _ = _bucketed(A, d, o, 3, 50_000, threads=4)
    assert got == oracle.bwt(A, d, o, threads=4)


# --- the golden full-size digests (tools/make_golden_digests.py) ---------------

@pytest.mark.parametrize("cfg", ["c3", "c4", "c5"])
def test_golden_digest_files_are_consistent(cfg):
    """Self-consistency of the oracle-written digest files: bucket ranges tile
    [0, n), the symbol counts add up to n with exactly m terminators, the
    windows lie inside B and agree with the bucket layout's length."""
    gd = json.load(open(os.path.join(GOLD, "%s_bwt_digest.json" % cfg)))
    n, m = gd["n"], gd["m"]
    pos = 0
    for b in gd["buckets"]:
        assert b["start"] == pos and b["len"] > 0
        pos += b["len"]
    assert pos == n
    cnt = gd["symbol_counts"]
    assert sum(cnt.values()) == n and cnt["$"] == m
    for w in gd["windows"]:
        assert 0 <= w["start"] and w["start"] + len(w["bytes"]) <= n
        assert set(w["bytes"]) <= set("$ACGT")


def test_golden_c3_digest_against_the_input():
    """The c3 digest against properties of the INPUT (no oracle call): the
    BWT's symbol multiset is the input's plus m terminators, and B[0..4096) --
    the rows of $_0..$_4095 -- are the last symbols of strings 0..4095
    (SURVEY 8(c) invariants)."""
    gd = json.load(open(os.path.join(GOLD, "c3_bwt_digest.json")))
    d, o = synth.uniform(20_000_000, 100, seed=1)
    assert gd["m"] == len(o) - 1 and gd["n"] == int(o[-1]) + len(o) - 1
    for c in "ACGT":
        assert gd["symbol_counts"][c] == int(np.count_nonzero(d == ord(c)))
    w0 = next(w for w in gd["windows"] if w["start"] == 0)["bytes"].encode()
    last = d[(o[1:len(w0) + 1] - 1).astype(np.int64)].tobytes()
    assert w0 == last
