"""Brute-force models used to PIN the oracle (tests only).

These are deliberately different computations from oracle.cpp:

* the string set is materialised as the integer text
  T = S_0 $_0 ... S_{m-1} $_{m-1} with $_j -> j and c -> m + code(c)
  (so $_0 < ... < $_{m-1} < c_1), and suffixes of T are compared as
  whole Python tuples -- no "stop at the first terminator" shortcut;
* the single-string case uses the textbook rotation definition of the BWT
  (sort all rotations of S$, take the last column);
* Algorithm 1 / Algorithm 2 are transcribed step by step (P:54-76,
  P:106-123), ranks by a literal count over the flat B_ext.
"""
from __future__ import annotations


def int_text(strings, alphabet="ACGT"):
    m = len(strings)
    code = {ch: i + 1 for i, ch in enumerate(alphabet)}
    T = []
    owner = []
    for j, s in enumerate(strings):
        for k, ch in enumerate(s):
            T.append(m + code[ch.upper()])
            owner.append((j, k))
        T.append(j)
        owner.append((j, len(s)))
    return T, owner


def brute_bwt(strings, alphabet="ACGT"):
    """Eq.(1) B[i] = T[(SA[i]-1) mod n] over the materialised integer text."""
    T, _ = int_text(strings, alphabet)
    n = len(T)
    if n == 0:
        return ""
    Tt = tuple(T)
    sa = sorted(range(n), key=lambda p: Tt[p:])
    m = len(strings)
    out = []
    for p in sa:
        x = T[(p - 1) % n]
        out.append("$" if x < m else alphabet[x - m - 1])
    return "".join(out)


def brute_sa_jk(strings, alphabet="ACGT"):
    """SA of the set as (string, offset) pairs (full-suffix tuple comparison)."""
    T, owner = int_text(strings, alphabet)
    Tt = tuple(T)
    sa = sorted(range(len(T)), key=lambda p: Tt[p:])
    return [owner[p] for p in sa]


def rotation_bwt(s, alphabet="ACGT"):
    """Textbook BWT of one string: last column of the sorted rotations of s$."""
    order = {"$": 0}
    order.update({ch: i + 1 for i, ch in enumerate(alphabet)})
    t = s + "$"
    rots = sorted((t[i:] + t[:i] for i in range(len(t))), key=lambda r: [order[c] for c in r])
    return "".join(r[-1] for r in rots)


def brute_g(ext, block, alphabet="ACGT"):
    """g[slot] = number of external suffixes smaller than each new suffix,
    by pairwise comparison of suffixes of the materialised T (ext then block)."""
    strings = list(ext) + list(block)
    T, owner = int_text(strings, alphabet)
    Tt = tuple(T)
    n_ext = sum(len(s) + 1 for s in ext)
    ext_pos = range(n_ext)
    g = []
    for q in range(n_ext, len(T)):
        g.append(sum(1 for p in ext_pos if Tt[p:] < Tt[q:]))
    return g


def count_before(B, c, i):
    return sum(1 for x in B[:i] if x == c)


def C_array(B, alphabet="ACGT"):
    order = "$" + alphabet
    C = {}
    acc = 0
    for ch in order:
        C[ch] = acc
        acc += sum(1 for x in B if x == ch)
    return C


def alg2_compute_ranks(block, B_ext, m_ext, alphabet="ACGT"):
    """Algorithm 2 with i := m_ext (reading R1) and slot =
    offs[j] + k (reading R2); rank by literal count (Eq.(2))."""
    C = C_array(B_ext, alphabet)
    g = []
    for P in block:
        row = [0] * (len(P) + 1)
        k = len(P)
        i = m_ext
        row[k] = i
        while k > 0:
            k -= 1
            c = P[k].upper()
            i = C[c] + count_before(B_ext, c, i)
            row[k] = i
        g.extend(row)
    return g


def slot_jk(block):
    out = []
    for j, P in enumerate(block):
        for k in range(len(P) + 1):
            out.append((j, k))
    return out


def alg1_incremental(blocks, alphabet="ACGT", sa_fn=None):
    """Algorithm 1 with every step written naively:
    SA_int by brute-force sort of the block alone, B_int by P:63,
    g by Algorithm 2, g_sa by the gather of P:70, Insert at g_sa[i]+i."""
    B_ext = ""
    m_ext = 0
    for block in blocks:
        jk = brute_sa_jk(block, alphabet) if sa_fn is None else sa_fn(block)
        slots = slot_jk(block)
        slot_of = {p: s for s, p in enumerate(slots)}
        sa = [slot_of[p] for p in jk]
        b_int = "".join(block[j][k - 1].upper() if k > 0 else "$" for (j, k) in jk)
        g = alg2_compute_ranks(block, B_ext, m_ext, alphabet)
        g_sa = [g[s] for s in sa]
        out = list(B_ext)
        for i, (x, sym) in enumerate(zip(g_sa, b_int)):
            out.insert(x + i, sym)
        B_ext = "".join(out)
        m_ext += len(block)
    return B_ext


def lf_invert(B, m, alphabet="ACGT"):
    """Recover every string from the BWT: row j (< m) is suffix $_j, so
    walking LF backwards from it spells S_j reversed (FM-index LF)."""
    C = C_array(B, alphabet)
    out = []
    for j in range(m):
        i = j
        s = []
        while B[i] != "$":
            c = B[i]
            s.append(c)
            i = C[c] + count_before(B, c, i)
        out.append("".join(reversed(s)))
    return out


def naive_count(pattern, strings):
    total = 0
    for s in strings:
        for a in range(len(s) - len(pattern) + 1):
            if s[a:a + len(pattern)] == pattern:
                total += 1
    return total
