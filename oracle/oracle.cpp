/*
 * oracle.cpp -- the plain, slow, obviously-correct CPU ORACLE for set-bwte
 * (arXiv 1410.0562).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1410_0562_b200/) never imports, links or executes anything here, and
 * this file shares no code, header, table or constant with the CUDA path.
 *
 * Every function states the passage of /root/reference/PAPER.md ("P:<line>")
 * it writes out.  Readings of the paper (where it is silent or at odds with
 * itself) are the ones listed in DESIGN.md section "Readings".
 *
 * Problem statement (Sec.2): the BWT of a string set S_0..S_{m-1}
 * over an ordered alphabet c_1 < ... < c_sigma is the BWT of
 *     T = S_0 $_0 S_1 $_1 ... S_{m-1} $_{m-1},   $_0 < ... < $_{m-1} < c_1,
 * with B[i] = T[(SA[i]-1) mod n] (Eq.(1)).  Output collapses every
 * $_j to the byte '$' (reading R5).
 *
 * Input convention for every entry point: `alphabet` is a NUL-terminated
 * string of distinct bytes in increasing symbol order (e.g. "ACGT"); a byte
 * maps to its index in `alphabet`, case-insensitively.  String j is
 * bytes[off[j] .. off[j+1]).  Return value 0 = OK, -1 = invalid argument,
 * -2 = a byte not in the alphabet (its global byte position is written to
 * *bad_pos when bad_pos != NULL).
 *
 * Parity status of each function is listed in DESIGN.md "Oracle pins".
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <ctype.h>
#include <vector>
#include <algorithm>
#include <parallel/algorithm>
#include <omp.h>

namespace {

/* A suffix of T, identified by its string (global index) and its offset k in
 * that string, 0 <= k <= |S_j| (k == |S_j| is the terminator suffix $_j). */
struct Suf {
    uint32_t j;
    uint32_t k;
};

struct Text {
    std::vector<int16_t> code;   /* symbol code per input byte, 1..sigma */
    const uint64_t* off;         /* string j = code[off[j] .. off[j+1]) */
    uint64_t m;
};

/* Map bytes to codes 1..sigma (0 is reserved for terminators, which are never
 * stored: they are implied by the string ends). */
int encode(const char* alphabet, const uint8_t* bytes, const uint64_t* off,
           uint64_t m, Text* t, uint64_t* bad_pos) {
    if (!alphabet || !off) return -1;
    int16_t map[256];
    for (int i = 0; i < 256; ++i) map[i] = -1;
    int sigma = (int)strlen(alphabet);
    if (sigma < 1 || sigma > 255) return -1;
    for (int i = 0; i < sigma; ++i) {
        unsigned char ch = (unsigned char)alphabet[i];
        if (ch == '$') return -1;
        int16_t code = (int16_t)(i + 1);
        if (map[toupper(ch)] != -1 && map[toupper(ch)] != code) return -1;
        map[toupper(ch)] = code;
        map[tolower(ch)] = code;
    }
    uint64_t nbytes = off[m];
    for (uint64_t j = 0; j < m; ++j)
        if (off[j] > off[j + 1]) return -1;
    if (off[0] != 0) return -1;
    t->code.resize(nbytes);
    for (uint64_t p = 0; p < nbytes; ++p) {
        int16_t c = map[bytes[p]];
        if (c < 0) {
            if (bad_pos) *bad_pos = p;
            return -2;
        }
        t->code[p] = c;
    }
    t->off = off;
    t->m = m;
    return 0;
}

inline uint64_t len_of(const Text& t, uint32_t j) { return t.off[j + 1] - t.off[j]; }

/* Symbol at offset k of string j, as an integer of the ordered alphabet
 * {$ (any) < c_1 < ... < c_sigma}: 0 stands for "the terminator $_j". */
inline int sym_at(const Text& t, uint32_t j, uint64_t k) {
    return k == len_of(t, j) ? 0 : t.code[t.off[j] + k];
}

/* Lexicographic comparison of two suffixes of T.
 * Walk both suffixes symbol by symbol.  The first terminator met decides:
 * a terminator is smaller than every real symbol, and two terminators
 * $_a, $_b compare by string index a < b.  Because all terminators are
 * distinct, a comparison never reaches past a terminator, so walking inside
 * one string each is the same as comparing the two suffixes of T.
 * (reading R6; pinned by tests/test_oracle_pins.py against a
 * brute force over the materialised integer text T.) */
inline bool suf_less(const Text& t, const Suf& a, const Suf& b) {
    uint64_t ka = a.k, kb = b.k;
    for (;;) {
        int x = sym_at(t, a.j, ka);
        int y = sym_at(t, b.j, kb);
        if (x == 0 && y == 0) return a.j < b.j;
        if (x != y) return x < y;
        ++ka;
        ++kb;
    }
}

void sort_sufs(const Text& t, std::vector<Suf>& v, int threads) {
    auto cmp = [&t](const Suf& a, const Suf& b) { return suf_less(t, a, b); };
    if (threads > 1) {
        omp_set_num_threads(threads);
        __gnu_parallel::sort(v.begin(), v.end(), cmp);
    } else {
        std::sort(v.begin(), v.end(), cmp);
    }
}

/* All suffixes of strings [j0, j1), in string-major "slot" order:
 * slot(j,k) = sum_{j'<j}(|S_j'|+1) + k  (Alg.2, reading R2). */
std::vector<Suf> all_suffixes(const Text& t, uint32_t j0, uint32_t j1) {
    std::vector<Suf> v;
    uint64_t n = 0;
    for (uint32_t j = j0; j < j1; ++j) n += len_of(t, j) + 1;
    v.reserve(n);
    for (uint32_t j = j0; j < j1; ++j)
        for (uint64_t k = 0; k <= len_of(t, j); ++k) v.push_back(Suf{j, (uint32_t)k});
    return v;
}

}  // namespace

extern "C" {

/* Total suffix count n = sum(|S_j|+1) (P:57 as a count, reading R3). */
uint64_t oracle_num_suffixes(const uint64_t* off, uint64_t m) { return off[m] + m; }

/* One-shot BWT of the string set, Eq.(1) P:33-35 with T as in P:36-37.
 * out receives n = off[m] + m bytes; every terminator is written '$'. */
int oracle_bwt(const char* alphabet, const uint8_t* bytes, const uint64_t* off, uint64_t m,
               uint8_t* out, int threads, uint64_t* bad_pos) {
    Text t;
    int rc = encode(alphabet, bytes, off, m, &t, bad_pos);
    if (rc) return rc;
    if (m >= 0xffffffffull) return -1;
    std::vector<Suf> sa = all_suffixes(t, 0, (uint32_t)m);
    sort_sufs(t, sa, threads);
    /* B[i] = T[(SA[i]-1) mod n]: the symbol before suffix (j,k) is S_j[k-1]
     * when k > 0, else the terminator that precedes S_j in T ($_{j-1}, or
     * $_{m-1} by the wrap-around when j = 0). */
    for (uint64_t i = 0; i < sa.size(); ++i) {
        const Suf& s = sa[i];
        out[i] = s.k > 0 ? bytes[off[s.j] + s.k - 1] : (uint8_t)'$';
    }
    /* Upper-case output: the alphabet's own byte for each code. */
    for (uint64_t i = 0; i < sa.size(); ++i) {
        if (out[i] == '$') continue;
        out[i] = (uint8_t)alphabet[t.code[off[sa[i].j] + sa[i].k - 1] - 1];
    }
    return 0;
}

/* The same one-shot BWT (Eq.(1) P:33-35 on T of P:36-37) in a BUCKETED,
 * low-memory mode (SURVEY.md section 8(c) "Bucketed mode"), for sets whose
 * suffix ids do not fit in RAM at once (configs c3-c5, up to 6 G suffixes).
 *
 *   1. Every suffix (j,k) gets a bucket key: its first h symbols as the digits
 *      of a base-(sigma+1) number, the terminator and every position after it
 *      written as digit 0 (the smallest symbol).  If two suffixes have
 *      different keys, the first differing digit is a position where both are
 *      still inside their strings, or where exactly one of them meets its
 *      terminator; either way suf_less decides the same way as the keys.  So
 *      bucket order is suffix order, and sorting each bucket with suf_less
 *      and emitting the buckets in key order is the full sort.
 *   2. Count the members of every bucket (one pass over all suffixes).
 *   3. Take the buckets in key order, as many as fit in `batch_cap` suffixes
 *      (at least one), collect their members, sort each bucket with suf_less
 *      (the library sort, as in oracle_bwt) and emit B for it (Eq.(1)).
 *
 * Output: `emit(chunk, len, bucket_key, ctx)` is called once per non-empty
 * bucket, in order; the concatenation of the chunks is oracle_bwt's output.
 * Memory: the codes of the text plus batch_cap * 9 bytes.  The buckets of a
 * batch are sorted in parallel (a library sort each); their order is fixed by
 * the keys, so the schedule does not change the output. */
typedef void (*oracle_emit_fn)(const uint8_t* chunk, uint64_t len, uint64_t bucket, void* ctx);

int oracle_bwt_bucketed(const char* alphabet, const uint8_t* bytes, const uint64_t* off,
                        uint64_t m, int h, uint64_t batch_cap, oracle_emit_fn emit, void* ctx,
                        int threads, uint64_t* bad_pos) {
    if (h < 1 || h > 8 || !emit || batch_cap == 0) return -1;
    Text t;
    int rc = encode(alphabet, bytes, off, m, &t, bad_pos);
    if (rc) return rc;
    if (m >= 0xffffffffull) return -1;
    const uint64_t base = (uint64_t)strlen(alphabet) + 1;
    uint64_t nb = 1;
    for (int d = 0; d < h; ++d) nb *= base;
    if (nb > (1ull << 24)) return -1;
    if (threads < 1) threads = 1;
    auto key_of = [&](uint32_t j, uint64_t k) {
        const uint64_t L = len_of(t, j);
        uint64_t key = 0;
        for (int d = 0; d < h; ++d) {
            const uint64_t p = k + (uint64_t)d;
            const uint64_t x = p < L ? (uint64_t)t.code[t.off[j] + p] : 0; /* $ and after */
            key = key * base + x;
        }
        return key;
    };
    /* 2. bucket sizes, per thread (static schedule: the same string ranges
     *    per thread in every pass below). */
    std::vector<std::vector<uint64_t>> cnt(threads, std::vector<uint64_t>(nb, 0));
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t j = 0; j < (int64_t)m; ++j) {
        std::vector<uint64_t>& c = cnt[omp_get_thread_num()];
        const uint64_t L = len_of(t, (uint32_t)j);
        for (uint64_t k = 0; k <= L; ++k) ++c[key_of((uint32_t)j, k)];
    }
    std::vector<uint64_t> total(nb, 0);
    for (int th = 0; th < threads; ++th)
        for (uint64_t b = 0; b < nb; ++b) total[b] += cnt[th][b];
    std::vector<Suf> v;
    std::vector<uint8_t> out;
    for (uint64_t b0 = 0; b0 < nb;) {
        /* 3. the batch [b0, b1) */
        uint64_t b1 = b0, size = 0;
        while (b1 < nb && (b1 == b0 || size + total[b1] <= batch_cap)) size += total[b1++];
        if (size == 0) { b0 = b1; continue; }
        /* where each thread writes each bucket's members inside the batch */
        std::vector<uint64_t> start(b1 - b0 + 1, 0);
        for (uint64_t b = b0; b < b1; ++b) start[b - b0 + 1] = start[b - b0] + total[b];
        std::vector<std::vector<uint64_t>> wr(threads, std::vector<uint64_t>(b1 - b0));
        for (uint64_t b = b0; b < b1; ++b) {
            uint64_t acc = start[b - b0];
            for (int th = 0; th < threads; ++th) { wr[th][b - b0] = acc; acc += cnt[th][b]; }
        }
        v.assign(size, Suf{0, 0});
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t j = 0; j < (int64_t)m; ++j) {
            std::vector<uint64_t>& w = wr[omp_get_thread_num()];
            const uint64_t L = len_of(t, (uint32_t)j);
            for (uint64_t k = 0; k <= L; ++k) {
                const uint64_t key = key_of((uint32_t)j, k);
                if (key >= b0 && key < b1) v[w[key - b0]++] = Suf{(uint32_t)j, (uint32_t)k};
            }
        }
        out.resize(size);
        /* sort every bucket of the batch with the library sort: the buckets
         * in parallel (one thread each), a bucket holding more than a quarter
         * of the batch with the parallel library sort */
        auto cmp = [&t](const Suf& a, const Suf& b) { return suf_less(t, a, b); };
        std::vector<uint64_t> big;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
        for (int64_t b = (int64_t)b0; b < (int64_t)b1; ++b) {
            const uint64_t s0 = start[b - b0], s1 = start[b - b0 + 1];
            if (s1 - s0 > size / 4 && threads > 1) {
#pragma omp critical
                big.push_back((uint64_t)b);
                continue;
            }
            std::sort(v.begin() + s0, v.begin() + s1, cmp);
        }
        for (uint64_t b : big) {
            omp_set_num_threads(threads);
            __gnu_parallel::sort(v.begin() + start[b - b0], v.begin() + start[b - b0 + 1], cmp);
        }
        /* B[i] = T[(SA[i]-1) mod n], Eq.(1): S_j[k-1] if k > 0, else '$' */
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < (int64_t)size; ++i) {
            const Suf& s = v[i];
            out[i] = s.k > 0 ? (uint8_t)alphabet[t.code[off[s.j] + s.k - 1] - 1] : (uint8_t)'$';
        }
        for (uint64_t b = b0; b < b1; ++b) {
            const uint64_t s0 = start[b - b0], s1 = start[b - b0 + 1];
            if (s0 != s1) emit(out.data() + s0, s1 - s0, b, ctx);
        }
        b0 = b1;
    }
    return 0;
}

/* ConstructSA of one block (Alg.1): the block's strings are sorted among
 * themselves only, terminators ordered by string index.  sa_out
 * receives n_suf slot ids, slot(j,k) = off[j] + j + k (string-major layout,
 * reading R2). */
int oracle_block_sa(const char* alphabet, const uint8_t* bytes, const uint64_t* off, uint64_t m,
                    uint64_t* sa_out, int threads, uint64_t* bad_pos) {
    Text t;
    int rc = encode(alphabet, bytes, off, m, &t, bad_pos);
    if (rc) return rc;
    std::vector<Suf> sa = all_suffixes(t, 0, (uint32_t)m);
    sort_sufs(t, sa, threads);
    for (uint64_t i = 0; i < sa.size(); ++i) sa_out[i] = off[sa[i].j] + sa[i].j + sa[i].k;
    return 0;
}

/* B_int := B(S_jk, SA_int) (Alg.1): for SA entry (j,k) the symbol
 * S_j[k-1] when k > 0, else '$'.  Takes the slot ids oracle_block_sa wrote. */
int oracle_block_bint(const char* alphabet, const uint8_t* bytes, const uint64_t* off, uint64_t m,
                      const uint64_t* sa, uint8_t* bint_out, uint64_t* bad_pos) {
    Text t;
    int rc = encode(alphabet, bytes, off, m, &t, bad_pos);
    if (rc) return rc;
    uint64_t n = off[m] + m;
    /* slot -> (j, k) by walking the string-major layout */
    std::vector<uint32_t> str_of(n);
    std::vector<uint32_t> k_of(n);
    for (uint64_t j = 0; j < m; ++j)
        for (uint64_t k = 0; k <= off[j + 1] - off[j]; ++k) {
            str_of[off[j] + j + k] = (uint32_t)j;
            k_of[off[j] + j + k] = (uint32_t)k;
        }
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t s = sa[i];
        if (s >= n) return -1;
        uint32_t j = str_of[s], k = k_of[s];
        bint_out[i] = k > 0 ? (uint8_t)alphabet[t.code[off[j] + k - 1] - 1] : (uint8_t)'$';
    }
    return 0;
}

/* ComputeRanks, by its definition rather than by Alg.2: g[slot(j,k)] is the
 * number of suffixes already in B_ext that are lexicographically smaller than
 * the new suffix (j,k) ("suffix P^k is lexicographically
 * larger than precisely i suffixes in B_ext").  The external strings are the
 * first m_ext strings of the set (global indices 0..m_ext-1), the block's
 * strings follow them (indices m_ext..); both are given as one string set of
 * m_ext + m_blk strings.  g_out receives sum_{block}(|P|+1) u64 values in the
 * block's slot order.  Implementation: sort all ext+block suffixes together
 * and count the external ones passed. */
int oracle_compute_ranks(const char* alphabet, const uint8_t* bytes, const uint64_t* off,
                         uint64_t m_ext, uint64_t m_blk, uint64_t* g_out, int threads,
                         uint64_t* bad_pos) {
    Text t;
    uint64_t m = m_ext + m_blk;
    int rc = encode(alphabet, bytes, off, m, &t, bad_pos);
    if (rc) return rc;
    std::vector<Suf> all = all_suffixes(t, 0, (uint32_t)m);
    sort_sufs(t, all, threads);
    uint64_t slot_base = off[m_ext] + m_ext; /* first slot of the block */
    uint64_t ext_seen = 0;
    for (const Suf& s : all) {
        if (s.j < m_ext) {
            ++ext_seen;
        } else {
            uint64_t slot = off[s.j] + s.j + s.k - slot_base;
            g_out[slot] = ext_seen;
        }
    }
    return 0;
}

/* rank(c,k,B) = |{i < k : B[i] = c}|, Eq.(2), by a literal scan. */
uint64_t oracle_rank(const uint8_t* B, uint64_t n, uint8_t c, uint64_t k) {
    if (k > n) k = n;
    uint64_t r = 0;
    for (uint64_t i = 0; i < k; ++i) r += (B[i] == c);
    return r;
}

/* Insert(B_int, g_sa, B_ext) (Alg.1, Sec.5): for i in order,
 * insert B_int[i] into the growing flat sequence at absolute position
 * g_sa[i] + i (reading R4: g_sa counts external suffixes only, and the i
 * symbols already inserted before it shift it by i; equal g_sa keep SA order).
 * A literal list insertion with memmove.  out has room for n_ext + n_suf. */
int oracle_insert(const uint8_t* b_ext, uint64_t n_ext, const uint8_t* b_int,
                  const uint64_t* g_sa, uint64_t n_suf, uint8_t* out) {
    memcpy(out, b_ext, n_ext);
    uint64_t cur = n_ext;
    for (uint64_t i = 0; i < n_suf; ++i) {
        uint64_t p = g_sa[i] + i;
        if (p > cur) return -1;
        memmove(out + p + 1, out + p, cur - p);
        out[p] = b_int[i];
        ++cur;
    }
    return 0;
}

/* Rank of one suffix (j,k) of T among all n suffixes: the number of suffixes
 * smaller than it (the definition of its SA position).  Used to check
 * sampled BWT positions at sizes where a full sort is too slow:
 * B[rank(j,k)] must equal the symbol preceding (j,k) (Eq.(1)). */
int oracle_suffix_rank(const char* alphabet, const uint8_t* bytes, const uint64_t* off, uint64_t m,
                       uint64_t j, uint64_t k, uint64_t* rank_out, int threads, uint64_t* bad_pos) {
    Text t;
    int rc = encode(alphabet, bytes, off, m, &t, bad_pos);
    if (rc) return rc;
    if (j >= m || k > off[j + 1] - off[j]) return -1;
    Suf q{(uint32_t)j, (uint32_t)k};
    uint64_t cnt = 0;
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) reduction(+ : cnt) schedule(dynamic, 1024)
    for (int64_t jj = 0; jj < (int64_t)m; ++jj) {
        uint64_t L = off[jj + 1] - off[jj];
        for (uint64_t kk = 0; kk <= L; ++kk)
            cnt += suf_less(t, Suf{(uint32_t)jj, (uint32_t)kk}, q) ? 1 : 0;
    }
    *rank_out = cnt;
    return 0;
}

/* Occurrences of each pattern as a substring of the strings, every offset
 * counted (the definition the FM-index count answers; SPEC's
 * naive_count_occurrences).  Literal comparison at every start position; a
 * match never spans two strings.  Case-insensitive like the rest. */
int oracle_count(const char* alphabet, const uint8_t* bytes, const uint64_t* off, uint64_t m,
                 const uint8_t* pat, const uint64_t* poff, uint64_t q, uint64_t* out,
                 int threads) {
    if (!alphabet || !off || !poff || !out) return -1;
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
    for (int64_t t = 0; t < (int64_t)q; ++t) {
        const uint64_t pl = poff[t + 1] - poff[t];
        uint64_t cnt = 0;
        if (pl == 0) {
            cnt = off[m] + m;  /* the empty pattern: every suffix (reading of SETBWTE docs) */
        } else {
            for (uint64_t j = 0; j < m; ++j) {
                const uint64_t L = off[j + 1] - off[j];
                for (uint64_t a = 0; a + pl <= L; ++a) {
                    uint64_t k = 0;
                    while (k < pl && toupper(bytes[off[j] + a + k]) == toupper(pat[poff[t] + k])) ++k;
                    cnt += (k == pl);
                }
            }
        }
        out[t] = cnt;
    }
    return 0;
}

}  /* extern "C" */
