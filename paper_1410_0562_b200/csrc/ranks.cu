// ranks.cu -- A3 ComputeRanks and the fused A2 + A4 step.
//
// ComputeRanks (Lemma 1, Algorithm 2): for every string
// P_j of the block, independently,
//     i := m_ext                      (reading R1; the paper prints n_ext)
//     g[offs[j] + |P_j|] := i
//     for k = |P_j|-1 .. 0:  c := P_j[k];  i := C[c] + rank(c, i, B_ext);
//                            g[offs[j] + k] := i
// One thread walks one string backwards; each LF step is one 32-byte Blk
// sector plus one superblock counter (common.cuh dict_rank).
//
// Gather (Alg.1), fused: for each SA position i,
//     s = SA_int[i];  B_int[i] = P[k-1] or '$';  pos[i] = g[s] + i
// where pos[i] = g_sa[i] + i is the final position of B_int[i] in the new
// B_ext (reading R4).
//
// g and pos are stored as u32 while the index stays below 2^32 symbols and as
// u64 beyond (G = uint32_t / uint64_t): the narrower g of one block is small
// enough to stay L2-resident between ComputeRanks and the gather.
#include <stdlib.h>

#include <algorithm>

#include "internal.h"

namespace setbwte {

template <class G>
__device__ __forceinline__ void store4(G* dst, G a, G b, G c, G d, bool keep);
template <>
__device__ __forceinline__ void store4<uint32_t>(uint32_t* dst, uint32_t a, uint32_t b, uint32_t c,
                                                 uint32_t d, bool keep) {
    // g is read back at random by the gather right after ComputeRanks: when
    // the block's g fits in L2 keep it there (evict-last; measured +1 % on
    // c2).  A larger g must NOT be pinned: its evict-last lines would crowd
    // out the bucketed gather's working set (gather.cu; measured 9 % L2 hits)
    if (keep) {
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(dst), "r"(a),
                     "r"(b), "r"(c), "r"(d), "l"(pol));
    } else {
        asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(a), "r"(b), "r"(c),
                     "r"(d));
    }
}
template <>
__device__ __forceinline__ void store4<uint64_t>(uint64_t* dst, uint64_t a, uint64_t b, uint64_t c,
                                                 uint64_t d, bool) {
    asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(dst), "l"(a), "l"(b), "l"(c),
                 "l"(d));
}

// D = const Blk* (one array) or Dict (a sharded dictionary, NEXT-3).  5 CTAs/SM
// (<= 48 registers, no spills): the LF walk is latency-bound, more warps in
// flight beat the 62-register build (c2 +2.3 %)
#ifndef SB_RANK_MINB
#define SB_RANK_MINB 5
#endif
// N5 (sigma = 5): a symbol of code 4 (nbit plane) steps through the N plane
// of the dictionary: i := C[4] + rank_n(i); B_int records it as 5.
template <class G, class D, bool N5>
__global__ void __launch_bounds__(256, SB_RANK_MINB) compute_ranks_kernel(
    const uint32_t* __restrict__ text, const uint64_t* __restrict__ slot_off, uint64_t j0,
    uint64_t j1, uint64_t slot_base, const D blk, const uint64_t* __restrict__ sb,
    const uint64_t* __restrict__ Cd, uint64_t m_ext, G* __restrict__ g, uint8_t* __restrict__ bslot,
    bool bing, const uint32_t* __restrict__ nbit, const NBlk* __restrict__ nblk,
    const uint64_t* __restrict__ nsb, bool g_keep) {
    const uint64_t C0 = Cd[0], C1 = Cd[1], C2 = Cd[2], C3 = Cd[3];
    const uint64_t C4 = N5 ? Cd[4] : 0;
    for (uint64_t j = j0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < j1;
         j += (uint64_t)gridDim.x * blockDim.x) {
        // local slot indices: [l0, le], le = terminator
        const uint64_t l0 = slot_off[j] - slot_base;
        const uint64_t le = slot_off[j + 1] - 1 - slot_base;
        uint64_t i = m_ext;
        g[le] = (G)i;
        // blocks too large for the SA payload: the walk also records B_int per
        // slot (the symbol it reads at q is B_int of the suffix at q+1; a
        // string's first suffix has '$'), so the gather reads one byte per
        // suffix instead of two random text lookups
        if (bslot) bslot[l0] = 4;
        uint64_t lp = le;  // next step computes slot lp-1
        uint64_t wi = ~0ull, nwi = ~0ull;
        uint32_t word = 0, nword = 0;
        // the symbol at global slot p: code 0..3, or 4 (sigma = 5)
        auto sym = [&](uint64_t p) -> uint32_t {
            if ((p >> 4) != wi) {
                wi = p >> 4;
                word = __ldg(text + wi);
            }
            uint32_t c = (word >> (30 - 2 * (uint32_t)(p & 15))) & 3u;
            if (N5) {
                if ((p >> 5) != nwi) {
                    nwi = p >> 5;
                    nword = __ldg(nbit + nwi);
                }
                if ((nword >> (31 - (uint32_t)(p & 31))) & 1u) c = 4u;
            }
            return c;
        };
        auto step = [&](uint64_t q) -> uint64_t {  // LF step for local slot q
            const uint64_t p = q + slot_base;
            const uint32_t c = sym(p);
            if (bslot) bslot[q + 1] = (uint8_t)(c == 4u ? 5u : c);
            if (N5 && c == 4u) {
                i = C4 + dict_rank_n(nblk, nsb, i);
            } else {
                const uint64_t Cc = c == 0 ? C0 : c == 1 ? C1 : c == 2 ? C2 : C3;
                i = Cc + dict_rank(blk, sb, c, i);
            }
            return i;
        };
        if (sizeof(G) == 8 && bing) {
            // u64 g without SA payload: B_int rides in g's top byte (g < 2^56).
            // B_int of the suffix at q+1 is the symbol read at q, so each g
            // is stored one step late, with that symbol
            uint64_t pq = le, pv = i;
            for (uint64_t q = le; q-- > l0;) {
                const uint64_t v = step(q);
                const uint32_t c = sym(q + slot_base);
                g[pq] = (G)(pv | ((uint64_t)(c == 4u ? 5u : c) << 56));
                pq = q;
                pv = v;
            }
            g[pq] = (G)(pv | (4ull << 56));  // a string's first suffix: '$'
            continue;
        }
        // single steps down to a 4-aligned local slot, then 4 steps per
        // vector store (one store instruction instead of four)
        while (lp > l0 && (lp & 3) != 0) {
            --lp;
            g[lp] = (G)step(lp);
        }
        while (lp >= l0 + 4) {
            const G a3 = (G)step(lp - 1);
            const G a2 = (G)step(lp - 2);
            const G a1 = (G)step(lp - 3);
            const G a0 = (G)step(lp - 4);
            lp -= 4;
            store4<G>(g + lp, a0, a1, a2, a3, g_keep);
        }
        while (lp > l0) {
            --lp;
            g[lp] = (G)step(lp);
        }
    }
}

cudaError_t launch_compute_ranks(Profiler& prof, cudaStream_t s, const uint32_t* text,
                                 const uint64_t* slot_off, uint64_t j0, uint64_t j1,
                                 uint64_t slot_base, const Dict& blk, const uint64_t* sb,
                                 const uint64_t* d_C, uint64_t m_ext, uint64_t n_steps, void* g,
                                 int gw, uint8_t* bslot, bool bing, const N5Dict* n5,
                                 bool one_wave) {
    if (j1 <= j0) return cudaSuccess;
    // algorithmic bytes per LF step (= base): one 32 B Blk sector + one 8 B
    // superblock counter + g write + 0.25 B packed symbol; per string: 16 B
    // slot offsets + the terminator g.  Units = LF steps.
    const uint64_t nstr = j1 - j0;
    const double bytes = (40.25 + gw) * (double)n_steps + (16.0 + gw) * (double)nstr;
    // keep g in L2 for the gather only while it fits (<= 96 MB; larger blocks use the bucketed gather)
    const bool g_keep = (double)gw * (double)(n_steps + nstr) <= 96.0 * 1024 * 1024;
    if (n5) {
        // sigma = 5 (never sharded): the plain-array kernel with the N plane
        const unsigned grid = grid_for(nstr, 256, 1u << 20);
        if (gw == 4)
            SB_LAUNCH(prof, s, "compute_ranks", bytes, n_steps,
                      (compute_ranks_kernel<uint32_t, const Blk*, true><<<grid, 256, 0, s>>>(
                          text, slot_off, j0, j1, slot_base, blk.ptr[0], sb, d_C, m_ext,
                          (uint32_t*)g, bslot, false, n5->nbit, n5->nblk, n5->nsb, g_keep)));
        else
            SB_LAUNCH(prof, s, "compute_ranks", bytes, n_steps,
                      (compute_ranks_kernel<uint64_t, const Blk*, true><<<grid, 256, 0, s>>>(
                          text, slot_off, j0, j1, slot_base, blk.ptr[0], sb, d_C, m_ext,
                          (uint64_t*)g, bslot, bing, n5->nbit, n5->nblk, n5->nsb, g_keep)));
        return cudaGetLastError();
    }
    // one_wave (a dictionary larger than L2): ONE wave of 3 CTAs per SM
    // walking the strings with the grid stride -- as fast alone as 5 resident
    // CTAs/SM (the walk is DRAM-bound), and it leaves SM slots to the sort
    // lanes' kernels beside it (c3 step 197.5 -> 188.7 ms, alternated runs).
    // An L2-resident dictionary (c2) is latency-bound: every CTA it can get.
    unsigned grid = grid_for(nstr, 256, one_wave ? 148u * 3u : 1u << 20);
    if (const char* e = getenv("SETBWTE_RANK_GRID")) grid = std::min<unsigned>(grid_for(nstr, 256, 1u << 20), (unsigned)atoi(e));
    if (gw == 4) {
        if (blk.P == 1)
            SB_LAUNCH(prof, s, "compute_ranks", bytes, n_steps,
                      (compute_ranks_kernel<uint32_t, const Blk*, false><<<grid, 256, 0, s>>>(
                          text, slot_off, j0, j1, slot_base, blk.ptr[0], sb, d_C, m_ext,
                          (uint32_t*)g, bslot, false, nullptr, nullptr, nullptr, g_keep)));
        else
            SB_LAUNCH(prof, s, "compute_ranks", bytes, n_steps,
                      (compute_ranks_kernel<uint32_t, Dict, false><<<grid, 256, 0, s>>>(
                          text, slot_off, j0, j1, slot_base, blk, sb, d_C, m_ext, (uint32_t*)g,
                          bslot, false, nullptr, nullptr, nullptr, g_keep)));
    } else {
        if (blk.P == 1)
            SB_LAUNCH(prof, s, "compute_ranks", bytes, n_steps,
                      (compute_ranks_kernel<uint64_t, const Blk*, false><<<grid, 256, 0, s>>>(
                          text, slot_off, j0, j1, slot_base, blk.ptr[0], sb, d_C, m_ext,
                          (uint64_t*)g, bslot, bing, nullptr, nullptr, nullptr, g_keep)));
        else
            SB_LAUNCH(prof, s, "compute_ranks", bytes, n_steps,
                      (compute_ranks_kernel<uint64_t, Dict, false><<<grid, 256, 0, s>>>(
                          text, slot_off, j0, j1, slot_base, blk, sb, d_C, m_ext, (uint64_t*)g,
                          bslot, bing, nullptr, nullptr, nullptr, g_keep)));
    }
    return cudaGetLastError();
}

// Fused A2 + A4 (+ the superblock slices Insert needs): pos[i], B_int[i], and
// sb_start[s] = first i with pos[i] >= s * 2^16 (the "vectorised binary
// search" of P:158 as one pass: every superblock boundary has one writer).
// U consecutive runs of blockDim elements per CTA iteration: U independent
// random g reads in flight per thread (so fewer threads keep as many reads
// in flight); a warp's lanes always hold 32 consecutive positions.
template <class G, int U>
__global__ void gather_kernel(const uint32_t* __restrict__ text, const uint32_t* __restrict__ term,
                              uint64_t slot_base, const uint32_t* __restrict__ sa,
                              const G* __restrict__ g, uint32_t n_suf, G* __restrict__ pos,
                              uint8_t* __restrict__ bint, uint64_t* __restrict__ sb_start,
                              uint64_t nsb, const uint8_t* __restrict__ bslot, bool bing,
                              uint32_t smask, const uint32_t* __restrict__ nbit) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t per = (uint64_t)U * blockDim.x;
    for (uint64_t base = blockIdx.x * per; base < n_suf; base += (uint64_t)gridDim.x * per) {
        uint32_t e[U];
        uint64_t gvv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + (uint64_t)u * blockDim.x + threadIdx.x;
            // streaming (evict-first) SA / pos / B_int accesses leave L2 to g
            e[u] = i < n_suf ? __ldcs(sa + i) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + (uint64_t)u * blockDim.x + threadIdx.x;
            SB_ASSERT(i >= n_suf || (e[u] & smask) < n_suf);
            gvv[u] = (i < n_suf && g) ? (uint64_t)__ldg(g + (e[u] & smask)) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + (uint64_t)u * blockDim.x + threadIdx.x;
            const bool v = i < n_suf;
            uint64_t pv = 0;
            if (v) {
                const uint32_t sl = e[u] & smask;
                uint64_t gv = gvv[u];
                const uint8_t bg = (uint8_t)(gv >> 56);
                if (bing) gv &= (1ull << 56) - 1ull;
                pv = gv + i;
                __stcs(pos + i, (G)pv);
                uint8_t b;
                if (bing) {
                    b = bg;  // B_int stored in g's top byte by ComputeRanks
                } else if (smask != 0xFFFFFFFFu) {
                    b = (uint8_t)(e[u] >> kPayloadShift);  // B_int carried by the SA entry
                } else if (bslot) {
                    b = __ldg(bslot + sl);  // recorded by ComputeRanks
                } else {
                    const uint64_t p = slot_base + sl;
                    if (sl == 0 || term_bit(term, p - 1)) b = 4;  // '$': suffix starts a string
                    else if (nbit && term_bit(nbit, p - 1)) b = 5;
                    else b = (uint8_t)text_sym(text, p - 1);
                }
                // B_int byte: code bits 0-1, '$' flag 4; code 4 of sigma = 5
                // (carried as 5) is stored like '$' plus the N flag 8 (NBlk)
                if (b == 5) b = 12;
                __stcs(reinterpret_cast<signed char*>(bint) + i, (signed char)b);
            }
            if (sb_start) {
                uint64_t prev = __shfl_up_sync(0xFFFFFFFFu, pv, 1);
                if (v) {
                    if (lane == 0 && i > 0) {
                        const uint32_t sl1 = sa[i - 1] & smask;
                        uint64_t g1 = g ? (uint64_t)__ldg(g + sl1) : 0ull;
                        if (bing) g1 &= (1ull << 56) - 1ull;
                        prev = g1 + (i - 1);
                    }
                    const uint64_t cur = pv >> kSbShift;
                    const uint64_t first = i > 0 ? (prev >> kSbShift) + 1 : 0;
                    for (uint64_t s = first; s <= cur && s <= nsb; ++s) sb_start[s] = i;
                    if (i + 1 == n_suf)
                        for (uint64_t s = cur + 1; s <= nsb; ++s) sb_start[s] = n_suf;
                }
            }
        }
    }
}

cudaError_t launch_gather(Profiler& prof, cudaStream_t s, const uint32_t* text,
                          const uint32_t* term, uint64_t slot_base, const uint32_t* sa,
                          const void* g, uint32_t n_suf, void* pos, int gw, uint8_t* bint,
                          uint64_t* sb_start, uint64_t nsb, const uint8_t* bslot,
                          uint64_t payload_limit, bool bing, const uint32_t* nbit) {
    const uint32_t smask = sa_slot_mask(n_suf, payload_limit);
    // bytes per suffix: 4 (SA) + gw (g) + gw (pos) + 1 (B_int) + 0.375 (symbol
    // + term bit); when g does not fit in L2 (> 96 MB) the random g read is
    // one 32-byte sector ("44 B at 32 B-sector granularity if
    // g misses L2"; the same convention as ComputeRanks' Blk reads)
    const bool g_l2 = (double)gw * n_suf <= 96.0 * 1024 * 1024;
    const double bytes = (5.375 + (g_l2 ? (double)gw : 32.0) + gw) * n_suf;
    // (U = 2 or 4 reads in flight per thread with a 2-8x smaller grid measured
    // slower on c3: 45-48 vs 42.3 ms)
    const unsigned grid = grid_for(n_suf, 256, 148u * 64u);
    if (gw == 4)
        SB_LAUNCH(prof, s, "gather", bytes, n_suf,
                  (gather_kernel<uint32_t, 1><<<grid, 256, 0, s>>>(
                      text, term, slot_base, sa, (const uint32_t*)g, n_suf, (uint32_t*)pos, bint,
                      sb_start, nsb, bslot, false, smask, nbit)));
    else
        SB_LAUNCH(prof, s, "gather", bytes, n_suf,
                  (gather_kernel<uint64_t, 1><<<grid, 256, 0, s>>>(
                      text, term, slot_base, sa, (const uint64_t*)g, n_suf, (uint64_t*)pos, bint,
                      sb_start, nsb, bslot, bing, smask, nbit)));
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// BWT merge ("the same LF/insert machinery with B_int
// given"): the strings of a second index O are added after those of the
// index H.  O's own BWT is B_int in O's row order; g_sa[r] (the number of
// H-suffixes smaller than O's suffix at row r) follows from walking every
// string of O backwards in both indexes at once (Lemma 1 P:95-100 applied
// to O for the row and to H for the rank):
//     r := j (row of $_j in O);  g := m_H;  g_sa[r] := g
//     while O.B[r] != '$':  c := O.B[r];  r := C_O[c] + rank_O(c, r);
//                           g := C_H[c] + rank_H(c, g);  g_sa[r] := g
// Every row of O is visited once; then pos[r] = g_sa[r] + r as in Alg.1.
template <class G>
__global__ void __launch_bounds__(256) merge_ranks_kernel(
    const Blk* __restrict__ oblk, const uint64_t* __restrict__ osb, const uint64_t* __restrict__ oC,
    uint64_t m_o, const Blk* __restrict__ hblk, const uint64_t* __restrict__ hsb,
    const uint64_t* __restrict__ hC, uint64_t init, G* __restrict__ gsa) {
    const uint64_t hC0 = hblk ? hC[0] : 0, hC1 = hblk ? hC[1] : 0, hC2 = hblk ? hC[2] : 0,
                   hC3 = hblk ? hC[3] : 0;
    const uint64_t oC0 = oC[0], oC1 = oC[1], oC2 = oC[2], oC3 = oC[3];
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < m_o;
         j += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = j, g = init;
        gsa[r] = (G)g;
        for (;;) {
            uint64_t w0, w1, w2, w3;
            asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3)
                : "l"(oblk + (r >> 6)));
            const uint32_t bit = (uint32_t)(r & 63);
            if ((w3 >> bit) & 1ull) break;  // '$': row of the string's first suffix
            const uint32_t c = (uint32_t)((w1 >> bit) & 1ull) | ((uint32_t)((w2 >> bit) & 1ull) << 1);
            const uint64_t ro = __ldg(osb + ((r >> kSbShift) << 2) + c) +
                                ((w0 >> (16 * c)) & 0xFFFFull) +
                                (uint64_t)__popcll(match_plane(c, w1, w2, w3) & ((1ull << bit) - 1ull));
            r = (c == 0 ? oC0 : c == 1 ? oC1 : c == 2 ? oC2 : oC3) + ro;
            g = hblk ? (c == 0 ? hC0 : c == 1 ? hC1 : c == 2 ? hC2 : hC3) + dict_rank(hblk, hsb, c, g)
                     : 0ull;
            gsa[r] = (G)g;
        }
    }
}

// pos[r] = g_sa[r] + r, B_int[r] = O.B[r] (code | '$' flag) and the superblock
// slices of pos (as in gather_kernel).
template <class G>
__global__ void merge_pos_kernel(const Blk* __restrict__ oblk, uint64_t n_o, const G* __restrict__ gsa,
                                 G* __restrict__ pos, uint8_t* __restrict__ bint,
                                 uint64_t* __restrict__ sb_start, uint64_t nsb) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t iters = (n_o + stride - 1) / stride;
    for (uint64_t it = 0; it < iters; ++it) {
        const uint64_t i = it * stride + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
        const bool v = i < n_o;
        uint64_t pv = 0;
        if (v) {
            pv = (uint64_t)__ldcs(gsa + i) + i;
            __stcs(pos + i, (G)pv);
            const Blk* b = oblk + (i >> 6);
            const uint32_t bit = (uint32_t)(i & 63);
            const uint64_t lo = __ldg(&b->lo), hi = __ldg(&b->hi), dol = __ldg(&b->dol);
            const uint8_t sym = ((dol >> bit) & 1ull)
                                    ? (uint8_t)4
                                    : (uint8_t)(((lo >> bit) & 1ull) | (((hi >> bit) & 1ull) << 1));
            bint[i] = sym;
        }
        uint64_t prev = __shfl_up_sync(0xFFFFFFFFu, pv, 1);
        if (v) {
            if (lane == 0 && i > 0) prev = (uint64_t)gsa[i - 1] + (i - 1);
            const uint64_t cur = pv >> kSbShift;
            const uint64_t first = i > 0 ? (prev >> kSbShift) + 1 : 0;
            for (uint64_t s = first; s <= cur && s <= nsb; ++s) sb_start[s] = i;
            if (i + 1 == n_o)
                for (uint64_t s = cur + 1; s <= nsb; ++s) sb_start[s] = n_o;
        }
    }
}

cudaError_t launch_merge_ranks(Profiler& prof, cudaStream_t s, const Blk* oblk, const uint64_t* osb,
                               const uint64_t* oC, uint64_t m_o, uint64_t n_o, const Blk* hblk,
                               const uint64_t* hsb, const uint64_t* hC, uint64_t init, void* gsa,
                               int gw) {
    if (m_o == 0) return cudaSuccess;
    // per LF step: two Blk sectors + two superblock counters + the g_sa write
    const double bytes = (80.0 + gw) * (double)(n_o - m_o) + (double)gw * m_o;
    const unsigned grid = grid_for(m_o, 256, 1u << 20);
    if (gw == 4) {
        SB_LAUNCH(prof, s, "merge_ranks", bytes, n_o - m_o,
                  merge_ranks_kernel<uint32_t><<<grid, 256, 0, s>>>(oblk, osb, oC, m_o, hblk, hsb, hC,
                                                                    init, (uint32_t*)gsa));
    } else {
        SB_LAUNCH(prof, s, "merge_ranks", bytes, n_o - m_o,
                  merge_ranks_kernel<uint64_t><<<grid, 256, 0, s>>>(oblk, osb, oC, m_o, hblk, hsb, hC,
                                                                    init, (uint64_t*)gsa));
    }
    return cudaGetLastError();
}

cudaError_t launch_merge_pos(Profiler& prof, cudaStream_t s, const Blk* oblk, uint64_t n_o,
                             const void* gsa, void* pos, int gw, uint8_t* bint, uint64_t* sb_start,
                             uint64_t nsb) {
    if (n_o == 0) return cudaSuccess;
    const double bytes = (2.0 * gw + 1.0 + 0.5) * (double)n_o;
    const unsigned grid = grid_for(n_o, 256, 148u * 64u);
    if (gw == 4) {
        SB_LAUNCH(prof, s, "merge_pos", bytes, n_o,
                  merge_pos_kernel<uint32_t><<<grid, 256, 0, s>>>(oblk, n_o, (const uint32_t*)gsa,
                                                                  (uint32_t*)pos, bint, sb_start, nsb));
    } else {
        SB_LAUNCH(prof, s, "merge_pos", bytes, n_o,
                  merge_pos_kernel<uint64_t><<<grid, 256, 0, s>>>(oblk, n_o, (const uint64_t*)gsa,
                                                                  (uint64_t*)pos, bint, sb_start, nsb));
    }
    return cudaGetLastError();
}

}  // namespace setbwte
