// insert.cu -- A5 Insert + rebuild of the B_ext rank dictionary, plus the
// query kernels (Eq.(2) rank, BWT decode).
//
// Insert (Alg.1, Sec.5): the new sequence B_ext' has
// n_out = n_in + n_ins symbols; output position o holds B_int[i] when
// o = pos[i] (= g_sa[i] + i, strictly increasing, reading R4) and otherwise
// the next B_ext symbol in order.  The paper's paged array with a vectorised
// binary search over page offsets becomes a flat merge: one CTA
// per 2^16-symbol output superblock binary-searches its slice of pos[] once,
// counts inserted symbols per 64-symbol output word in shared memory, and one
// warp per word merges the inserted symbols with a funnel-shifted window of
// the old planes, building the new planes with __ballot_sync.  The same CTA
// writes the u16 in-superblock counters ("sampled relative counters")
// and its superblock totals; a second kernel scans the totals into the u64
// superblock counters ("global counters") and C (Lemma 1).
#include <stdlib.h>

#include <algorithm>

#include "internal.h"

namespace setbwte {

namespace {
constexpr int kInsNt = 1024;  // one thread per output word of a superblock
static_assert(kInsNt == kBlkPerSb, "insert: one thread per Blk of the superblock");
constexpr int kInsWarps = kInsNt / 32;

template <class G>
__device__ __forceinline__ uint64_t lower_bound_g(const G* __restrict__ a, uint64_t n, uint64_t x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint64_t funnel(uint64_t a, uint64_t b, uint32_t sh) {
    return sh == 0 ? a : (a >> sh) | (b << (64 - sh));
}
}  // namespace

// Inclusive warp scan.
__device__ __forceinline__ uint32_t warp_incl(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= (uint32_t)o) v += y;
    }
    return v;
}

// Merge one 64-symbol output word: the inserted symbols (offset t in the word,
// code+$ bits b) in order, the external symbols (window x*, 64 consecutive
// external symbols) filling the other positions; one 32-symbol half at a time
// so every shift is 32-bit.  STAGED: entries come from shared memory.
// N5 (sigma = 5): a fourth plane (xn / oo[.][3]) for the code-4 flag (B_int bit 3).
template <bool STAGED, class G, bool N5 = false>
__device__ __forceinline__ void merge_word(uint32_t (&oo)[2][4], uint64_t xl, uint64_t xh,
                                           uint64_t xd, uint64_t xn, uint32_t lim, uint32_t cnt,
                                           const uint16_t* ent, const G* __restrict__ pos,
                                           const uint8_t* __restrict__ bint, uint64_t a,
                                           uint64_t ow0) {
    uint32_t k = 0, used = 0;  // inserted consumed, external bits consumed
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
        const uint32_t base = 32u * hf;
        const uint32_t wl = (uint32_t)(xl >> used), wh = (uint32_t)(xh >> used),
                       wd = (uint32_t)(xd >> used), wn = N5 ? (uint32_t)(xn >> used) : 0u;
        uint32_t al = 0, ah = 0, ad = 0, an = 0, filled = 0, u = 0;
        const uint32_t hl = lim > base ? min(lim - base, 32u) : 0u;
        while (k < cnt) {
            uint32_t t, b;
            if (STAGED) {
                const uint32_t e = ent[k];
                t = e & 63u;
                b = e >> 6;
            } else {
                t = (uint32_t)((uint64_t)__ldg(pos + a + k) - ow0);
                b = __ldg(bint + a + k);
            }
            if (t >= base + 32u) break;
            const uint32_t tt = t - base;
            const uint32_t run = tt - filled;
            const uint32_t m = (1u << run) - 1u;  // run <= 31
            al |= ((wl >> u) & m) << filled;
            ah |= ((wh >> u) & m) << filled;
            ad |= ((wd >> u) & m) << filled;
            if (N5) an |= ((wn >> u) & m) << filled;
            u += run;
            al |= (b & 1u) << tt;
            ah |= ((b >> 1) & 1u) << tt;
            ad |= ((b >> 2) & 1u) << tt;
            if (N5) an |= ((b >> 3) & 1u) << tt;
            filled = tt + 1;
            ++k;
        }
        if (hl > filled) {
            const uint32_t run = hl - filled;
            const uint32_t m = run == 32 ? ~0u : (1u << run) - 1u;
            al |= ((wl >> u) & m) << filled;
            ah |= ((wh >> u) & m) << filled;
            ad |= ((wd >> u) & m) << filled;
            if (N5) an |= ((wn >> u) & m) << filled;
            u += run;
        }
        used += u;
        oo[hf][0] = al;
        oo[hf][1] = ah;
        oo[hf][2] = ad;
        oo[hf][3] = an;
    }
}

// inserted entries staged in shared memory per superblock (dynamic shared
// memory): enough for a block that adds up to ~60 % new symbols
constexpr uint32_t kStage = 40960;

// D = const Blk* (one array) or Dict (a sharded dictionary, NEXT-3)
// N5 (sigma = 5): also merges the N plane (in_nblk -> out_nblk) and writes the
// superblock totals of code 4 into ntot.
template <class G, class D, bool N5>
__global__ void __launch_bounds__(kInsNt) insert_kernel(
    const D in_blk, uint64_t n_in, const G* __restrict__ pos,
    const uint8_t* __restrict__ bint, uint64_t n_ins, Blk* __restrict__ out_blk, uint64_t n_out,
    uint64_t* __restrict__ sb_tot, const uint64_t* __restrict__ sb_start, uint64_t sb_begin,
    uint64_t sb_end, const NBlk* __restrict__ in_nblk, NBlk* __restrict__ out_nblk,
    uint64_t* __restrict__ ntot) {
    // in_blk / out_blk are indexed by absolute Blk number; the host-tier path
    // and a sharded index pass pointers biased by their window (only the
    // window is touched); in_blk may be split into shards (Dict)
    __shared__ uint32_t wcnt[kBlkPerSb];
    extern __shared__ uint16_t ent[];  // kStage: (offset in word) | (B_int code+$ << 6)
    __shared__ uint32_t wsum[5][kInsWarps];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint64_t sbi = sb_begin + blockIdx.x; sbi < sb_end; sbi += gridDim.x) {
        const uint64_t o0 = sbi << kSbShift;
        wcnt[tid] = 0;
        __syncthreads();
        const uint64_t i_lo = sb_start[sbi], i_hi = sb_start[sbi + 1];
        const bool staged = i_hi - i_lo <= kStage;
        // pass 1 (coalesced): inserted symbols per output word, staged entries;
        // four independent loads in flight per thread while four whole rounds
        // of the CTA remain, then one element per round (a late c3 block has
        // ~4400 per superblock: unconditional 4-wide rounds wasted half the
        // issue slots on predicated-off elements)
        uint64_t i0 = i_lo + tid;
        for (; i0 + 3ull * kInsNt < i_hi; i0 += 4 * kInsNt) {
            uint32_t rel[4], bb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t i = i0 + (uint64_t)u * kInsNt;
                rel[u] = (uint32_t)((uint64_t)__ldg(pos + i) - o0);
                bb[u] = staged ? (uint32_t)__ldg(bint + i) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t i = i0 + (uint64_t)u * kInsNt;
                atomicAdd(&wcnt[rel[u] >> 6], 1u);
                if (staged) ent[i - i_lo] = (uint16_t)((rel[u] & 63u) | (bb[u] << 6));
            }
        }
        for (; i0 < i_hi; i0 += kInsNt) {
            const uint32_t rel = (uint32_t)((uint64_t)__ldg(pos + i0) - o0);
            const uint32_t bb = staged ? (uint32_t)__ldg(bint + i0) : 0u;
            atomicAdd(&wcnt[rel >> 6], 1u);
            if (staged) ent[i0 - i_lo] = (uint16_t)((rel & 63u) | (bb << 6));
        }
        __syncthreads();
        // exclusive scan over the 1024 words (two-level)
        const uint32_t cnt = wcnt[tid];
        const uint32_t incl = warp_incl(cnt, lane);
        if (lane == 31) wsum[0][warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const uint32_t x = wsum[0][lane];
            wsum[0][lane] = warp_incl(x, lane) - x;
        }
        __syncthreads();
        const uint32_t arel = wsum[0][warp] + incl - cnt;  // inserted before this word
        const uint64_t a = i_lo + arel;
        // one thread merges one 64-symbol output word
        const uint64_t ow0 = o0 + ((uint64_t)tid << 6);
        const bool wvalid = ow0 <= n_out;
        uint64_t ol = 0, oh = 0, od = 0, on = 0;
        uint32_t c4[5] = {0, 0, 0, 0, 0};
        if (wvalid) {
            const uint64_t e0 = ow0 - a;  // external symbols before this word
            uint64_t xl = 0, xh = 0, xd = 0, xn = 0;
            if (e0 < n_in) {
                const uint64_t eb = e0 >> 6;
                const uint32_t sh = (uint32_t)(e0 & 63);
                uint64_t b0[4], b1[4] = {0, 0, 0, 0};
                asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                    : "=l"(b0[0]), "=l"(b0[1]), "=l"(b0[2]), "=l"(b0[3])
                    : "l"(blk_at(in_blk, eb)));
                if (sh != 0 && ((eb + 1) << 6) < n_in)
                    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                        : "=l"(b1[0]), "=l"(b1[1]), "=l"(b1[2]), "=l"(b1[3])
                        : "l"(blk_at(in_blk, eb + 1)));
                xl = funnel(b0[1], b1[1], sh);
                xh = funnel(b0[2], b1[2], sh);
                xd = funnel(b0[3], b1[3], sh);
                if (N5) {
                    const uint64_t n0 = __ldg(&in_nblk[eb].n);
                    const uint64_t n1 =
                        (sh != 0 && ((eb + 1) << 6) < n_in) ? __ldg(&in_nblk[eb + 1].n) : 0ull;
                    xn = funnel(n0, n1, sh);
                }
            }
            // merge one 32-symbol half at a time: all shifts stay 32-bit
            const uint64_t span = n_out - ow0;
            const uint32_t lim = span >= 64 ? 64u : (uint32_t)span;
            if (cnt == 64 && (a & 15) == 0) {
                // every symbol of the word is inserted (e.g. the first block):
                // its planes are B_int[a .. a+64) bit-sliced, 8 bytes at a time
                const uint4* src = reinterpret_cast<const uint4*>(bint + a);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint4 v = __ldg(src + q);
                    const uint64_t w2[2] = {((uint64_t)v.y << 32) | v.x, ((uint64_t)v.w << 32) | v.z};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t sh8 = 16 * q + 8 * h;
                        // bit k of byte j -> bit j (the "multiply gather" of 8 flag bits)
                        const uint64_t m = 0x0101010101010101ull, mul = 0x0102040810204080ull;
                        ol |= (((w2[h] & m) * mul) >> 56) << sh8;
                        oh |= ((((w2[h] >> 1) & m) * mul) >> 56) << sh8;
                        od |= ((((w2[h] >> 2) & m) * mul) >> 56) << sh8;
                        if (N5) on |= ((((w2[h] >> 3) & m) * mul) >> 56) << sh8;
                    }
                }
            } else {
                uint32_t oo[2][4];
                if (staged)
                    merge_word<true, G, N5>(oo, xl, xh, xd, xn, lim, cnt, ent + arel, pos, bint,
                                            a, ow0);
                else
                    merge_word<false, G, N5>(oo, xl, xh, xd, xn, lim, cnt, ent, pos, bint, a,
                                             ow0);
                ol = (uint64_t)oo[0][0] | ((uint64_t)oo[1][0] << 32);
                oh = (uint64_t)oo[0][1] | ((uint64_t)oo[1][1] << 32);
                od = (uint64_t)oo[0][2] | ((uint64_t)oo[1][2] << 32);
                if (N5) on = (uint64_t)oo[0][3] | ((uint64_t)oo[1][3] << 32);
            }
            const uint64_t V = lim == 64 ? ~0ull : ((1ull << lim) - 1ull);  // real positions
            // per code (match_plane): 1 = lo & ~hi, 2 = ~lo & hi, 3 = lo & hi,
            // 0 = neither, over the non-'$' positions
            const uint64_t nd = ~od & V;
            const uint32_t nl = __popcll(ol & nd), nh = __popcll(oh & nd);
            const uint32_t n3 = __popcll(ol & oh & nd), na = __popcll(nd);
            c4[0] = na - nl - nh + n3;
            c4[1] = nl - n3;
            c4[2] = nh - n3;
            c4[3] = n3;
            if (N5) c4[4] = __popcll(on & V);
        }
        // in-superblock exclusive prefix of the per-word counts (4 codes, + N);
        // codes in 16-bit pairs (a warp's 32 words hold <= 2048 of each)
        constexpr int NC = N5 ? 5 : 4;
        uint32_t inc[NC];
        {
            const uint32_t i01 = warp_incl(c4[0] | (c4[1] << 16), lane);
            const uint32_t i23 = warp_incl(c4[2] | (c4[3] << 16), lane);
            inc[0] = i01 & 0xFFFFu;
            inc[1] = i01 >> 16;
            inc[2] = i23 & 0xFFFFu;
            inc[3] = i23 >> 16;
            if (N5) inc[NC - 1] = warp_incl(c4[4], lane);
        }
        if (lane == 31) {
#pragma unroll
            for (int c = 0; c < NC; ++c) wsum[c][warp] = inc[c];
        }
        __syncthreads();
        if (warp < NC) {
            const uint32_t x = wsum[warp][lane];
            const uint32_t y = warp_incl(x, lane);
            wsum[warp][lane] = y - x;
            if (lane == 31) {
                if (warp < 4) sb_tot[sbi * 4 + warp] = y;
                else ntot[sbi] = y;
            }
        }
        __syncthreads();
        if (wvalid) {
            SB_ASSERT(((sbi << (kSbShift - 6)) + tid) <= (n_out >> 6));
            uint64_t w0 = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                w0 |= (uint64_t)(uint16_t)(wsum[c][warp] + inc[c] - c4[c]) << (16 * c);
            asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(out_blk + (sbi << (kSbShift - 6)) + tid),
                         "l"(w0), "l"(ol), "l"(oh), "l"(od));
            if (N5) {
                const uint64_t ncnt = (uint64_t)(wsum[4][warp] + inc[NC - 1] - c4[4]);
                asm volatile("st.global.v2.u64 [%0], {%1,%2};" ::"l"(out_nblk + (sbi << (kSbShift - 6)) + tid),
                             "l"(on), "l"(ncnt));
            }
        }
        __syncthreads();
    }
}

// Exclusive scan of the superblock totals -> u64 superblock counters, and C.
// One CTA: each thread owns a contiguous run of superblocks; the run totals
// are scanned with warp shuffles (no shared-memory Hillis-Steele rounds).
__global__ void __launch_bounds__(1024) sb_scan_kernel(const uint64_t* __restrict__ sb_tot,
                                                       uint64_t nsb, uint64_t* __restrict__ sb,
                                                       uint64_t m_new, uint64_t* __restrict__ Cd) {
    __shared__ uint64_t wtot[32][4];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t per = (nsb + 1023) / 1024;
    const uint64_t b = tid * per, e = min(b + per, nsb);
    uint64_t acc[4] = {0, 0, 0, 0};
    for (uint64_t i = b; i < e; ++i) {
        const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(sb_tot + i * 4);
        const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(sb_tot + i * 4 + 2);
        acc[0] += x.x;
        acc[1] += x.y;
        acc[2] += y.x;
        acc[3] += y.y;
    }
    uint64_t inc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        inc[c] = acc[c];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t v = __shfl_up_sync(0xFFFFFFFFu, inc[c], o);
            if (lane >= (uint32_t)o) inc[c] += v;
        }
    }
    if (lane == 31)
        for (int c = 0; c < 4; ++c) wtot[warp][c] = inc[c];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint64_t x = wtot[lane][c];
            uint64_t y = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t v = __shfl_up_sync(0xFFFFFFFFu, y, o);
                if (lane >= (uint32_t)o) y += v;
            }
            wtot[lane][c] = y - x;  // exclusive over warps
        }
    }
    __syncthreads();
    uint64_t run[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) run[c] = wtot[warp][c] + inc[c] - acc[c];
    for (uint64_t i = b; i < e; ++i) {
        const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(sb_tot + i * 4);
        const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(sb_tot + i * 4 + 2);
        *reinterpret_cast<ulonglong2*>(sb + i * 4) = make_ulonglong2(run[0], run[1]);
        *reinterpret_cast<ulonglong2*>(sb + i * 4 + 2) = make_ulonglong2(run[2], run[3]);
        run[0] += x.x;
        run[1] += x.y;
        run[2] += y.x;
        run[3] += y.y;
    }
    if (tid == 1023) {
        // C[c] = #symbols < c: all m '$' plus the smaller codes (Lemma 1);
        // thread 1023's running counts are the totals over all superblocks
        uint64_t acc2 = m_new;
        for (int c = 0; c < 4; ++c) {
            Cd[c] = acc2;
            acc2 += run[c];
        }
        Cd[4] = acc2;  // = n (consistency)
    }
}

template <class D, bool N5>
cudaError_t launch_insert_kernel(Profiler& prof, cudaStream_t s, const D in_blk, uint64_t n_in,
                                 const void* pos, int gw, const uint8_t* bint, uint64_t n_ins,
                                 Blk* out_blk, uint64_t n_out, uint64_t* sb_tot,
                                 const uint64_t* sb_start, uint64_t sb_begin, uint64_t sb_end,
                                 unsigned grid, double bytes, double frac, const N5Ins* n5) {
    SB_CHECK(cudaFuncSetAttribute(insert_kernel<uint32_t, D, N5>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kStage * 2)));
    SB_CHECK(cudaFuncSetAttribute(insert_kernel<uint64_t, D, N5>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kStage * 2)));
    const NBlk* nin = n5 ? n5->in : nullptr;
    NBlk* nout = n5 ? n5->out : nullptr;
    uint64_t* ntot = n5 ? n5->ntot : nullptr;
    if (gw == 4) {
        SB_LAUNCH(prof, s, "insert", bytes, (uint64_t)(frac * n_out),
                  (insert_kernel<uint32_t, D, N5><<<grid, kInsNt, kStage * 2, s>>>(
                      in_blk, n_in, (const uint32_t*)pos, bint, n_ins, out_blk, n_out, sb_tot,
                      sb_start, sb_begin, sb_end, nin, nout, ntot)));
    } else {
        SB_LAUNCH(prof, s, "insert", bytes, (uint64_t)(frac * n_out),
                  (insert_kernel<uint64_t, D, N5><<<grid, kInsNt, kStage * 2, s>>>(
                      in_blk, n_in, (const uint64_t*)pos, bint, n_ins, out_blk, n_out, sb_tot,
                      sb_start, sb_begin, sb_end, nin, nout, ntot)));
    }
    return cudaGetLastError();
}

cudaError_t launch_insert_range(Profiler& prof, cudaStream_t s, const Dict& in_blk, uint64_t n_in,
                                const void* pos, int gw, const uint8_t* bint, uint64_t n_ins,
                                Blk* out_blk, uint64_t* sb_tot, const uint64_t* sb_start,
                                uint64_t sb_begin, uint64_t sb_end, const N5Ins* n5) {
    const uint64_t n_out = n_in + n_ins;
    const uint64_t nsb_r = sb_end - sb_begin;
    if (nsb_r == 0) return cudaSuccess;
    // algorithmic bytes of the range: its share of B_ext read + B_ext' written
    // (4 bits/symbol each; + 2 bits/symbol of N plane with sigma = 5) + (gw + 1)
    // B per inserted symbol of the range
    const double frac = (double)nsb_r / (double)((n_out >> kSbShift) + 1);
    const double dsym = n5 ? 0.75 : 0.5;
    const double bytes = frac * (dsym * (double)n_in + dsym * (double)n_out + (gw + 1.0) * (double)n_ins);
    unsigned grid = (unsigned)(nsb_r < 148u * 64u ? nsb_r : 148u * 64u);
    if (const char* e = getenv("SETBWTE_INSERT_GRID"))
        grid = std::min<unsigned>(grid, (unsigned)atoi(e));
    if (n5)  // sigma = 5: one plain array (no shards, no host tier)
        SB_CHECK((launch_insert_kernel<const Blk*, true>(prof, s, in_blk.ptr[0], n_in, pos, gw, bint,
                                                         n_ins, out_blk, n_out, sb_tot, sb_start,
                                                         sb_begin, sb_end, grid, bytes, frac, n5)));
    else if (in_blk.P == 1)
        SB_CHECK((launch_insert_kernel<const Blk*, false>(prof, s, in_blk.ptr[0], n_in, pos, gw, bint,
                                                          n_ins, out_blk, n_out, sb_tot, sb_start,
                                                          sb_begin, sb_end, grid, bytes, frac,
                                                          nullptr)));
    else
        SB_CHECK((launch_insert_kernel<Dict, false>(prof, s, in_blk, n_in, pos, gw, bint, n_ins,
                                                    out_blk, n_out, sb_tot, sb_start, sb_begin,
                                                    sb_end, grid, bytes, frac, nullptr)));
    return cudaSuccess;
}

cudaError_t launch_sb_scan(Profiler& prof, cudaStream_t s, const uint64_t* sb_tot, uint64_t nsb,
                           uint64_t* out_sb, uint64_t m_new, uint64_t* d_C) {
    SB_LAUNCH(prof, s, "sb_scan", 64.0 * nsb, nsb,
              sb_scan_kernel<<<1, 1024, 0, s>>>(sb_tot, nsb, out_sb, m_new, d_C));
    return cudaGetLastError();
}

// sigma = 5: exclusive scan of the per-superblock code-4 totals -> nsb (one CTA).
__global__ void __launch_bounds__(1024) nsb_scan_kernel(const uint64_t* __restrict__ ntot,
                                                        uint64_t nsb, uint64_t* __restrict__ out) {
    __shared__ uint64_t wtot[32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t per = (nsb + 1023) / 1024;
    const uint64_t b = tid * per, e = min(b + per, nsb);
    uint64_t acc = 0;
    for (uint64_t i = b; i < e; ++i) acc += ntot[i];
    uint64_t inc = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= (uint32_t)o) inc += v;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint64_t x = wtot[lane];
        uint64_t y = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t v = __shfl_up_sync(0xFFFFFFFFu, y, o);
            if (lane >= (uint32_t)o) y += v;
        }
        wtot[lane] = y - x;
    }
    __syncthreads();
    uint64_t run = wtot[warp] + inc - acc;
    for (uint64_t i = b; i < e; ++i) {
        const uint64_t x = ntot[i];
        out[i] = run;
        run += x;
    }
}

cudaError_t launch_nsb_scan(Profiler& prof, cudaStream_t s, const uint64_t* ntot, uint64_t nsb,
                            uint64_t* out) {
    SB_LAUNCH(prof, s, "sb_scan", 16.0 * nsb, nsb, nsb_scan_kernel<<<1, 1024, 0, s>>>(ntot, nsb, out));
    return cudaGetLastError();
}

cudaError_t launch_insert(Profiler& prof, cudaStream_t s, const Dict& in_blk, uint64_t n_in,
                          const void* pos, int gw, const uint8_t* bint, uint64_t n_ins,
                          Blk* out_blk, uint64_t* out_sb, uint64_t* sb_tot,
                          const uint64_t* sb_start, uint64_t m_new, uint64_t* d_C,
                          const N5Ins* n5) {
    const uint64_t n_out = n_in + n_ins;
    const uint64_t nsb = (n_out >> kSbShift) + 1;
    SB_CHECK(launch_insert_range(prof, s, in_blk, n_in, pos, gw, bint, n_ins, out_blk, sb_tot,
                                 sb_start, 0, nsb, n5));
    if (n5) SB_CHECK(launch_nsb_scan(prof, s, n5->ntot, nsb, n5->nsb_out));
    return launch_sb_scan(prof, s, sb_tot, nsb, out_sb, m_new, d_C);
}

// FM-index count by backward search (Lemma 1 P:97-100 applied to
// the interval [lo, hi) of rows whose suffixes start with the pattern's
// processed tail): per pattern P, for k = |P|-1..0: c = P[k];
// lo = C[c] + rank(c, lo), hi = C[c] + rank(c, hi); count = hi - lo.
// A byte outside the alphabet makes the count 0; the empty pattern counts n.
__global__ void count_kernel(const Dict blk, const uint64_t* __restrict__ sb,
                             uint64_t n, const uint64_t* __restrict__ Cd,
                             const uint8_t* __restrict__ code_of, const uint8_t* __restrict__ pat,
                             const uint64_t* __restrict__ poff, uint64_t q,
                             uint64_t* __restrict__ out, N5Dict n5) {
    const uint64_t C0 = Cd[0], C1 = Cd[1], C2 = Cd[2], C3 = Cd[3], C4 = Cd[4];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < q;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = poff[t], b = poff[t + 1];
        uint64_t lo = 0, hi = n;
        for (uint64_t k = b; k > a && lo < hi; --k) {
            const uint8_t c = code_of[pat[k - 1]];
            if (c == 4 && n5.nblk) {  // sigma = 5: the fifth symbol's plane
                lo = C4 + dict_rank_n(n5.nblk, n5.nsb, lo);
                hi = C4 + dict_rank_n(n5.nblk, n5.nsb, hi);
                continue;
            }
            if (c > 3) {
                lo = hi = 0;
                break;
            }
            const uint64_t Cc = c == 0 ? C0 : c == 1 ? C1 : c == 2 ? C2 : C3;
            lo = Cc + dict_rank(blk, sb, c, lo);
            hi = Cc + dict_rank(blk, sb, c, hi);
        }
        out[t] = hi > lo ? hi - lo : 0;
    }
}

cudaError_t launch_count(Profiler& prof, cudaStream_t s, const Dict& blk, const uint64_t* sb,
                         uint64_t n, const uint64_t* d_C, const uint8_t* code_of,
                         const uint8_t* pat, const uint64_t* poff, uint64_t q, uint64_t* out,
                         const N5Dict* n5) {
    if (q == 0) return cudaSuccess;
    const N5Dict nd = n5 ? *n5 : N5Dict{};
    SB_LAUNCH(prof, s, "fm_count", 0, q,
              count_kernel<<<grid_for(q, 128, 148u * 64u), 128, 0, s>>>(blk, sb, n, d_C, code_of,
                                                                        pat, poff, q, out, nd));
    return cudaGetLastError();
}

__global__ void rank_batch_kernel(const Dict blk, const uint64_t* __restrict__ sb,
                                  uint64_t n, const uint8_t* __restrict__ code_of,
                                  const uint8_t* __restrict__ cq, const uint64_t* __restrict__ kq,
                                  uint64_t q, uint64_t* __restrict__ out, N5Dict n5) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < q;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint8_t c = cq[t];
        const uint64_t k = kq[t];
        uint64_t r = ~0ull;
        if (k <= n) {
            if (c == '$') {
                uint64_t sum = 0;
                for (uint32_t x = 0; x < 4; ++x) sum += dict_rank(blk, sb, x, k);
                if (n5.nblk) sum += dict_rank_n(n5.nblk, n5.nsb, k);
                r = k - sum;  // reading R12
            } else {
                const uint8_t code = code_of[c];
                if (code < 4) r = dict_rank(blk, sb, code, k);
                else if (code == 4 && n5.nblk) r = dict_rank_n(n5.nblk, n5.nsb, k);
            }
        }
        out[t] = r;
    }
}

cudaError_t launch_rank_batch(Profiler& prof, cudaStream_t s, const Dict& blk, const uint64_t* sb,
                              uint64_t n, const uint8_t* code_of, const uint8_t* c,
                              const uint64_t* k, uint64_t q, uint64_t* out, const N5Dict* n5) {
    if (q == 0) return cudaSuccess;
    const N5Dict nd = n5 ? *n5 : N5Dict{};
    SB_LAUNCH(prof, s, "rank_query", 49.0 * q, q,
              rank_batch_kernel<<<grid_for(q, 256, 148u * 64u), 256, 0, s>>>(blk, sb, n, code_of,
                                                                             c, k, q, out, nd));
    return cudaGetLastError();
}

// BWT decode: one thread per 64-symbol Blk, 4 x 16-byte stores of ASCII.
__global__ void decode_kernel(const Dict blk, uint64_t n,
                              const uint8_t* __restrict__ sym_ascii, uint8_t* __restrict__ out,
                              const NBlk* __restrict__ nblk) {
    const uint32_t sym4 = sym_ascii[4];  // sigma = 5: the fifth symbol (nblk != null)
    // code -> byte lookup via byte_perm: selector nibble c picks sym[c]
    const uint32_t tab = (uint32_t)sym_ascii[0] | ((uint32_t)sym_ascii[1] << 8) |
                         ((uint32_t)sym_ascii[2] << 16) | ((uint32_t)sym_ascii[3] << 24);
    const uint64_t nb = (n + 63) >> 6;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb;
         b += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t w[4];
        asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
            : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(dict_blk(blk, b)));
        const uint64_t lo = w[1], hi = w[2], dl = w[3];
        const uint64_t nn = nblk ? __ldg(&nblk[b].n) : 0ull;
        uint32_t o[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            uint32_t v = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int p = 4 * q + t;
                const uint32_t c = (uint32_t)(((lo >> p) & 1ull) | (((hi >> p) & 1ull) << 1));
                uint32_t ch = __byte_perm(tab, 0, c);  // sym_ascii[c] in byte 0
                if ((dl >> p) & 1ull) ch = ((nn >> p) & 1ull) ? sym4 : (uint32_t)'$';
                v |= (ch & 0xFFu) << (8 * t);
            }
            o[q] = v;
        }
        const uint64_t base = b << 6;
        if (base + 64 <= n && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
            uint4* dst = reinterpret_cast<uint4*>(out + base);
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        } else {
            const uint32_t cnt = (uint32_t)min((uint64_t)64, n - base);
            for (uint32_t t = 0; t < cnt; ++t) out[base + t] = (uint8_t)(o[t >> 2] >> (8 * (t & 3)));
        }
    }
}

cudaError_t launch_decode(Profiler& prof, cudaStream_t s, const Dict& blk, uint64_t n,
                          const uint8_t* sym_ascii, uint8_t* out, const NBlk* nblk) {
    if (n == 0) return cudaSuccess;
    SB_LAUNCH(prof, s, "decode", 1.5 * n, n,
              decode_kernel<<<grid_for((n + 63) >> 6, 128, 148u * 64u), 128, 0, s>>>(
                  blk, n, sym_ascii, out, nblk));
    return cudaGetLastError();
}

__global__ void bint_ascii_kernel(const uint8_t* __restrict__ bint, uint32_t n,
                                  const uint8_t* __restrict__ sym_ascii, uint8_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint8_t b = bint[i];
        out[i] = (b & 8) ? sym_ascii[4] : (b & 4) ? (uint8_t)'$' : sym_ascii[b & 3];
    }
}

cudaError_t launch_bint_ascii(Profiler& prof, cudaStream_t s, const uint8_t* bint,
                              uint32_t n_suf, const uint8_t* sym_ascii, uint8_t* out) {
    if (n_suf == 0) return cudaSuccess;
    SB_LAUNCH(prof, s, "bint_ascii", 2.0 * n_suf, n_suf,
              bint_ascii_kernel<<<grid_for(n_suf, 256), 256, 0, s>>>(bint, n_suf, sym_ascii, out));
    return cudaGetLastError();
}

}  // namespace setbwte
