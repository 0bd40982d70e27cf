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
#include "internal.h"

namespace setbwte {

namespace {
constexpr int kInsNt = 512;
constexpr int kInsWarps = kInsNt / 32;

__device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t* __restrict__ a, uint64_t n,
                                                    uint64_t x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint64_t funnel(uint64_t a, uint64_t b, uint32_t sh) {
    return sh == 0 ? a : (a >> sh) | (b << (64 - sh));
}
}  // namespace

__global__ void __launch_bounds__(kInsNt) insert_kernel(
    const Blk* __restrict__ in_blk, uint64_t n_in, const uint64_t* __restrict__ pos,
    const uint8_t* __restrict__ bint, uint64_t n_ins, Blk* __restrict__ out_blk, uint64_t n_out,
    uint64_t* __restrict__ sb_tot) {
    __shared__ uint32_t wstart[kBlkPerSb + 1];
    __shared__ uint64_t w_lo[kBlkPerSb], w_hi[kBlkPerSb], w_dol[kBlkPerSb];
    __shared__ uint16_t w_cnt[4][kBlkPerSb];
    __shared__ uint32_t scan_tmp[kInsWarps][4];
    __shared__ uint64_t i_range[2];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t nsb = (n_out >> kSbShift) + 1;
    for (uint64_t sbi = blockIdx.x; sbi < nsb; sbi += gridDim.x) {
        const uint64_t o0 = sbi << kSbShift;
        if (tid == 0) i_range[0] = lower_bound_u64(pos, n_ins, o0);
        if (tid == 32) i_range[1] = lower_bound_u64(pos, n_ins, o0 + (1ull << kSbShift));
        for (uint32_t w = tid; w <= (uint32_t)kBlkPerSb; w += kInsNt) wstart[w] = 0;
        __syncthreads();
        const uint64_t i_lo = i_range[0], i_hi = i_range[1];
        for (uint64_t i = i_lo + tid; i < i_hi; i += kInsNt)
            atomicAdd(&wstart[(uint32_t)((__ldg(pos + i) - o0) >> 6)], 1u);
        __syncthreads();
        // exclusive scan of wstart[0..1024) -> wstart, wstart[1024] = total
        {
            const uint32_t a0 = wstart[2 * tid], a1 = wstart[2 * tid + 1];
            uint32_t incl = a0 + a1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= (uint32_t)o) incl += y;
            }
            if (lane == 31) scan_tmp[warp][0] = incl;
            __syncthreads();
            uint32_t pre = 0;
            for (uint32_t w = 0; w < warp; ++w) pre += scan_tmp[w][0];
            const uint32_t ex = pre + incl - a0 - a1;
            __syncthreads();
            wstart[2 * tid] = ex;
            wstart[2 * tid + 1] = ex + a0;
            if (tid == kInsNt - 1) wstart[kBlkPerSb] = ex + a0 + a1;
            __syncthreads();
        }
        const uint64_t span = n_out - o0;  // >= 0 by the grid range
        const uint32_t wmax = (uint32_t)min((uint64_t)kBlkPerSb, (span >> 6) + 1);
        for (uint32_t w = warp; w < wmax; w += kInsWarps) {
            const uint64_t ow0 = o0 + ((uint64_t)w << 6);
            const uint64_t a = i_lo + wstart[w];
            const uint32_t cnt = wstart[w + 1] - wstart[w];
            uint64_t M = 0;
            for (uint32_t q = lane; q < cnt; q += 32) M |= 1ull << (__ldg(pos + a + q) - ow0);
            const uint32_t Mlo = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)M);
            const uint32_t Mhi = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)(M >> 32));
            M = ((uint64_t)Mhi << 32) | Mlo;
            // window of 64 external symbols starting at e_base = ow0 - a
            const uint64_t e_base = ow0 - a;
            uint64_t xl = 0, xh = 0, xd = 0;
            if (e_base < n_in) {
                const uint64_t eb = e_base >> 6;
                const uint32_t sh = (uint32_t)(e_base & 63);
                const Blk* b0 = in_blk + eb;
                const uint64_t l0 = __ldg(&b0->lo), h0 = __ldg(&b0->hi), d0 = __ldg(&b0->dol);
                uint64_t l1 = 0, h1 = 0, d1 = 0;
                if (sh != 0 && ((eb + 1) << 6) < n_in) {
                    l1 = __ldg(&b0[1].lo);
                    h1 = __ldg(&b0[1].hi);
                    d1 = __ldg(&b0[1].dol);
                }
                xl = funnel(l0, l1, sh);
                xh = funnel(h0, h1, sh);
                xd = funnel(d0, d1, sh);
            }
            uint32_t code[2], dol[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t t = lane + 32 * h;
                const uint32_t r = __popcll(M & ((1ull << t) - 1ull));
                if ((M >> t) & 1ull) {
                    const uint8_t b = __ldg(bint + a + r);
                    code[h] = b & 3u;
                    dol[h] = b >> 2;
                } else {
                    const uint32_t x = t - r;
                    code[h] = (uint32_t)(((xl >> x) & 1ull) | (((xh >> x) & 1ull) << 1));
                    dol[h] = (uint32_t)((xd >> x) & 1ull);
                }
                if (ow0 + t >= n_out) {
                    code[h] = 0;
                    dol[h] = 0;
                }
            }
            const uint64_t lo = (uint64_t)__ballot_sync(0xFFFFFFFFu, code[0] & 1u) |
                                ((uint64_t)__ballot_sync(0xFFFFFFFFu, code[1] & 1u) << 32);
            const uint64_t hi = (uint64_t)__ballot_sync(0xFFFFFFFFu, code[0] >> 1) |
                                ((uint64_t)__ballot_sync(0xFFFFFFFFu, code[1] >> 1) << 32);
            const uint64_t dl = (uint64_t)__ballot_sync(0xFFFFFFFFu, dol[0]) |
                                ((uint64_t)__ballot_sync(0xFFFFFFFFu, dol[1]) << 32);
            if (lane < 4) {
                const uint64_t V = (n_out - ow0 >= 64) ? ~0ull : ((1ull << (n_out - ow0)) - 1ull);
                w_cnt[lane][w] = (uint16_t)__popcll(match_plane(lane, lo, hi, dl) & V);
            }
            if (lane == 0) {
                w_lo[w] = lo;
                w_hi[w] = hi;
                w_dol[w] = dl;
            }
        }
        __syncthreads();
        // exclusive scan of the per-word counts (4 codes) over the superblock
        {
            uint32_t v0[4], v1[4], incl[4];
            const uint32_t wa = 2 * tid, wb = 2 * tid + 1;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                v0[c] = wa < wmax ? w_cnt[c][wa] : 0u;
                v1[c] = wb < wmax ? w_cnt[c][wb] : 0u;
                incl[c] = v0[c] + v1[c];
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl[c], o);
                    if (lane >= (uint32_t)o) incl[c] += y;
                }
            }
            if (lane == 31) {
#pragma unroll
                for (int c = 0; c < 4; ++c) scan_tmp[warp][c] = incl[c];
            }
            __syncthreads();
            uint32_t pre[4] = {0, 0, 0, 0}, tot[4] = {0, 0, 0, 0};
            for (uint32_t w = 0; w < (uint32_t)kInsWarps; ++w) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (w < warp) pre[c] += scan_tmp[w][c];
                    tot[c] += scan_tmp[w][c];
                }
            }
            Blk* ob = out_blk + (sbi << (kSbShift - 6));
            if (wa < wmax) {
                Blk b;
#pragma unroll
                for (int c = 0; c < 4; ++c) b.cnt[c] = (uint16_t)(pre[c] + incl[c] - v0[c] - v1[c]);
                b.lo = w_lo[wa];
                b.hi = w_hi[wa];
                b.dol = w_dol[wa];
                ob[wa] = b;
            }
            if (wb < wmax) {
                Blk b;
#pragma unroll
                for (int c = 0; c < 4; ++c) b.cnt[c] = (uint16_t)(pre[c] + incl[c] - v1[c]);
                b.lo = w_lo[wb];
                b.hi = w_hi[wb];
                b.dol = w_dol[wb];
                ob[wb] = b;
            }
            if (tid < 4) sb_tot[sbi * 4 + tid] = tot[tid];
            __syncthreads();
        }
    }
}

// Exclusive scan of the superblock totals -> u64 superblock counters, and C.
__global__ void __launch_bounds__(1024) sb_scan_kernel(const uint64_t* __restrict__ sb_tot,
                                                       uint64_t nsb, uint64_t* __restrict__ sb,
                                                       uint64_t m_new, uint64_t* __restrict__ Cd) {
    __shared__ uint64_t part[1024][4];
    const uint32_t tid = threadIdx.x;
    const uint64_t per = (nsb + 1023) / 1024;
    const uint64_t b = tid * per, e = min(b + per, nsb);
    uint64_t acc[4] = {0, 0, 0, 0};
    for (uint64_t i = b; i < e; ++i)
        for (int c = 0; c < 4; ++c) acc[c] += sb_tot[i * 4 + c];
    for (int c = 0; c < 4; ++c) part[tid][c] = acc[c];
    __syncthreads();
    for (uint32_t o = 1; o < 1024; o <<= 1) {
        uint64_t v[4] = {0, 0, 0, 0};
        if (tid >= o)
            for (int c = 0; c < 4; ++c) v[c] = part[tid - o][c];
        __syncthreads();
        for (int c = 0; c < 4; ++c) part[tid][c] += v[c];
        __syncthreads();
    }
    uint64_t run[4];
    for (int c = 0; c < 4; ++c) run[c] = tid ? part[tid - 1][c] : 0;
    for (uint64_t i = b; i < e; ++i)
        for (int c = 0; c < 4; ++c) {
            sb[i * 4 + c] = run[c];
            run[c] += sb_tot[i * 4 + c];
        }
    if (tid == 0) {
        // C[c] = #symbols < c: all m '$' plus the smaller codes (Lemma 1)
        uint64_t acc2 = m_new;
        for (int c = 0; c < 4; ++c) {
            Cd[c] = acc2;
            acc2 += part[1023][c];
        }
        Cd[4] = acc2;  // = n (consistency)
    }
}

cudaError_t launch_insert(Profiler& prof, cudaStream_t s, const Blk* in_blk, uint64_t n_in,
                          const uint64_t* pos, const uint8_t* bint, uint64_t n_ins,
                          Blk* out_blk, uint64_t* out_sb, uint64_t* sb_tot, uint64_t m_new,
                          uint64_t* d_C) {
    const uint64_t n_out = n_in + n_ins;
    const uint64_t nsb = (n_out >> kSbShift) + 1;
    // algorithmic bytes: read n_in/2 + write n_out/2 (4 bits/symbol) + 9 B per inserted
    const double bytes = 0.5 * (double)n_in + 0.5 * (double)n_out + 9.0 * (double)n_ins;
    SB_LAUNCH(prof, s, "insert", bytes, n_out,
              insert_kernel<<<(unsigned)(nsb < 148u * 64u ? nsb : 148u * 64u), kInsNt, 0, s>>>(
                  in_blk, n_in, pos, bint, n_ins, out_blk, n_out, sb_tot));
    SB_CHECK(cudaGetLastError());
    SB_LAUNCH(prof, s, "sb_scan", 64.0 * nsb, nsb,
              sb_scan_kernel<<<1, 1024, 0, s>>>(sb_tot, nsb, out_sb, m_new, d_C));
    return cudaGetLastError();
}

__global__ void rank_batch_kernel(const Blk* __restrict__ blk, const uint64_t* __restrict__ sb,
                                  uint64_t n, const uint8_t* __restrict__ code_of,
                                  const uint8_t* __restrict__ cq, const uint64_t* __restrict__ kq,
                                  uint64_t q, uint64_t* __restrict__ out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < q;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint8_t c = cq[t];
        const uint64_t k = kq[t];
        uint64_t r = ~0ull;
        if (k <= n) {
            if (c == '$') {
                uint64_t sum = 0;
                for (uint32_t x = 0; x < 4; ++x) sum += dict_rank(blk, sb, x, k);
                r = k - sum;  // reading R12
            } else {
                const uint8_t code = code_of[c];
                if (code < 4) r = dict_rank(blk, sb, code, k);
            }
        }
        out[t] = r;
    }
}

cudaError_t launch_rank_batch(Profiler& prof, cudaStream_t s, const Blk* blk, const uint64_t* sb,
                              uint64_t n, const uint8_t* code_of, const uint8_t* c,
                              const uint64_t* k, uint64_t q, uint64_t* out) {
    if (q == 0) return cudaSuccess;
    SB_LAUNCH(prof, s, "rank_query", 49.0 * q, q,
              rank_batch_kernel<<<grid_for(q, 256, 148u * 64u), 256, 0, s>>>(blk, sb, n, code_of,
                                                                             c, k, q, out));
    return cudaGetLastError();
}

__global__ void decode_kernel(const Blk* __restrict__ blk, uint64_t n,
                              const uint8_t* __restrict__ sym_ascii, uint8_t* __restrict__ out) {
    const uint8_t a0 = sym_ascii[0], a1 = sym_ascii[1], a2 = sym_ascii[2], a3 = sym_ascii[3];
    const uint64_t nb = (n + 63) >> 6;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = blk[b].lo, hi = blk[b].hi, dl = blk[b].dol;
        const uint64_t base = b << 6;
        const uint32_t cnt = (uint32_t)min((uint64_t)64, n - base);
        for (uint32_t t = 0; t < cnt; ++t) {
            uint8_t ch;
            if ((dl >> t) & 1ull) {
                ch = '$';
            } else {
                const uint32_t c = (uint32_t)(((lo >> t) & 1ull) | (((hi >> t) & 1ull) << 1));
                ch = c == 0 ? a0 : c == 1 ? a1 : c == 2 ? a2 : a3;
            }
            out[base + t] = ch;
        }
    }
}

cudaError_t launch_decode(Profiler& prof, cudaStream_t s, const Blk* blk, uint64_t n,
                          const uint8_t* sym_ascii, uint8_t* out) {
    if (n == 0) return cudaSuccess;
    SB_LAUNCH(prof, s, "decode", 1.5 * n, n,
              decode_kernel<<<grid_for((n + 63) >> 6, 128, 148u * 64u), 128, 0, s>>>(blk, n,
                                                                                  sym_ascii, out));
    return cudaGetLastError();
}

__global__ void bint_ascii_kernel(const uint8_t* __restrict__ bint, uint32_t n,
                                  const uint8_t* __restrict__ sym_ascii, uint8_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint8_t b = bint[i];
        out[i] = (b & 4) ? (uint8_t)'$' : sym_ascii[b & 3];
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
