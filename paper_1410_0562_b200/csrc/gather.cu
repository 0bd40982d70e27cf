// gather.cu -- A4 g -> g_sa gather (Alg.1), bucketed so that the
// random reads of g hit L2.
//
// g is indexed by slot (string-major, the order ComputeRanks walks it) and is
// read in SA order: g_sa[i] = g[SA_int[i]], pos[i] = g_sa[i] + i (reading R4).
// For a block whose g does not fit in L2 (c3: 2^27 suffixes x 4 B = 512 MB)
// every read is a random 32-byte DRAM sector for 4 useful bytes -- the plain
// gather (ranks.cu) runs at the random-sector rate.  Here the permutation is
// applied in three coalesced passes instead:
//
//   A  partition: the SA entries of each tile of 4096 positions are split
//      stably by slot bucket (slot >> shift, each bucket's g slice <= 32 MB);
//      tile t's members of bucket d go to tmp[base[d] + row[d][t] + rank]
//      (row = exclusive scan of the per-tile counts over the tiles);
//   B  fetch: tmp2[k] = g[tmp[k]] in k order -- at any moment the resident
//      CTAs read inside one or two buckets, whose g slice sits in L2;
//   C  final: each tile recomputes the same stable ranks and reads its
//      elements' g values back from tmp2 (contiguous runs, one per bucket),
//      then writes pos, B_int and the superblock slices exactly as the plain
//      gather does.
//
// Algorithmic bytes: the stage keeps the plain gather's
// count (4 B SA + gw B g + gw B pos + 1 B B_int per suffix); the extra passes
// are the price of coalescing and show up as time, not as credited bytes.
#include <stdlib.h>

#include <algorithm>

#include "blockrank.cuh"
#include "internal.h"

namespace setbwte {
namespace {

constexpr int kGbNt = 512;
constexpr int kGbIpt = 8;
constexpr uint32_t kGbTile = kGbNt * kGbIpt;  // 4096 SA positions per tile

__device__ __forceinline__ uint32_t item_index(uint32_t tid, int it) {
    return (tid >> 5) * (32 * kGbIpt) + it * 32 + (tid & 31);
}

// per tile and bucket: member count, digit-major (cnt[d * ntiles + t])
template <int NB>
__global__ void __launch_bounds__(kGbNt) gb_hist_kernel(const uint32_t* __restrict__ sa,
                                                        uint32_t smask, uint32_t n,
                                                        uint32_t shift, uint32_t nb,
                                                        uint32_t ntiles,
                                                        uint32_t* __restrict__ cnt) {
    __shared__ uint32_t h[256];
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        if (threadIdx.x < 256) h[threadIdx.x] = 0;
        __syncthreads();
        const uint32_t t0 = t * kGbTile;
#pragma unroll
        for (int it = 0; it < kGbIpt; ++it) {
            const uint32_t i = t0 + item_index(threadIdx.x, it);
            if (i < n) atomicAdd(&h[(__ldcs(sa + i) & smask) >> shift], 1u);
        }
        __syncthreads();
        if (threadIdx.x < nb) cnt[(size_t)threadIdx.x * ntiles + t] = h[threadIdx.x];
        __syncthreads();
    }
}

// exclusive scan of each bucket's row over the tiles (one CTA per bucket);
// tot[d] = the bucket's size
__global__ void __launch_bounds__(1024) gb_rows_kernel(uint32_t* __restrict__ cnt, uint32_t ntiles,
                                                       uint32_t* __restrict__ tot) {
    __shared__ uint32_t ws[32];
    __shared__ uint32_t carry;
    uint32_t* row = cnt + (size_t)blockIdx.x * ntiles;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t c0 = 0; c0 < ntiles; c0 += 1024) {
        const uint32_t i = c0 + threadIdx.x;
        const uint32_t v = i < ntiles ? row[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        if (warp == 0) {
            const uint32_t w = ws[lane];
            uint32_t z = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, z, o);
                if (lane >= (uint32_t)o) z += y;
            }
            ws[lane] = z - w;
        }
        __syncthreads();
        const uint32_t base = carry;
        if (i < ntiles) row[i] = base + ws[warp] + x - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry = base + ws[31] + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) tot[blockIdx.x] = carry;
}

// Load one tile of SA entries, its digits, and rank them stably by bucket.
// off[d] (shared) = where the tile's first member of bucket d goes in tmp,
// minus its tile-local sorted position.
template <int NB>
__device__ __forceinline__ void gb_tile(const uint32_t* __restrict__ sa, uint32_t smask,
                                        uint32_t n, uint32_t shift, uint32_t nb, uint32_t ntiles,
                                        const uint32_t* __restrict__ row,
                                        const uint32_t* __restrict__ tot, uint32_t t,
                                        uint32_t (&e)[kGbIpt], uint32_t (&dig)[kGbIpt],
                                        uint32_t (&dest)[kGbIpt], uint32_t* wcnt, uint32_t* dstart,
                                        uint32_t* tmp, uint32_t* off) {
    const uint32_t t0 = t * kGbTile;
#pragma unroll
    for (int it = 0; it < kGbIpt; ++it) {
        const uint32_t i = t0 + item_index(threadIdx.x, it);
        e[it] = i < n ? __ldg(sa + i) : 0u;
        dig[it] = i < n ? (e[it] & smask) >> shift : (1u << NB);
    }
    block_rank<kGbNt, kGbIpt, NB>(dig, dest, wcnt, dstart, tmp);
    if (threadIdx.x < nb) {
        // bucket base: the sizes of the lower buckets (nb <= 256 totals)
        uint32_t b = 0;
        for (uint32_t q = 0; q < threadIdx.x; ++q) b += tot[q];
        off[threadIdx.x] = b + row[(size_t)threadIdx.x * ntiles + t] - dstart[threadIdx.x];
    }
    __syncthreads();
}

template <int NB, class G>
__global__ void __launch_bounds__(kGbNt) gb_part_kernel(const uint32_t* __restrict__ sa,
                                                        uint32_t smask, uint32_t n,
                                                        uint32_t shift, uint32_t nb,
                                                        uint32_t ntiles,
                                                        const uint32_t* __restrict__ row,
                                                        const uint32_t* __restrict__ tot,
                                                        uint32_t* __restrict__ out,
                                                        G* __restrict__ kpos) {
    __shared__ uint32_t wcnt[(kGbNt / 32) * 256];
    __shared__ uint32_t dstart[260], tmp[32], off[256];
    __shared__ uint32_t s_slot[kGbTile];
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        uint32_t e[kGbIpt], dig[kGbIpt], dest[kGbIpt];
        gb_tile<NB>(sa, smask, n, shift, nb, ntiles, row, tot, t, e, dig, dest, wcnt, dstart, tmp,
                    off);
        // every element's place k in the partition, in SA order: the final
        // pass reads g_sa[i] back from there without ranking again
        const uint32_t t0 = t * kGbTile;
#pragma unroll
        for (int it = 0; it < kGbIpt; ++it)
            if (dig[it] < (1u << NB)) {
                s_slot[dest[it]] = e[it] & smask;
                __stcs(kpos + t0 + item_index(threadIdx.x, it), (G)(off[dig[it]] + dest[it]));
            }
        __syncthreads();
        // coalesced write-out: a bucket's members of the tile are one run
        const uint32_t tn = min(kGbTile, n - t * kGbTile);
        for (uint32_t k = threadIdx.x; k < tn; k += kGbNt) {
            const uint32_t sl = s_slot[k];
            __stcs(out + off[sl >> shift] + k, sl);
        }
        __syncthreads();
    }
}

// tmp2[k] = g[slot[k]] in k order (the g reads stay inside one bucket's
// slice).  ONE wave of CTAs (148 x 8 resident), one element per thread per
// step, walking k with the grid stride.  Measured (ncu, c3 block, 2^27
// suffixes): this form reads 1.1 GB of DRAM at 61 % L2 hits; a 4x-unrolled
// grid-stride form with two waves of CTAs read 12.4 GB, and 4 loads per
// thread inside per-CTA chunks of 1024 read 11.3 GB -- more loads in flight
// per thread defeat the L2 reuse on this part.
template <class G>
__global__ void __launch_bounds__(256) gb_fetch_kernel(const uint32_t* __restrict__ slot,
                                                       const G* __restrict__ g, uint32_t n,
                                                       G* __restrict__ out) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        __stcs(out + k, __ldg(g + __ldcs(slot + k)));
}

// pos, B_int and sb_start from the fetched g values (the tail of gather_kernel):
// pos[i] holds the element's place k in the partition (gb_part_kernel), so
// g_sa[i] = gval[k] -- a streaming pass, no ranking.
template <class G>
__global__ void __launch_bounds__(256) gb_final_kernel(
    const uint32_t* __restrict__ sa, uint32_t smask, uint32_t n, const G* __restrict__ gv_b,
    const G* __restrict__ g, G* __restrict__ pos, uint8_t* __restrict__ bint,
    uint64_t* __restrict__ sb_start, uint64_t nsb, const uint8_t* __restrict__ bslot, bool bing,
    const uint32_t* __restrict__ text, const uint32_t* __restrict__ term,
    const uint32_t* __restrict__ nbit, uint64_t slot_base) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t iters = (n + stride - 1) / stride;  // warp-uniform trip count
    for (uint64_t itr = 0; itr < iters; ++itr) {
        const uint64_t i = itr * stride + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
        const bool v = i < n;
        uint64_t pv = 0;
        if (v) {
            const uint32_t e = __ldcs(sa + i);
            const uint64_t k = (uint64_t)__ldcs(pos + i);
            uint64_t gvv = (uint64_t)__ldg(gv_b + k);  // evict-normal: neighbours reuse the sector
            const uint8_t bg = (uint8_t)(gvv >> 56);
            if (bing) gvv &= (1ull << 56) - 1ull;
            pv = gvv + i;
            __stcs(pos + i, (G)pv);
            const uint32_t sl = e & smask;
            uint8_t b;
            if (bing) {
                b = bg;
            } else if (smask != 0xFFFFFFFFu) {
                b = (uint8_t)(e >> kPayloadShift);
            } else if (bslot) {
                b = __ldg(bslot + sl);
            } else {
                const uint64_t p = slot_base + sl;
                if (sl == 0 || term_bit(term, p - 1)) b = 4;
                else if (nbit && term_bit(nbit, p - 1)) b = 5;
                else b = (uint8_t)text_sym(text, p - 1);
            }
            if (b == 5) b = 12;  // code 4 of sigma = 5: '$' flag + N flag
            __stcs(reinterpret_cast<signed char*>(bint) + i, (signed char)b);
        }
        if (sb_start) {
            uint64_t prev = __shfl_up_sync(0xFFFFFFFFu, pv, 1);
            if (v) {
                if (lane == 0 && i > 0) {
                    const uint32_t sl1 = sa[i - 1] & smask;
                    uint64_t g1 = (uint64_t)__ldg(g + sl1);
                    if (bing) g1 &= (1ull << 56) - 1ull;
                    prev = g1 + (i - 1);
                }
                const uint64_t cur = pv >> kSbShift;
                const uint64_t first = i > 0 ? (prev >> kSbShift) + 1 : 0;
                for (uint64_t s = first; s <= cur && s <= nsb; ++s) sb_start[s] = i;
                if (i + 1 == n)
                    for (uint64_t s = cur + 1; s <= nsb; ++s) sb_start[s] = n;
            }
        }
    }
}

template <int NB, class G>
cudaError_t run_bucketed(Profiler& prof, cudaStream_t s, const uint32_t* sa, uint32_t smask,
                         uint32_t n, uint32_t shift, uint32_t nb, const G* g, G* pos,
                         uint8_t* bint, uint64_t* sb_start, uint64_t nsb, const uint8_t* bslot,
                         bool bing, const uint32_t* text, const uint32_t* term,
                         const uint32_t* nbit, uint64_t slot_base, const GatherScratch& ws,
                         double bytes) {
    const uint32_t ntiles = (n + kGbTile - 1) / kGbTile;
    const unsigned grid_t = std::min<uint32_t>(ntiles, 148u * 4u);
    uint32_t* tot = ws.rows + (size_t)nb * ntiles;
    SB_LAUNCH(prof, s, "gather_part", 0, 0,
              (gb_hist_kernel<NB><<<grid_t, kGbNt, 0, s>>>(sa, smask, n, shift, nb, ntiles,
                                                           ws.rows)));
    SB_CHECK(cudaGetLastError());
    SB_LAUNCH(prof, s, "gather_part", 0, 0,
              (gb_rows_kernel<<<nb, 1024, 0, s>>>(ws.rows, ntiles, tot)));
    SB_CHECK(cudaGetLastError());
    SB_LAUNCH(prof, s, "gather_part", 0, 0,
              (gb_part_kernel<NB, G><<<grid_t, kGbNt, 0, s>>>(sa, smask, n, shift, nb, ntiles,
                                                              ws.rows, tot, ws.slot, pos)));
    SB_CHECK(cudaGetLastError());
    G* gv_b = reinterpret_cast<G*>(ws.gval);
    SB_LAUNCH(prof, s, "gather_fetch", 0, 0,
              (gb_fetch_kernel<G><<<148u * 8u, 256, 0, s>>>(ws.slot, g, n, gv_b)));
    SB_CHECK(cudaGetLastError());
    SB_LAUNCH(prof, s, "gather", bytes, n,
              (gb_final_kernel<G><<<grid_for(n, 256, 148u * 8u), 256, 0, s>>>(
                  sa, smask, n, gv_b, g, pos, bint, sb_start, nsb, bslot, bing, text, term, nbit,
                  slot_base)));
    return cudaGetLastError();
}

}  // namespace

size_t gather_scratch_bytes(uint32_t n, int gw) {
    const size_t ntiles = (n + kGbTile - 1) / kGbTile;
    return 4 * ((size_t)n + 256 * ntiles + 256 + 64) + (size_t)gw * n + 256;
}

uint32_t gather_buckets_shift(uint32_t n, int gw, int mode) {
    // mode 1 (auto): only when g does not fit in L2 (> 96 MB); each bucket's
    // g slice <= 32 MB (more buckets than 256 widen the slices instead);
    // mode 2 (forced, tests): at least 8 buckets whatever the size
    if (mode == 0 || n < 2) return 0;
    if (mode == 1 && (uint64_t)n * gw <= (96ull << 20)) return 0;
    int lg = 0;
    while ((1ull << lg) < n) ++lg;  // n <= 2^lg
    int shift = gw == 4 ? 23 : 22;
    if (mode == 2) shift = std::max(0, lg - 3);
    shift = std::max(shift, lg - 8);  // <= 256 buckets
    if (((uint64_t)(n - 1) >> shift) == 0) return 0;  // one bucket: nothing to gain
    return (uint32_t)shift;
}

cudaError_t launch_gather_bucketed(Profiler& prof, cudaStream_t s, const uint32_t* text,
                                   const uint32_t* term, uint64_t slot_base, const uint32_t* sa,
                                   const void* g, uint32_t n_suf, void* pos, int gw,
                                   uint8_t* bint, uint64_t* sb_start, uint64_t nsb,
                                   const uint8_t* bslot, uint64_t payload_limit, bool bing,
                                   const uint32_t* nbit, uint32_t shift,
                                   const GatherScratch& ws) {
    const uint32_t smask = sa_slot_mask(n_suf, payload_limit);
    const uint32_t nb = (uint32_t)(((uint64_t)(n_suf - 1) >> shift) + 1);
    // the plain gather's algorithmic bytes (ranks.cu launch_gather): the
    // random g read counted as one 32-byte sector (g here exceeds L2)
    const double bytes = (5.375 + 32.0 + gw) * n_suf;
    if (nb <= 32) {
        if (gw == 4)
            return run_bucketed<5, uint32_t>(prof, s, sa, smask, n_suf, shift, nb,
                                             (const uint32_t*)g, (uint32_t*)pos, bint, sb_start,
                                             nsb, bslot, false, text, term, nbit, slot_base, ws,
                                             bytes);
        return run_bucketed<5, uint64_t>(prof, s, sa, smask, n_suf, shift, nb, (const uint64_t*)g,
                                         (uint64_t*)pos, bint, sb_start, nsb, bslot, bing, text,
                                         term, nbit, slot_base, ws, bytes);
    }
    if (gw == 4)
        return run_bucketed<8, uint32_t>(prof, s, sa, smask, n_suf, shift, nb, (const uint32_t*)g,
                                         (uint32_t*)pos, bint, sb_start, nsb, bslot, false, text,
                                         term, nbit, slot_base, ws, bytes);
    return run_bucketed<8, uint64_t>(prof, s, sa, smask, n_suf, shift, nb, (const uint64_t*)g,
                                     (uint64_t*)pos, bint, sb_start, nsb, bslot, bing, text, term,
                                     nbit, slot_base, ws, bytes);
}

}  // namespace setbwte
