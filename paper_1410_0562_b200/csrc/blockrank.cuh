// blockrank.cuh -- stable ranking of a tile of items by a small digit
// (shared by the ConstructSA digit passes, sort.cu, and the bucketed gather,
// gather.cu).
#pragma once
#include <stdint.h>

namespace setbwte {

// Lanes of the warp holding the same NB-bit digit (a ballot per bit: short
// fixed latency, unlike MATCH.ANY whose result latency serialised the ranking
// loops -- ncu, profiles/).
template <int NB>
__device__ __forceinline__ uint32_t peers_of(uint32_t d) {
    // per bit: test into a predicate, ballot it, replicate the lane's bit
    // (selp), and fold  diff |= bal ^ rep  in one 3-input LOP3 (LUT 0xF6 =
    // a | (b ^ c)); peers = lanes whose digit has no differing bit = ~diff
    uint32_t diff = 0u;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        asm("{\n\t"
            ".reg .pred p;\n\t"
            ".reg .b32 t, bal, rep;\n\t"
            "and.b32 t, %1, %2;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 bal, p, 0xffffffff;\n\t"
            "selp.b32 rep, 0xffffffff, 0, p;\n\t"
            "lop3.b32 %0, %0, bal, rep, 0xF6;\n\t"
            "}"
            : "+r"(diff)
            : "r"(d), "r"(1u << b));
    }
    return ~diff;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------
// Block-level stable ranking of up to NT*IPT items by an NB-bit digit
// (NB <= 8).  Item `it` of a thread is tile element warp*32*IPT + it*32 + lane;
// invalid items carry digit 1 << NB (0x100 for NB = 8).  On return dest[it]
// is the item's position in the tile stably sorted by digit, dstart[d] the
// first position of digit d (dstart[256] = number of valid items; digits
// >= 2^NB are empty).  wcnt: NW*256 u32 of shared memory.
// ---------------------------------------------------------------------------
template <int NT, int IPT, int NB = 8>
__device__ __forceinline__ void block_rank(const uint32_t (&dig)[IPT], uint32_t (&dest)[IPT],
                                           uint32_t* wcnt, uint32_t* dstart, uint32_t* tmp) {
    static_assert(NB >= 1 && NB <= 8, "digit bits");
    constexpr uint32_t kInvalid = 1u << NB;
    constexpr int NW = NT / 32;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t i = tid; i < NW * 256; i += NT) wcnt[i] = 0;
    __syncthreads();
    uint32_t* mine = wcnt + warp * 256;
    // all MATCH.ANY first (independent, their latency overlaps), then the
    // in-order per-warp counter updates: every lane reads its digit's counter
    // (broadcast among peers), the lowest peer writes it back advanced.
    // peers by ballots (MATCH.ANY measured slower here: MIO-pipe throughput);
    // a full tile has no invalid items and needs only the 8 digit bits
    uint32_t peers[IPT];
    const bool full = __all_sync(0xFFFFFFFFu, dig[IPT - 1] < kInvalid);
#pragma unroll
    for (int it = 0; it < IPT; ++it)
        peers[it] = full ? peers_of<NB>(dig[it]) : peers_of<NB + 1>(dig[it]);
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
        const uint32_t d = dig[it];
        const bool ok = d < kInvalid;
        const uint32_t b = ok ? mine[d] : 0u;
        dest[it] = b + __popc(peers[it] & lt);
        if (ok && (peers[it] & lt) == 0) mine[d] = b + __popc(peers[it]);
        __syncwarp();
    }
    __syncthreads();
    // per digit: prefix over the warps, then an exclusive scan over the 256
    // digits; thread tid owns digits [tid*DPT, tid*DPT+DPT) (NT >= 256: DPT = 1)
    constexpr int DPT = NT >= 256 ? 1 : 256 / NT;
    constexpr int NACT = NT >= 256 ? 256 : NT;  // threads owning digits
    uint32_t tot[DPT];
    uint32_t local = 0;
    if (tid < NACT) {
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            const uint32_t d = tid * DPT + q;
            uint32_t acc = 0;
            for (int w = 0; w < NW; ++w) {
                const uint32_t t = wcnt[w * 256 + d];
                wcnt[w * 256 + d] = acc;
                acc += t;
            }
            tot[q] = acc;
            local += acc;
        }
    }
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31 && tid < NACT) tmp[warp] = incl;
    __syncthreads();
    if (tid < NACT) {
        uint32_t run = incl - local;
        for (uint32_t w = 0; w < warp; ++w) run += tmp[w];
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            dstart[tid * DPT + q] = run;
            run += tot[q];
        }
        if (tid == NACT - 1) dstart[256] = run;
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
        const uint32_t d = dig[it];
        if (d < kInvalid) dest[it] += dstart[d] + mine[d];
    }
}

}  // namespace setbwte
