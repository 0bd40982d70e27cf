// pack.cu -- A0: ingest an append into the packed slot layout (common.cuh),
// validating every byte against the alphabet, and the greedy block partition.
//
// Alg.1 P:55 iterates "for each block S_jk"; P:46-49 partitions the strings
// into K blocks of roughly M suffixes (reading R8: a block ends at the first
// string boundary where it holds >= M suffixes).
#include <algorithm>

#include "internal.h"

namespace setbwte {

// slot_off[j] = offsets[j] + j; flags non-CSR offsets; gfirst[g] = the string
// owning slot 32g (each string writes the groups that start inside it); the
// terminator bitmap gets string j's last slot (term must be zero on entry).
__global__ void slot_off_kernel(const uint64_t* __restrict__ off, uint64_t m, uint64_t n_bytes,
                                uint64_t n_slots, uint64_t* __restrict__ slot_off,
                                uint32_t* __restrict__ gfirst, uint32_t* __restrict__ term,
                                int* __restrict__ bad) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j <= m;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t o = off[j];
        slot_off[j] = o + j;
        if (j == 0 && o != 0) *bad = 1;
        if (j == m && o != n_bytes) *bad = 1;
        if (j < m) {
            const uint64_t o1 = off[j + 1];
            if (o1 < o) {
                *bad = 1;
                continue;
            }
            const uint64_t a = o + j, e = o1 + j + 1;  // slots [a, e)
            for (uint64_t g = (a + 31) >> 5; (g << 5) < e; ++g) gfirst[g] = (uint32_t)j;
            if (e - 1 < n_slots) atomicOr(term + ((e - 1) >> 5), 1u << (31 - ((e - 1) & 31)));
        }
    }
}

// One warp per 1024 slots (32 groups of 32): the warp stages the <= 1024
// ASCII bytes of its slots in shared memory with 16-byte loads, then packs
// the groups one after the other, one slot per lane: a slot's string (hence
// its byte position, slot minus the terminators before it) comes from the
// terminator bitmap, and the group's two text words are two warp OR
// reductions (lane q keeps group q's words for one coalesced store).
constexpr int kPackWarps = 8;
__global__ void __launch_bounds__(kPackWarps * 32) pack_kernel(
    const uint8_t* __restrict__ bytes, uint64_t n_bytes, const uint32_t* __restrict__ gfirst,
    uint64_t m, uint64_t n_slots, const uint8_t* __restrict__ code_of_g,
    uint32_t* __restrict__ text, const uint32_t* __restrict__ term, uint32_t* __restrict__ nbit,
    unsigned long long* __restrict__ err_pos, uint64_t g_begin, uint64_t g_end) {
    // nbit (sigma = 5): code 4 is stored as 2-bit code 0 plus a set nbit bit
    const uint32_t maxc = nbit ? 4u : 3u;
    constexpr uint32_t kWin = 1024 + 80;
    __shared__ __align__(16) uint8_t sbuf[kPackWarps][kWin];
    __shared__ uint8_t code_of[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) code_of[i] = code_of_g[i];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* sb = sbuf[wib];
    const uint64_t nw = (uint64_t)gridDim.x * kPackWarps;
    for (uint64_t wbase = (g_begin << 5) + (((uint64_t)blockIdx.x * kPackWarps + wib) << 10);
         wbase < (g_end << 5); wbase += nw << 10) {
        const uint64_t g = (wbase >> 5) + lane;
        const bool gv = g < g_end;
        const uint32_t tw = gv ? term[g] : 0u;
        // terminators before this lane's group, within the warp's 1024 slots
        uint32_t rel = __popc(tw);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, rel, d);
            if (lane >= (uint32_t)d) rel += y;
        }
        rel -= __popc(tw);
        const uint64_t j0 = min((uint64_t)gfirst[wbase >> 5], m - 1);
        const uint64_t bp_first = wbase - min(j0, wbase);
        const uint64_t al = bp_first & ~15ull;
        for (uint32_t k = lane; k < kWin / 16; k += 32) {
            const uint64_t a = al + 16ull * k;
            if (a + 16 <= n_bytes) {
                *reinterpret_cast<uint4*>(sb + 16 * k) = __ldg(reinterpret_cast<const uint4*>(bytes + a));
            } else {
                for (int q = 0; q < 16; ++q) sb[16 * k + q] = a + q < n_bytes ? bytes[a + q] : 0;
            }
        }
        __syncwarp();
        uint32_t my_w0 = 0, my_w1 = 0, my_nb = 0;
        // window index of slot (q, lane) = its byte position - al, where the
        // byte position is slot - j0 - terminators before it; 32-bit bounds:
        // slots below n_slots, bytes below n_bytes and inside the window
        const uint32_t l0 = (uint32_t)(bp_first - al) + lane;
        const uint32_t slot_lim = (uint32_t)min(n_slots - min(n_slots, wbase), (uint64_t)1024);
        const uint32_t win_lim = (uint32_t)min(n_bytes - min(n_bytes, al), (uint64_t)kWin);
#pragma unroll 4
        for (uint32_t q = 0; q < 32; ++q) {
            const uint32_t twq = __shfl_sync(0xFFFFFFFFu, tw, q);
            const uint32_t relq = __shfl_sync(0xFFFFFFFFu, rel, q);
            const uint32_t before = lane ? __popc(twq >> (32 - lane)) : 0u;
            const uint32_t li = l0 + 32u * q - relq - before;
            const bool is_t = (twq >> (31 - lane)) & 1u;
            uint32_t code = 0;
            bool n5 = false;
            if (!is_t && 32u * q + lane < slot_lim && li < win_lim) {
                const uint32_t c = code_of[sb[li]];
                if (c > maxc) atomicMin(err_pos, (unsigned long long)(al + li));
                else if (c == 4) n5 = true;
                else code = c;
            }
            const uint32_t v = code << (30 - 2 * (lane & 15));
            const uint32_t w0 = __reduce_or_sync(0xFFFFFFFFu, lane < 16 ? v : 0u);
            const uint32_t w1 = __reduce_or_sync(0xFFFFFFFFu, lane < 16 ? 0u : v);
            const uint32_t nb = __brev(__ballot_sync(0xFFFFFFFFu, n5));
            if (lane == q) {
                my_w0 = w0;
                my_w1 = w1;
                my_nb = nb;
            }
        }
        if (gv) {
            reinterpret_cast<uint2*>(text)[g] = make_uint2(my_w0, my_w1);
            if (nbit) nbit[g] = my_nb;
        }
        __syncwarp();
    }
}

cudaError_t launch_pack_prepare(Profiler& prof, cudaStream_t s, const uint64_t* d_off, uint64_t m,
                                uint64_t n_bytes, Packed pk, int* d_bad_offsets) {
    const uint64_t n_groups = (pk.n_slots + 31) >> 5;
    // the terminator bitmap (and its zero padding) is written here, by bit
    SB_CHECK(cudaMemsetAsync(pk.term, 0, (n_groups + 4) * sizeof(uint32_t), s));
    SB_LAUNCH(prof, s, "slot_offsets", 16.0 * (m + 1), m + 1,
              slot_off_kernel<<<grid_for(m + 1, 256), 256, 0, s>>>(
                  d_off, m, n_bytes, pk.n_slots, pk.slot_off, pk.gfirst, pk.term, d_bad_offsets));
    SB_CHECK(cudaGetLastError());
    // padding words past the end must read as zero
    SB_CHECK(cudaMemsetAsync(pk.text + 2 * n_groups, 0, 4 * sizeof(uint32_t), s));
    if (pk.nbit) SB_CHECK(cudaMemsetAsync(pk.nbit + n_groups, 0, 4 * sizeof(uint32_t), s));
    return cudaSuccess;
}

cudaError_t launch_pack_range(Profiler& prof, cudaStream_t s, const uint8_t* d_bytes,
                              uint64_t m, uint64_t n_bytes, const uint8_t* d_code_of, Packed pk,
                              uint64_t g_begin, uint64_t g_end, unsigned long long* d_err_pos) {
    if (g_end <= g_begin) return cudaSuccess;
    const uint64_t slots = std::min(g_end << 5, pk.n_slots) - (g_begin << 5);
    // algorithmic bytes: 1 B read per base + 3 bits written per slot
    const uint64_t n_warps = ((g_end - g_begin) + 31) >> 5;
    SB_LAUNCH(prof, s, "pack", 1.375 * (double)slots, slots,
              pack_kernel<<<grid_for(n_warps, kPackWarps, 148u * 16u), kPackWarps * 32, 0, s>>>(
                  d_bytes, n_bytes, pk.gfirst, m, pk.n_slots, d_code_of, pk.text, pk.term,
                  pk.nbit, d_err_pos, g_begin, g_end));
    return cudaGetLastError();
}

cudaError_t launch_pack(Profiler& prof, cudaStream_t s, const uint8_t* d_bytes,
                        const uint64_t* d_off, uint64_t m, uint64_t n_bytes,
                        const uint8_t* d_code_of, Packed pk, unsigned long long* d_err_pos,
                        int* d_bad_offsets) {
    SB_CHECK(launch_pack_prepare(prof, s, d_off, m, n_bytes, pk, d_bad_offsets));
    return launch_pack_range(prof, s, d_bytes, m, n_bytes, d_code_of, pk, 0,
                             (pk.n_slots + 31) >> 5, d_err_pos);
}

__global__ void partition_kernel(const uint64_t* __restrict__ slot_off, uint64_t m, uint64_t M,
                                 uint64_t* __restrict__ bounds, uint64_t* __restrict__ k_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint64_t k = 0, j0 = 0;
    bounds[0] = 0;
    bounds[1] = 0;
    while (j0 < m) {
        const uint64_t target = slot_off[j0] + M;
        // first j1 > j0 with slot_off[j1] >= target, else m
        uint64_t lo = j0 + 1, hi = m;
        if (slot_off[m] < target) {
            lo = m;
        } else {
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (slot_off[mid] >= target) hi = mid; else lo = mid + 1;
            }
        }
        ++k;
        bounds[2 * k] = lo;
        bounds[2 * k + 1] = slot_off[lo];
        j0 = lo;
    }
    *k_out = k;
}

cudaError_t launch_partition(Profiler& prof, cudaStream_t s, const uint64_t* d_slot_off,
                             uint64_t m, uint64_t M, uint64_t* d_bounds, uint64_t* d_k) {
    SB_LAUNCH(prof, s, "partition", 0, 0,
              partition_kernel<<<1, 32, 0, s>>>(d_slot_off, m, M, d_bounds, d_k));
    return cudaGetLastError();
}

__global__ void slices_kernel(const uint64_t* __restrict__ slot_off, uint64_t j0, uint64_t j1,
                              const uint64_t* __restrict__ bounds, int parts,
                              uint64_t* __restrict__ out) {
    // one CTA per block: block k = strings [bounds[2k], bounds[2k+2]) when
    // bounds is given (the whole append's partition), else [j0, j1)
    if (bounds) {
        j0 = bounds[2 * blockIdx.x];
        j1 = bounds[2 * blockIdx.x + 2];
    }
    out += (uint64_t)blockIdx.x * 2 * (parts + 1);
    const int r = threadIdx.x;
    if (r > parts) return;
    const uint64_t S0 = slot_off[j0], S1 = slot_off[j1];
    const uint64_t target = S0 + (S1 - S0) * (uint64_t)r / (uint64_t)parts;
    uint64_t lo = j0, hi = j1;  // first j in [j0, j1] with slot_off[j] >= target
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (slot_off[mid] >= target) hi = mid; else lo = mid + 1;
    }
    const uint64_t j = r == parts ? j1 : lo;
    out[r] = j;
    out[parts + 1 + r] = slot_off[j];
}

cudaError_t launch_slices(Profiler& prof, cudaStream_t s, const uint64_t* d_slot_off,
                          uint64_t j0, uint64_t j1, int parts, uint64_t* d_out) {
    SB_LAUNCH(prof, s, "slices", 0, 0,
              slices_kernel<<<1, 1024, 0, s>>>(d_slot_off, j0, j1, nullptr, parts, d_out));
    return cudaGetLastError();
}

cudaError_t launch_slices_blocks(Profiler& prof, cudaStream_t s, const uint64_t* d_slot_off,
                                 const uint64_t* d_bounds, uint64_t K, int parts,
                                 uint64_t* d_out) {
    if (K == 0) return cudaSuccess;
    SB_LAUNCH(prof, s, "slices", 0, 0,
              slices_kernel<<<(unsigned)K, 1024, 0, s>>>(d_slot_off, 0, 0, d_bounds, parts, d_out));
    return cudaGetLastError();
}

}  // namespace setbwte
