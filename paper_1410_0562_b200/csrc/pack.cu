// pack.cu -- A0: ingest an append into the packed slot layout (common.cuh),
// validating every byte against the alphabet, and the greedy block partition.
//
// Alg.1 P:55 iterates "for each block S_jk"; P:46-49 partitions the strings
// into K blocks of roughly M suffixes (reading R8: a block ends at the first
// string boundary where it holds >= M suffixes).
#include "internal.h"

namespace setbwte {

// slot_off[j] = offsets[j] + j; flags non-CSR offsets.
__global__ void slot_off_kernel(const uint64_t* __restrict__ off, uint64_t m, uint64_t n_bytes,
                                uint64_t* __restrict__ slot_off, int* __restrict__ bad) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j <= m;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t o = off[j];
        slot_off[j] = o + j;
        if (j == 0 && o != 0) *bad = 1;
        if (j == m && o != n_bytes) *bad = 1;
        if (j < m && off[j + 1] < o) *bad = 1;
    }
}

// One thread per 32 slots: two text words + one terminator word.
__global__ void pack_kernel(const uint8_t* __restrict__ bytes, uint64_t n_bytes,
                            const uint64_t* __restrict__ slot_off, uint64_t m, uint64_t n_slots,
                            const uint8_t* __restrict__ code_of, uint32_t* __restrict__ text,
                            uint32_t* __restrict__ term, unsigned long long* __restrict__ err_pos) {
    const uint64_t n_groups = (n_slots + 31) >> 5;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n_groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s0 = g << 5;
        // largest j with slot_off[j] <= s0
        uint64_t lo = 0, hi = m;  // invariant: slot_off[lo] <= s0 < slot_off[hi] (when valid)
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (slot_off[mid] <= s0) lo = mid; else hi = mid;
        }
        uint64_t j = lo;
        uint64_t next = slot_off[j + 1];
        uint32_t w0 = 0, w1 = 0, tw = 0;
        const int cnt = (int)min((uint64_t)32, n_slots - s0);
        for (int t = 0; t < cnt; ++t) {
            const uint64_t s = s0 + t;
            while (s >= next && j + 1 < m) { ++j; next = slot_off[j + 1]; }
            uint32_t code = 0;
            if (s == next - 1) {
                tw |= 1u << (31 - t);
            } else {
                const uint64_t bp = s - j;  // byte position: slots minus terminators before
                if (bp < n_bytes) {
                    const uint8_t c = code_of[bytes[bp]];
                    if (c > 3) atomicMin(err_pos, (unsigned long long)bp); else code = c;
                }
            }
            if (t < 16) w0 |= code << (30 - 2 * t); else w1 |= code << (30 - 2 * (t - 16));
        }
        text[2 * g] = w0;
        text[2 * g + 1] = w1;
        term[g] = tw;
    }
}

cudaError_t launch_pack(Profiler& prof, cudaStream_t s, const uint8_t* d_bytes,
                        const uint64_t* d_off, uint64_t m, uint64_t n_bytes,
                        const uint8_t* d_code_of, Packed pk, unsigned long long* d_err_pos,
                        int* d_bad_offsets) {
    SB_LAUNCH(prof, s, "slot_offsets", 16.0 * (m + 1), m + 1,
              slot_off_kernel<<<grid_for(m + 1, 256), 256, 0, s>>>(d_off, m, n_bytes, pk.slot_off,
                                                                   d_bad_offsets));
    SB_CHECK(cudaGetLastError());
    const uint64_t n_groups = (pk.n_slots + 31) >> 5;
    // padding words past the end must read as zero
    SB_CHECK(cudaMemsetAsync(pk.text + 2 * n_groups, 0, 4 * sizeof(uint32_t), s));
    SB_CHECK(cudaMemsetAsync(pk.term + n_groups, 0, 4 * sizeof(uint32_t), s));
    // algorithmic bytes: 1 B read per base + 3 bits written per slot
    SB_LAUNCH(prof, s, "pack", (double)n_bytes + 0.375 * pk.n_slots, n_bytes,
              pack_kernel<<<grid_for(n_groups, 256, 148u * 64u), 256, 0, s>>>(
                  d_bytes, n_bytes, pk.slot_off, m, pk.n_slots, d_code_of, pk.text, pk.term,
                  d_err_pos));
    return cudaGetLastError();
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
                              int parts, uint64_t* __restrict__ out) {
    const int r = threadIdx.x;
    if (r > parts) return;
    const uint64_t S0 = slot_off[j0], S1 = slot_off[j1];
    const uint64_t target = S0 + (S1 - S0) * (uint64_t)r / (uint64_t)parts;
    uint64_t lo = j0, hi = j1;  // first j in [j0, j1] with slot_off[j] >= target
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (slot_off[mid] >= target) hi = mid; else lo = mid + 1;
    }
    out[r] = r == parts ? j1 : lo;
}

cudaError_t launch_slices(Profiler& prof, cudaStream_t s, const uint64_t* d_slot_off,
                          uint64_t j0, uint64_t j1, int parts, uint64_t* d_out) {
    SB_LAUNCH(prof, s, "slices", 0, 0,
              slices_kernel<<<1, 1024, 0, s>>>(d_slot_off, j0, j1, parts, d_out));
    return cudaGetLastError();
}

}  // namespace setbwte
