// microbench.cu -- roofline microbenchmarks of SURVEY §8(d) N16, measured on
// the GPU box beside the bench (tools/microbench.sh writes the JSON to
// profiles/).  Standalone: nvcc -O3 -gencode arch=compute_100a,code=sm_100a.
//
//   hbm_copy          128-bit streaming copy over 2 x 2 GiB (cross-check of
//                     MEASURED_PEAKS.json)
//   gather32_hbm      one random 32-byte-aligned 32-byte load per thread over
//                     a 2 GiB buffer (the practical ceiling of ComputeRanks'
//                     dictionary reads when B_ext does not fit L2)
//   gather32_l2       the same over 48 MiB (c2's B_ext is L2-resident)
//   gather4_hbm       random 4-byte loads over 512 MiB (the gather's g reads)
//   red_l2            random u32 atomicAdd without return into 2^24 counters
//   atom_l2           random u32 atomicAdd with return into 2^24 counters
//   scatter4          random-permutation 4-byte stores into 64 MiB
//   pcie_h2d/d2h      pinned cudaMemcpyAsync of 1 GiB
//   zc_gather32       random 32-byte loads from mapped pinned host memory
//                     (the c5 host-tier ComputeRanks ceiling)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__global__ void copy_kernel(const uint4* __restrict__ a, uint4* __restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}

// q queries, each one 32-byte load (two 16-byte halves of the same sector)
__global__ void gather32_kernel(const uint4* __restrict__ buf, uint64_t nsec, uint64_t q,
                                uint64_t seed, uint64_t* __restrict__ sink) {
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = mix(i ^ seed) % nsec;
        const uint4 x = __ldg(buf + 2 * s), y = __ldg(buf + 2 * s + 1);
        acc += x.x ^ y.w;
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

__global__ void gather4_kernel(const uint32_t* __restrict__ buf, uint64_t n, uint64_t q,
                               uint64_t seed, uint64_t* __restrict__ sink) {
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q;
         i += (uint64_t)gridDim.x * blockDim.x)
        acc += __ldg(buf + mix(i ^ seed) % n);
    if (acc == 0x123456789ull) sink[0] = acc;
}

__global__ void red_kernel(uint32_t* __restrict__ cnt, uint32_t nb, uint64_t q, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q;
         i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + (uint32_t)(mix(i ^ seed) % nb), 1u);
}

__global__ void atom_kernel(uint32_t* __restrict__ cnt, uint32_t nb, uint64_t q, uint64_t seed,
                            uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = atomicAdd(cnt + (uint32_t)(mix(i ^ seed) % nb), 1u);
}

// i -> (a*i + c) mod 2^k is a permutation: random-looking distinct stores
__global__ void scatter4_kernel(uint32_t* __restrict__ out, uint32_t logn) {
    const uint32_t n = 1u << logn, mask = n - 1;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t j = (i * 2654435761u + 12345u) & mask;
        const uint32_t k = ((j >> 7) | (j << (logn - 7))) & mask;  // rotate: spread consecutive i
        out[k] = i;
    }
}

struct Timer {
    cudaEvent_t a, b;
    Timer() {
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
    }
    void start() { CK(cudaEventRecord(a)); }
    float stop() {
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        return ms;
    }
};

template <class F>
static float best_of(int reps, F f) {
    Timer t;
    f();  // warm-up
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        t.start();
        f();
        const float ms = t.stop();
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
    const int grid = sms * 16, nt = 256;
    uint64_t* sink;
    CK(cudaMalloc(&sink, 64));
    printf("{\n  \"sms\": %d, \"l2_bytes\": %d,\n", sms, l2);

    {  // HBM copy
        const uint64_t bytes = 2ull << 30;
        uint4 *a, *b;
        CK(cudaMalloc(&a, bytes));
        CK(cudaMalloc(&b, bytes));
        CK(cudaMemset(a, 1, bytes));
        const float ms = best_of(10, [&] { copy_kernel<<<grid * 4, nt>>>(a, b, bytes / 16); });
        printf("  \"hbm_copy_gbs\": %.1f,\n", 2.0 * bytes / ms / 1e6);
        CK(cudaFree(b));
        // random 32-byte gathers over the same 2 GiB
        const uint64_t q = 1ull << 26;
        const float g = best_of(10, [&] { gather32_kernel<<<grid * 4, nt>>>(a, bytes / 32, q, 7, sink); });
        printf("  \"gather32_hbm_gsectors_s\": %.2f, \"gather32_hbm_gbs\": %.1f,\n", q / g / 1e6,
               32.0 * q / g / 1e6);
        const float g4 = best_of(10, [&] {
            gather4_kernel<<<grid * 4, nt>>>(reinterpret_cast<const uint32_t*>(a), (512ull << 20) / 4, q,
                                             9, sink);
        });
        printf("  \"gather4_512MiB_gloads_s\": %.2f,\n", q / g4 / 1e6);
        // L2-resident random gathers (48 MiB window of the same buffer)
        const float gl = best_of(10, [&] {
            gather32_kernel<<<grid * 4, nt>>>(a, (48ull << 20) / 32, q, 11, sink);
        });
        printf("  \"gather32_l2_48MiB_gsectors_s\": %.2f, \"gather32_l2_48MiB_gbs\": %.1f,\n",
               q / gl / 1e6, 32.0 * q / gl / 1e6);
        // random 4-byte loads over growing footprints: where random reads stop
        // hitting L2 (the gather's g array is 4 B x block suffixes)
        printf("  \"gather4_by_footprint_gloads_s\": {");
        const int mbs[] = {16, 32, 48, 64, 80, 96, 112, 128, 256};
        for (int k = 0; k < 9; ++k) {
            const uint64_t n4 = ((uint64_t)mbs[k] << 20) / 4;
            const float t = best_of(10, [&] {
                gather4_kernel<<<grid * 4, nt>>>(reinterpret_cast<const uint32_t*>(a), n4, q, 17 + k, sink);
            });
            printf("%s\"%d\": %.1f", k ? ", " : "", mbs[k], q / t / 1e6);
        }
        printf("},\n");
        CK(cudaFree(a));
    }
    {  // atomics into 2^24 counters (64 MiB, L2-resident)
        const uint32_t nb = 1u << 24;
        const uint64_t q = 1ull << 24;
        uint32_t *cnt, *out;
        CK(cudaMalloc(&cnt, nb * 4ull));
        CK(cudaMalloc(&out, q * 4));
        CK(cudaMemset(cnt, 0, nb * 4ull));
        const float r = best_of(10, [&] { red_kernel<<<grid * 4, nt>>>(cnt, nb, q, 3); });
        printf("  \"red_2p24_counters_gops\": %.2f,\n", q / r / 1e6);
        const float at = best_of(10, [&] { atom_kernel<<<grid * 4, nt>>>(cnt, nb, q, 5, out); });
        printf("  \"atom_2p24_counters_gops\": %.2f,\n", q / at / 1e6);
        const float s4 = best_of(10, [&] { scatter4_kernel<<<grid * 4, nt>>>(out, 24); });
        printf("  \"scatter4_64MiB_gstores_s\": %.2f,\n", q / s4 / 1e6);
        CK(cudaFree(cnt));
        CK(cudaFree(out));
    }
    {  // PCIe
        const uint64_t bytes = 1ull << 30;
        void *h, *d;
        CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
        CK(cudaMalloc(&d, bytes));
        memset(h, 1, bytes);
        const float h2d = best_of(5, [&] { CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice)); });
        const float d2h = best_of(5, [&] { CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost)); });
        printf("  \"pcie_h2d_gbs\": %.1f, \"pcie_d2h_gbs\": %.1f,\n", bytes / h2d / 1e6, bytes / d2h / 1e6);
        void* hd;
        CK(cudaHostGetDevicePointer(&hd, h, 0));
        const uint64_t q = 1ull << 22;
        const float zc = best_of(5, [&] {
            gather32_kernel<<<grid * 4, nt>>>(reinterpret_cast<const uint4*>(hd), bytes / 32, q, 13, sink);
        });
        printf("  \"zc_gather32_msectors_s\": %.1f, \"zc_gather32_gbs\": %.2f\n", q / zc / 1e3,
               32.0 * q / zc / 1e6);
        CK(cudaFreeHost(h));
        CK(cudaFree(d));
    }
    printf("}\n");
    return 0;
}
