// gsort_probe.cu -- sizing the "order late blocks by g" idea:
// how long does sorting one c3 block's (g, slot) pairs by g take on this
// B200?  Uses CUB's radix sort (a measurement tool, not the product path):
// 2^27 pairs, g uniform below n_ext (31 bits), slots 0..n-1.
#include <cstdio>
#include <cstdint>
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

__global__ void fill(uint32_t* g, uint32_t* v, uint32_t n, uint32_t nbits) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull + 12345;
        x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33;
        g[i] = (uint32_t)x & ((1u << nbits) - 1u);
        v[i] = i;
    }
}

int main() {
    const uint32_t n = 1u << 27;
    uint32_t *k0, *k1, *v0, *v1;
    cudaMalloc(&k0, 4ull * n); cudaMalloc(&k1, 4ull * n);
    cudaMalloc(&v0, 4ull * n); cudaMalloc(&v1, 4ull * n);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (uint32_t nbits : {28u, 31u}) {
        fill<<<148 * 8, 256>>>(k0, v0, n, nbits);
        cub::DoubleBuffer<uint32_t> K(k0, k1), V(v0, v1);
        size_t tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp, K, V, n, 0, nbits);
        void* dt; cudaMalloc(&dt, tmp);
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
            fill<<<148 * 8, 256>>>(k0, v0, n, nbits);
            cub::DoubleBuffer<uint32_t> K2(k0, k1), V2(v0, v1);
            cudaEventRecord(a);
            cub::DeviceRadixSort::SortPairs(dt, tmp, K2, V2, n, 0, nbits);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("SortPairs 2^27 (u32 key, u32 value), %u key bits: %.3f ms (%.1f G pairs/s)\n",
               nbits, best, n / best / 1e6);
        cudaFree(dt);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
