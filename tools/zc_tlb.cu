// zero-copy random 32-byte reads over mapped pinned host buffers of growing size
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <sys/mman.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
__global__ void g32(const uint4* buf, uint64_t nsec, uint64_t q, uint64_t seed, uint64_t* sink) {
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = mix(i ^ seed) % nsec;
        uint64_t w0, w1, w2, w3;
        asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(buf + 2 * s));
        acc += w0 ^ w3;
    }
    if (acc == 7) sink[0] = acc;
}
int main() {
    uint64_t* sink; cudaMalloc(&sink, 64);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const uint64_t q = 1ull << 22;
    const int gbs[] = {256, 1024, 3072, 6144};
    for (int huge = 0; huge < 2; ++huge)
    for (int k = 0; k < 4; ++k) {
        const uint64_t bytes = (uint64_t)gbs[k] << 20;
        void* h = nullptr;
        if (huge) {
            h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
            madvise(h, bytes, MADV_HUGEPAGE);
            memset(h, 1, bytes);
            if (cudaHostRegister(h, bytes, cudaHostRegisterMapped) != cudaSuccess) { printf("register failed\n"); return 1; }
        } else {
            if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped) != cudaSuccess) { printf("alloc failed\n"); return 1; }
            memset(h, 1, bytes);
        }
        void* d; cudaHostGetDevicePointer(&d, h, 0);
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(a);
            g32<<<148 * 16, 256>>>((const uint4*)d, bytes / 32, q, 13 + r, sink);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf("%s %5d MB: %.1f M sectors/s\n", huge ? "thp+register" : "hostalloc", gbs[k], q / best / 1e3);
        if (huge) { cudaHostUnregister(h); munmap(h, bytes); } else cudaFreeHost(h);
    }
    return 0;
}
