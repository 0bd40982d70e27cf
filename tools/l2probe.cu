// l2probe.cu -- does a bucket-ordered random gather hit L2 on B200?
// out[k] = g[slot[k]], slot bucket-sorted (each bucket a window of W bytes of g).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void fetch_ldg(const uint32_t* __restrict__ slot, const uint32_t* __restrict__ g,
                          uint32_t n, uint32_t* __restrict__ out) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        out[k] = __ldg(g + __ldcs(slot + k));
}
__global__ void fetch_plain(const uint32_t* __restrict__ slot, const uint32_t* g,
                            uint32_t n, uint32_t* __restrict__ out) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        out[k] = g[slot[k]];
}
// block-contiguous: each block handles a contiguous chunk of k
__global__ void fetch_chunk(const uint32_t* __restrict__ slot, const uint32_t* __restrict__ g,
                            uint32_t n, uint32_t* __restrict__ out, uint32_t per) {
    const uint32_t b0 = blockIdx.x * per, b1 = min(n, b0 + per);
    for (uint32_t k = b0 + threadIdx.x; k < b1; k += blockDim.x)
        out[k] = __ldg(g + __ldcs(slot + k));
}

int main(int argc, char** argv) {
    const uint32_t n = 1u << 27;
    const int shift = argc > 1 ? atoi(argv[1]) : 23;
    if (argc > 2) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[2]));
        size_t v = 0;
        cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
        printf("set L2 fetch granularity %s -> %zu (%s)\n", argv[2], v, cudaGetErrorString(e));
    } else {
        size_t v = 0;
        cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
        printf("default L2 fetch granularity %zu\n", v);
    }
    std::vector<uint32_t> h(n);
    std::mt19937_64 rng(1);
    for (uint32_t i = 0; i < n; ++i) h[i] = (uint32_t)(rng() % n);
    // stable bucket sort by slot >> shift
    std::stable_sort(h.begin(), h.end(), [&](uint32_t a, uint32_t b) { return (a >> shift) < (b >> shift); });
    uint32_t *ds, *dg, *dout;
    cudaMalloc(&ds, 4ull * n); cudaMalloc(&dg, 4ull * n); cudaMalloc(&dout, 4ull * n);
    cudaMemcpy(ds, h.data(), 4ull * n, cudaMemcpyHostToDevice);
    cudaMemset(dg, 1, 4ull * n);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a); fetch_ldg<<<148 * 8, 256>>>(ds, dg, n, dout); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("shift %d ldg   %.3f ms\n", shift, ms);
        cudaEventRecord(a); fetch_plain<<<148 * 8, 256>>>(ds, dg, n, dout); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("shift %d plain %.3f ms\n", shift, ms);
        const uint32_t nbk = 148 * 64, per = (n + nbk - 1) / nbk;
        cudaEventRecord(a); fetch_chunk<<<nbk, 256>>>(ds, dg, n, dout, per); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("shift %d chunk %.3f ms\n", shift, ms);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
