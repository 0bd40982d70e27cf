// ldprobe.cu -- DRAM / L2 sectors moved per random 32-byte (or 4-byte) read
// on B200 for different load flavours (ld.global.nc, .cg, .cs, .lu,
// L1::no_allocate, L2::evict_first).  Run under ncu to read
// dram__sectors_read / lts__t_sectors_srcunit_tex_op_read per kernel.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33; return x;
}

template <int MODE>
__global__ void rd32(const uint4* __restrict__ buf, uint64_t nsec, uint64_t q, uint64_t* sink) {
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = mix(i * 0x9E3779B97F4A7C15ull + 7) % nsec;
        const void* p = buf + 2 * s;
        uint64_t w0, w1, w2, w3;
        if (MODE == 0)
            asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(p));
        else if (MODE == 1)
            asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(p));
        else if (MODE == 2)
            asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(p));
        else if (MODE == 3)
            asm volatile("ld.global.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(p));
        else if (MODE == 4)
            asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(p));
        else
            asm volatile("ld.global.cv.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(p));
        acc += w0 ^ w1 ^ w2 ^ w3;
    }
    if (acc == 7) sink[0] = acc;
}

template <int MODE>
__global__ void rd4(const uint32_t* __restrict__ buf, uint64_t n, uint64_t q, uint64_t* sink) {
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = mix(i * 0x9E3779B97F4A7C15ull + 11) % n;
        uint32_t w;
        if (MODE == 0) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(w) : "l"(buf + s));
        else asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(w) : "l"(buf + s));
        acc += w;
    }
    if (acc == 7) sink[0] = acc;
}

int main() {
    const uint64_t bytes = 1ull << 30;  // 1 GiB table (>> L2)
    const uint64_t q = 1ull << 27;      // 134 M random reads
    uint4* buf;
    uint64_t* sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, 64);
    cudaMemset(buf, 1, bytes);
    const uint64_t nsec = bytes / 32;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("%-28s %8.3f ms  %6.1f G reads/s\n", name, best, q / best / 1e6);
    };
    const int G = 148 * 8, T = 256;
    run("rd32 nc", [&] { rd32<0><<<G, T>>>(buf, nsec, q, sink); });
    run("rd32 cg", [&] { rd32<1><<<G, T>>>(buf, nsec, q, sink); });
    run("rd32 cs", [&] { rd32<2><<<G, T>>>(buf, nsec, q, sink); });
    run("rd32 L1::no_allocate", [&] { rd32<3><<<G, T>>>(buf, nsec, q, sink); });
    run("rd32 nc no_alloc evict_first", [&] { rd32<4><<<G, T>>>(buf, nsec, q, sink); });
    run("rd32 cv", [&] { rd32<5><<<G, T>>>(buf, nsec, q, sink); });
    run("rd4 nc", [&] { rd4<0><<<G, T>>>((const uint32_t*)buf, bytes / 4, q, sink); });
    run("rd4 cg", [&] { rd4<1><<<G, T>>>((const uint32_t*)buf, bytes / 4, q, sink); });
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
