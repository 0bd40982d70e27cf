// sort.cu -- A1 ConstructSA: MSD radix suffix sort of one block with
// unique-key sieving (Sec.3; Alg.1).
//
// Suffixes are "long integer keys made of multiple 32-bit words": key
// word d of the suffix at slot p is suffix_key(p, d) (common.cuh, reading R6).
// The sort refines SEGMENTS -- ranges of the final suffix array whose members
// agree on every key bit examined so far and are stored in slot order:
//
// * a LARGE segment (> kCapB members) takes one stable 8-bit digit pass
//   (histogram -> per-segment scan -> stable scatter) and splits into
//   children;
// * a SMALL segment (<= kCapB) is finished by one CTA in shared memory: a
//   bitonic sort of (run, key word, index) composites, repeated on the
//   still-tied runs with the next key word until none is left;
// * a bucket is SIEVED -- written to its final place and dropped from the
//   working set -- when it has one member, or when its members end inside the
//   key window with equal keys (identical suffixes, already in slot order =
//   string-index order).  This is the "sieves unique keys at each
//   iteration" of P:89 (reading R7).
//
// Ties are only ever broken by slot order, which the stable passes and the
// index field of the composites preserve, so the result is the unique SA of
// the block (reading R15).
#include <algorithm>

#include "internal.h"

namespace setbwte {

namespace {

constexpr uint32_t kCapA = 256;    // small class A: <= 256 members, 128 threads
constexpr uint32_t kNtA = 128;
constexpr uint32_t kCapB = 4096;   // small class B: <= 4096 members, 512 threads
constexpr uint32_t kNtB = 512;
constexpr uint32_t kChunk = 16384; // target chunk of a digit pass
constexpr uint32_t kMaxChunks = 1024;
constexpr int kDigNt = 256;        // digit-pass CTA
constexpr int kDigIpt = 8;
constexpr int kDigTile = kDigNt * kDigIpt;
constexpr int kDigWarps = kDigNt / 32;

struct Seg {
    uint32_t start, len, word, meta;  // meta: shift | buf << 8 | keys_valid << 9
};
struct SegX {
    uint32_t chunk_base, nchunks, chunk_len, skip;
};
struct Chunk {
    uint32_t seg, begin, end, pad;
};
// device counters
enum { C_LARGE_IN = 0, C_LARGE_OUT, C_SMALL_A, C_SMALL_B, C_CHUNKS, C_ACTIVE, C_N };

__device__ __forceinline__ uint32_t meta_shift(uint32_t m) { return m & 0xFF; }
__device__ __forceinline__ uint32_t meta_buf(uint32_t m) { return (m >> 8) & 1; }
__device__ __forceinline__ uint32_t meta_kv(uint32_t m) { return (m >> 9) & 1; }
__device__ __forceinline__ uint32_t make_meta(uint32_t shift, uint32_t buf, uint32_t kv) {
    return shift | (buf << 8) | (kv << 9);
}

__device__ __forceinline__ void emit_child(const Seg& c, Seg* large_out, Seg* small_a,
                                           Seg* small_b, uint32_t* ctr) {
    if (c.len <= kCapA) {
        small_a[atomicAdd(ctr + C_SMALL_A, 1u)] = c;
    } else if (c.len <= kCapB) {
        small_b[atomicAdd(ctr + C_SMALL_B, 1u)] = c;
    } else {
        large_out[atomicAdd(ctr + C_LARGE_OUT, 1u)] = c;
    }
}

__global__ void sort_init_kernel(uint32_t* __restrict__ sa0, uint32_t* __restrict__ saf,
                                 uint32_t n, Seg* large_in, Seg* small_a, Seg* small_b,
                                 uint32_t* ctr) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        sa0[i] = (uint32_t)i;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int c = 0; c < C_N; ++c) ctr[c] = 0;
        if (n == 1) {
            saf[0] = 0;
        } else if (n > 1) {
            Seg s{0u, n, 0u, make_meta(24, 0, 0)};
            if (n <= kCapA) small_a[ctr[C_SMALL_A]++] = s;
            else if (n <= kCapB) small_b[ctr[C_SMALL_B]++] = s;
            else large_in[ctr[C_LARGE_IN]++] = s;
        }
    }
}

// Split each large segment into <= kMaxChunks chunks of ~kChunk members.
__global__ void chunkify_kernel(const Seg* __restrict__ segs, SegX* __restrict__ segx,
                                Chunk* __restrict__ chunks, uint32_t* ctr) {
    const uint32_t n = ctr[C_LARGE_IN];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const Seg s = segs[i];
        uint32_t nch = (s.len + kChunk - 1) / kChunk;
        nch = nch > kMaxChunks ? kMaxChunks : nch;
        const uint32_t clen = (s.len + nch - 1) / nch;
        nch = (s.len + clen - 1) / clen;
        const uint32_t base = atomicAdd(ctr + C_CHUNKS, nch);
        atomicAdd(ctr + C_ACTIVE, s.len);
        segx[i] = SegX{base, nch, clen, 0u};
        for (uint32_t c = 0; c < nch; ++c) {
            const uint32_t b = s.start + c * clen;
            const uint32_t e = min(b + clen, s.start + s.len);
            chunks[base + c] = Chunk{i, b, e, 0u};
        }
    }
}

// Pass 1 of a digit pass: per-chunk histogram of the current 8-bit digit.
// Computes (and caches) the key word when the segment's keys are stale.
__global__ void __launch_bounds__(kDigNt) digit_hist_kernel(
    const Seg* __restrict__ segs, const Chunk* __restrict__ chunks, const uint32_t* ctr,
    uint32_t* __restrict__ sa0, uint32_t* __restrict__ sa1, uint32_t* __restrict__ k0,
    uint32_t* __restrict__ k1, const uint32_t* __restrict__ text,
    const uint32_t* __restrict__ term, uint64_t base, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    const uint32_t nch = ctr[C_CHUNKS];
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
        h[threadIdx.x] = 0;
        __syncthreads();
        const Chunk ch = chunks[c];
        const Seg s = segs[ch.seg];
        const uint32_t shift = meta_shift(s.meta);
        const uint32_t buf = meta_buf(s.meta);
        const bool kv = meta_kv(s.meta);
        const uint32_t* S = buf ? sa1 : sa0;
        uint32_t* K = buf ? k1 : k0;
        for (uint32_t p0 = ch.begin; p0 < ch.end; p0 += kDigNt) {
            const uint32_t p = p0 + threadIdx.x;
            const bool valid = p < ch.end;
            uint32_t d = 0x100;
            if (valid) {
                uint32_t key;
                if (kv) {
                    key = K[p];
                } else {
                    key = suffix_key(text, term, base + S[p], s.word);
                    K[p] = key;
                }
                d = (key >> shift) & 0xFF;
            }
            const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
            if (valid && lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&h[d], (uint32_t)__popc(peers));
        }
        __syncthreads();
        hist[(size_t)c * 256 + threadIdx.x] = h[threadIdx.x];
        __syncthreads();
    }
}

// Pass 2: per segment, exclusive scan of the chunk histograms, digit bases,
// sieve decisions and child segments.
__global__ void __launch_bounds__(256) digit_scan_kernel(
    const Seg* __restrict__ segs, SegX* __restrict__ segx, uint32_t* __restrict__ hist,
    uint32_t* __restrict__ dbase, Seg* large_out, Seg* small_a, Seg* small_b, uint32_t* ctr) {
    __shared__ uint32_t wsum[8];
    __shared__ int all_one;
    const uint32_t n = ctr[C_LARGE_IN];
    const uint32_t d = threadIdx.x, lane = d & 31, warp = d >> 5;
    for (uint32_t si = blockIdx.x; si < n; si += gridDim.x) {
        const Seg s = segs[si];
        const SegX x = segx[si];
        uint32_t run = 0;
        for (uint32_t c = x.chunk_base; c < x.chunk_base + x.nchunks; ++c) {
            const size_t idx = (size_t)c * 256 + d;
            const uint32_t v = hist[idx];
            hist[idx] = run;
            run += v;
        }
        if (d == 0) all_one = 0;
        // exclusive scan of run over the 256 digits
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        uint32_t wpre = 0;
        for (uint32_t w = 0; w < warp; ++w) wpre += wsum[w];
        const uint32_t excl = wpre + incl - run;
        if (run == s.len) all_one = 1;
        __syncthreads();
        const uint32_t shift = meta_shift(s.meta);
        const uint32_t buf = meta_buf(s.meta);
        const bool resolved = (run == 1) || (shift == 0 && (d & 15u) < (uint32_t)kKeySyms);
        uint32_t flag = 0;
        if (run > 0) {
            if (resolved) {
                flag = 0x80000000u;
            } else {
                Seg c;
                c.start = s.start + excl;
                c.len = run;
                const uint32_t cbuf = all_one ? buf : 1u - buf;
                if (shift == 0) {
                    c.word = s.word + 1;
                    c.meta = make_meta(24, cbuf, 0);
                } else {
                    c.word = s.word;
                    c.meta = make_meta(shift - 8, cbuf, 1);
                }
                emit_child(c, large_out, small_a, small_b, ctr);
                if (all_one) segx[si].skip = 1;
            }
        }
        dbase[(size_t)si * 256 + d] = (s.start + excl) | flag;
        __syncthreads();
    }
}

// Pass 3: stable scatter of each chunk by digit.  Sieved buckets go straight
// to the final SA, the others to the segment's other buffer.
__global__ void __launch_bounds__(kDigNt) digit_scatter_kernel(
    const Seg* __restrict__ segs, const SegX* __restrict__ segx, const Chunk* __restrict__ chunks,
    const uint32_t* ctr, const uint32_t* __restrict__ hist, const uint32_t* __restrict__ dbase,
    uint32_t* __restrict__ sa0, uint32_t* __restrict__ sa1, uint32_t* __restrict__ k0,
    uint32_t* __restrict__ k1, uint32_t* __restrict__ saf) {
    __shared__ uint32_t run_base[256];
    __shared__ uint32_t tile_cnt[256];
    __shared__ uint8_t fin[256];
    __shared__ uint32_t wcnt[kDigWarps][256];
    const uint32_t nch = ctr[C_CHUNKS];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
        const Chunk ch = chunks[c];
        if (segx[ch.seg].skip) continue;  // uniform across the CTA
        const Seg s = segs[ch.seg];
        const uint32_t shift = meta_shift(s.meta);
        const uint32_t buf = meta_buf(s.meta);
        const uint32_t* S = buf ? sa1 : sa0;
        const uint32_t* K = buf ? k1 : k0;
        uint32_t* S2 = buf ? sa0 : sa1;
        uint32_t* K2 = buf ? k0 : k1;
        const uint32_t db = dbase[(size_t)ch.seg * 256 + tid];
        run_base[tid] = (db & 0x7FFFFFFFu) + hist[(size_t)c * 256 + tid];
        fin[tid] = (uint8_t)(db >> 31);
        for (int w = 0; w < kDigWarps; ++w) wcnt[w][tid] = 0;
        __syncthreads();
        for (uint32_t t0 = ch.begin; t0 < ch.end; t0 += kDigTile) {
            uint32_t key[kDigIpt], slot[kDigIpt], dig[kDigIpt], lrank[kDigIpt];
#pragma unroll
            for (int it = 0; it < kDigIpt; ++it) {
                const uint32_t p = t0 + warp * (32 * kDigIpt) + it * 32 + lane;
                const bool valid = p < ch.end;
                key[it] = valid ? K[p] : 0u;
                slot[it] = valid ? S[p] : 0u;
                dig[it] = valid ? ((key[it] >> shift) & 0xFFu) : 0x100u;
                const uint32_t peers = __match_any_sync(0xFFFFFFFFu, dig[it]);
                const uint32_t leader = __ffs(peers) - 1;
                const uint32_t prior = __popc(peers & ((1u << lane) - 1u));
                uint32_t b = 0;
                if (valid && lane == leader) {
                    b = wcnt[warp][dig[it]];
                    wcnt[warp][dig[it]] = b + __popc(peers);
                }
                b = __shfl_sync(0xFFFFFFFFu, b, leader);
                lrank[it] = b + prior;
                __syncwarp();  // order the leader's wcnt update before the next item's read
            }
            __syncthreads();
            {
                uint32_t acc = 0;
                for (int w = 0; w < kDigWarps; ++w) {
                    const uint32_t t = wcnt[w][tid];
                    wcnt[w][tid] = acc;
                    acc += t;
                }
                tile_cnt[tid] = acc;
            }
            __syncthreads();
#pragma unroll
            for (int it = 0; it < kDigIpt; ++it) {
                if (dig[it] > 0xFFu) continue;
                const uint32_t dp = run_base[dig[it]] + wcnt[warp][dig[it]] + lrank[it];
                if (fin[dig[it]]) {
                    saf[dp] = slot[it];
                } else {
                    S2[dp] = slot[it];
                    K2[dp] = key[it];
                }
            }
            __syncthreads();
            run_base[tid] += tile_cnt[tid];
            for (int w = 0; w < kDigWarps; ++w) wcnt[w][tid] = 0;
            __syncthreads();
        }
    }
}

// Block-wide inclusive max-scan of a[0..P) (P elements, NT threads).
template <int NT>
__device__ void block_max_scan(uint16_t* a, uint32_t P, uint32_t* aux) {
    const uint32_t per = (P + NT - 1) / NT;
    const uint32_t b = threadIdx.x * per;
    const uint32_t e = min(b + per, P);
    uint32_t m = 0;
    for (uint32_t i = b; i < e; ++i) {
        m = max(m, (uint32_t)a[i]);
        a[i] = (uint16_t)m;
    }
    aux[threadIdx.x] = m;
    __syncthreads();
    for (uint32_t o = 1; o < NT; o <<= 1) {
        const uint32_t v = threadIdx.x >= o ? aux[threadIdx.x - o] : 0u;
        __syncthreads();
        aux[threadIdx.x] = max(aux[threadIdx.x], v);
        __syncthreads();
    }
    const uint32_t pre = threadIdx.x > 0 ? aux[threadIdx.x - 1] : 0u;
    for (uint32_t i = b; i < e; ++i) a[i] = (uint16_t)max((uint32_t)a[i], pre);
    __syncthreads();
}

template <int CAP, int NT>
constexpr size_t local_sort_smem() {
    return (size_t)CAP * (8 + 4 + 2 + 1) + (size_t)NT * 4 + 16;
}

// Finish a small segment in shared memory (all remaining key words).
template <int CAP, int NT>
__global__ void __launch_bounds__(NT) local_sort_kernel(
    const Seg* __restrict__ list, const uint32_t* ctr, int which, const uint32_t* __restrict__ sa0,
    const uint32_t* __restrict__ sa1, uint32_t* __restrict__ saf,
    const uint32_t* __restrict__ text, const uint32_t* __restrict__ term, uint64_t base) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* comp = reinterpret_cast<unsigned long long*>(smem_raw);
    uint32_t* slot = reinterpret_cast<uint32_t*>(comp + CAP);
    uint32_t* aux = slot + CAP;
    uint16_t* run = reinterpret_cast<uint16_t*>(aux + NT);
    uint8_t* act = reinterpret_cast<uint8_t*>(run + CAP);
    constexpr int IDXB = 12;  // index / run-start field width (CAP <= 4096)
    static_assert(CAP <= (1 << IDXB), "CAP too large for the composite");
    const uint32_t n = ctr[which];
    for (uint32_t si = blockIdx.x; si < n; si += gridDim.x) {
        const Seg s = list[si];
        const uint32_t len = s.len;
        uint32_t P = 2;
        while (P < len) P <<= 1;
        const uint32_t* S = meta_buf(s.meta) ? sa1 : sa0;
        for (uint32_t i = threadIdx.x; i < len; i += NT) {
            slot[i] = S[s.start + i];
            run[i] = 0;
            act[i] = 1;
        }
        __syncthreads();
        uint32_t word = s.word;
        for (;;) {
            for (uint32_t i = threadIdx.x; i < P; i += NT) {
                unsigned long long cmp;
                if (i < len) {
                    if (act[i]) {
                        const uint32_t key = suffix_key(text, term, base + slot[i], word);
                        cmp = ((unsigned long long)run[i] << (32 + IDXB)) |
                              ((unsigned long long)key << IDXB) | i;
                    } else {
                        cmp = ((unsigned long long)i << (32 + IDXB)) | i;
                    }
                } else {
                    cmp = ~0ull;
                }
                comp[i] = cmp;
            }
            __syncthreads();
            // bitonic sort of comp[0..P)
            for (uint32_t k = 2; k <= P; k <<= 1) {
                for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                    for (uint32_t t = threadIdx.x; t < (P >> 1); t += NT) {
                        const uint32_t i = 2 * t - (t & (j - 1));
                        const uint32_t q = i + j;
                        const unsigned long long a = comp[i], b = comp[q];
                        const bool up = (i & k) == 0;
                        if ((a > b) == up) {
                            comp[i] = b;
                            comp[q] = a;
                        }
                    }
                    __syncthreads();
                }
            }
            // permute slots; derive new tied runs
            uint32_t newslot[(CAP + NT - 1) / NT];
            int r = 0;
            for (uint32_t i = threadIdx.x; i < len; i += NT, ++r)
                newslot[r] = slot[comp[i] & ((1u << IDXB) - 1)];
            __syncthreads();
            r = 0;
            bool any = false;
            for (uint32_t i = threadIdx.x; i < len; i += NT, ++r) {
                slot[i] = newslot[r];
                const unsigned long long hi = comp[i] >> IDXB;
                const bool eqp = i > 0 && (comp[i - 1] >> IDXB) == hi;
                const bool eqn = i + 1 < len && (comp[i + 1] >> IDXB) == hi;
                const uint32_t key = (uint32_t)(hi & 0xFFFFFFFFull);
                const bool a = (eqp || eqn) && ((key & 15u) == (uint32_t)kKeySyms);
                act[i] = a;
                any |= a;
                run[i] = eqp ? 0 : (uint16_t)i;
            }
            __syncthreads();
            if (!__syncthreads_or(any)) break;
            block_max_scan<NT>(run, len, aux);
            ++word;
        }
        for (uint32_t i = threadIdx.x; i < len; i += NT) saf[s.start + i] = slot[i];
        __syncthreads();
    }
}

__global__ void sort_advance_kernel(uint32_t* ctr) {
    ctr[C_LARGE_IN] = ctr[C_LARGE_OUT];
    ctr[C_LARGE_OUT] = 0;
    ctr[C_CHUNKS] = 0;
}

__global__ void sort_zero_small_kernel(uint32_t* ctr) {
    ctr[C_SMALL_A] = 0;
    ctr[C_SMALL_B] = 0;
}

}  // namespace

cudaError_t sort_block(Profiler& prof, cudaStream_t s, SortScratch& ws, const uint32_t* text,
                       const uint32_t* term, uint64_t slot_base, uint32_t n_suf,
                       uint32_t* d_sa_final, SortStats* st) {
    if (n_suf == 0) return cudaSuccess;
    uint32_t *sa0, *sa1, *k0, *k1, *hist, *ctr, *dbase;
    Seg *la, *lb, *sma, *smb;
    Chunk* chunks;
    const size_t n = n_suf;
    const size_t max_large = n / (kCapB + 1) + 1;
    const size_t max_chunks = n / kChunk + max_large + 1;
    SB_CHECK(ensure(ws.sa0, n, &sa0));
    SB_CHECK(ensure(ws.sa1, n, &sa1));
    SB_CHECK(ensure(ws.k0, n, &k0));
    SB_CHECK(ensure(ws.k1, n, &k1));
    // segs_a / segs_b each hold: Seg[max_large] + SegX[max_large] + dbase[max_large*256]
    const size_t seg_bytes = max_large * (sizeof(Seg) + sizeof(SegX) + 256 * sizeof(uint32_t));
    uint8_t *ra, *rb;
    SB_CHECK(ensure(ws.segs_a, seg_bytes, &ra));
    SB_CHECK(ensure(ws.segs_b, seg_bytes, &rb));
    SB_CHECK(ensure(ws.small_a, n / 2 + 1, &sma));
    SB_CHECK(ensure(ws.small_b, n / (kCapA + 1) + 1, &smb));
    SB_CHECK(ensure(ws.chunks, max_chunks, &chunks));
    SB_CHECK(ensure(ws.hist, max_chunks * 256, &hist));
    SB_CHECK(ensure(ws.ctr, 16, &ctr));
    la = reinterpret_cast<Seg*>(ra);
    lb = reinterpret_cast<Seg*>(rb);
    SegX* segx = reinterpret_cast<SegX*>(ra + max_large * sizeof(Seg));
    dbase = reinterpret_cast<uint32_t*>(ra + max_large * (sizeof(Seg) + sizeof(SegX)));

    SB_LAUNCH(prof, s, "sort_init", 4.0 * n, n,
              sort_init_kernel<<<grid_for(n, 256), 256, 0, s>>>(sa0, d_sa_final, n_suf, la, sma,
                                                                 smb, ctr));
    SB_CHECK(cudaGetLastError());
    const unsigned g_small = 148u * 16u;
    constexpr size_t smem_a = local_sort_smem<kCapA, kNtA>();
    constexpr size_t smem_b = local_sort_smem<kCapB, kNtB>();
    static bool attr_done = false;
    if (!attr_done) {
        SB_CHECK(cudaFuncSetAttribute(local_sort_kernel<kCapA, kNtA>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a));
        SB_CHECK(cudaFuncSetAttribute(local_sort_kernel<kCapB, kNtB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b));
        attr_done = true;
    }
    uint32_t prev_active = 0;
    const unsigned g_dig = 148u * 8u;
    uint32_t h_ctr[C_N];
    for (;;) {
        // finish every small segment produced so far
        SB_LAUNCH(prof, s, "local_sort_a", 0, 0,
                  (local_sort_kernel<kCapA, kNtA><<<g_small, kNtA, smem_a, s>>>(
                      sma, ctr, C_SMALL_A, sa0, sa1, d_sa_final, text, term, slot_base)));
        SB_CHECK(cudaGetLastError());
        SB_LAUNCH(prof, s, "local_sort_b", 0, 0,
                  (local_sort_kernel<kCapB, kNtB><<<148u * 3u, kNtB, smem_b, s>>>(
                      smb, ctr, C_SMALL_B, sa0, sa1, d_sa_final, text, term, slot_base)));
        SB_CHECK(cudaGetLastError());
        SB_LAUNCH(prof, s, "sort_ctl", 0, 0, sort_zero_small_kernel<<<1, 1, 0, s>>>(ctr));
        SB_CHECK(cudaMemcpyAsync(h_ctr, ctr, sizeof(h_ctr), cudaMemcpyDeviceToHost, s));
        SB_CHECK(cudaStreamSynchronize(s));
        if (st && st->digit_passes > 0) {
            st->active_per_pass.push_back((uint32_t)(h_ctr[C_ACTIVE] - prev_active));
            prev_active = h_ctr[C_ACTIVE];
        }
        if (h_ctr[C_LARGE_IN] == 0) break;
        // one stable 8-bit digit pass over every large segment
        SB_LAUNCH(prof, s, "sort_chunkify", 0, 0,
                  chunkify_kernel<<<grid_for(h_ctr[C_LARGE_IN], 128), 128, 0, s>>>(la, segx, chunks,
                                                                                  ctr));
        SB_CHECK(cudaGetLastError());
        SB_LAUNCH(prof, s, "digit_hist", 0, 0,
                  digit_hist_kernel<<<g_dig, kDigNt, 0, s>>>(la, chunks, ctr, sa0, sa1, k0, k1,
                                                             text, term, slot_base, hist));
        SB_CHECK(cudaGetLastError());
        SB_LAUNCH(prof, s, "digit_scan", 0, 0,
                  digit_scan_kernel<<<grid_for(h_ctr[C_LARGE_IN], 1, 148u * 8u), 256, 0, s>>>(
                      la, segx, hist, dbase, lb, sma, smb, ctr));
        SB_CHECK(cudaGetLastError());
        SB_LAUNCH(prof, s, "digit_scatter", 0, 0,
                  digit_scatter_kernel<<<g_dig, kDigNt, 0, s>>>(la, segx, chunks, ctr, hist,
                                                                dbase, sa0, sa1, k0, k1,
                                                                d_sa_final));
        SB_CHECK(cudaGetLastError());
        SB_LAUNCH(prof, s, "sort_ctl", 0, 0, sort_advance_kernel<<<1, 1, 0, s>>>(ctr));
        SB_CHECK(cudaGetLastError());
        if (st) {
            st->digit_passes++;
        }
        std::swap(la, lb);
        std::swap(ra, rb);
        segx = reinterpret_cast<SegX*>(ra + max_large * sizeof(Seg));
        dbase = reinterpret_cast<uint32_t*>(ra + max_large * (sizeof(Seg) + sizeof(SegX)));
    }
    if (st) st->rounds++;
    return cudaSuccess;
}

}  // namespace setbwte
