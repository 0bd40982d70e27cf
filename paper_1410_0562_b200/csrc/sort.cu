// sort.cu -- A1 ConstructSA: MSD radix suffix sort of one block with
// unique-key sieving (Sec.3; Alg.1).
//
// Suffixes are "long integer keys made of multiple 32-bit words": key
// word d of the suffix at slot p is suffix_key(p, d) (common.cuh, reading R6).
// The sort refines SEGMENTS -- ranges of the final suffix array whose members
// agree on every key bit examined so far and are stored in slot order -- by
// size class:
//
//   LARGE  (> 4096)   one stable 8-bit MSD digit pass over all large segments:
//                     per-chunk histogram -> per-segment scan -> stable
//                     scatter staged through shared memory (coalesced runs);
//   SMALL  (33..512)  one warp per segment: stable LSD radix sort of the
//                     still-unknown key bits held in registers, exchanged
//                     through a per-warp shared-memory buffer (no CTA barriers);
//   MEDIUM (513..4096) one CTA per segment: the same LSD radix sort with the
//                     tile in shared memory;
//   TINY   (2..32)    one warp per segment: register bitonic sort across lanes.
//
// After a word is sorted, ties (equal key words whose 14 symbols are all real)
// move to the next word: runs of <= 32 are finished by one warp in registers,
// longer runs become new segments of the next round.  A bucket is SIEVED --
// written to its final place and dropped from the working set -- when it has
// one member, or when its members end inside the key window with equal keys
// (identical suffixes, already in slot order = string-index order).
// This is the "sieves unique keys at each iteration" of P:89 (reading R7).
//
// Ties are only ever broken by slot order, which every pass preserves
// (stable), so the result is the unique SA of the block (reading R15).
#include <stdlib.h>

#include <algorithm>
#include <cstring>

#include "blockrank.cuh"
#include "internal.h"

namespace setbwte {
namespace sortk {

constexpr uint32_t kTiny = 32;
constexpr uint32_t kCapS = 512;    // SMALL: one warp per segment, 16 items per lane
constexpr int kIpl = kCapS / 32;
constexpr int kWarpCta = 8;
constexpr uint32_t kCapM = 4096;   // MEDIUM: 512 threads, 8 items each
constexpr uint32_t kNtM = 512;
constexpr uint32_t kChunk = 16384; // largest chunk of a digit pass
constexpr uint32_t kMinChunk = 2048;
constexpr uint32_t kMaxChunks = 1024;
constexpr uint32_t kGroup = 32;    // chunks per prefix group
#ifndef SB_DIG_NT
#define SB_DIG_NT 512
#endif
#ifndef SB_DIG_IPT
#define SB_DIG_IPT 8
#endif
// SB_SCATTER_L2 (default 1): 0 = the scatter reads its input evict-first and writes the
// next pass's (key, slot) with streaming stores; 1 = plain stores and
// evict-normal reads, so a c2-sized pass can hit L2 in the next one
#ifndef SB_SCATTER_L2
#define SB_SCATTER_L2 1
#endif
constexpr int kDigNt = SB_DIG_NT;  // digit-pass CTA
constexpr int kDigIpt = SB_DIG_IPT;
constexpr int kDigTile = kDigNt * kDigIpt;

// BIT2..BIT16: 33..512 members whose unknown key bits fit in 16 (keys valid,
// shift <= 8): one warp sorts 32*NIT packed (key bits, index) u32 values with a
// register bitonic network.  SMALL: the other 33..512 segments (warp LSD radix).
// LOCALD2 / LOCALD: 513..2048 / 2049..4096 members with valid keys: the
// whole digit pass of the segment in one CTA (local_digit_kernel<256 / 512>).
enum { TINY = 0, BIT2, BIT4, BIT8, BIT16, SMALL, MED1K, MED2K, MEDIUM, LARGE, LOCALD, LOCALD2,
       NCLASS };
// misc counters
enum { M_CHUNKS = 0, M_ACTIVE, M_ELEMS_T, M_ELEMS_S, M_ELEMS_M, M_ELEMS_B, M_GROUPS, M_ACTIVE_LOC,
       M_LOOKUPS, M_N };

struct Seg {
    uint32_t start, len, word, meta;  // meta: shift | buf<<8 | keys_valid<<9 | iota<<10
};
struct SegX {
    uint32_t chunk_base, nchunks, group_base, skip;
};
struct Chunk {
    uint32_t seg, begin, end, group;
};
struct Group {
    uint32_t first_chunk, nchunks;
};
struct Lists {
    Seg* seg[NCLASS];
    uint32_t* cnt;  // NCLASS counters
    uint32_t local;  // 513..4096-member segments with valid keys take the one-CTA pass
};
struct Bufs {
    uint32_t* sa[2];
    uint32_t* key[2];
    uint32_t* saf;
    const uint32_t* text;
    const uint32_t* term;
    uint64_t base;
    uint32_t smask;  // slot bits of an SA entry (sa_slot_mask); ~0 without payload
    uint32_t n;         // suffixes of the block (debug bounds checks)
    const uint32_t* nbit;  // sigma = 5: code-4 plane of the text (common.cuh), else null
    uint32_t ksyms;        // symbols per key word: kKeySyms (14) or kKeySyms5 (9)
};

// Key word `word` of the suffix of an SA entry (text lookups).
__device__ __forceinline__ uint32_t key_of(const Bufs& B, uint32_t entry, uint32_t word) {
    if (B.nbit) return suffix_key5(B.text, B.term, B.nbit, B.base + (entry & B.smask), word);
    return suffix_key(B.text, B.term, B.base + (entry & B.smask), word);
}

// SA entry of block-local slot sl: the slot plus, with payload, its B_int
// symbol (the symbol before the suffix: its code 0..3, 4 = '$' at a string
// start, 5 = code 4 of sigma = 5).
__device__ __forceinline__ uint32_t sa_entry(const Bufs& B, uint32_t sl) {
    if (B.smask == 0xFFFFFFFFu) return sl;
    const uint64_t p = B.base + sl;
    uint32_t b;
    if (sl == 0 || term_bit(B.term, p - 1)) b = 4u;
    else if (B.nbit && term_bit(B.nbit, p - 1)) b = 5u;
    else b = text_sym(B.text, p - 1);
    return sl | (b << kPayloadShift);
}

__device__ __forceinline__ uint32_t meta_shift(uint32_t m) { return m & 0xFF; }
__device__ __forceinline__ uint32_t meta_buf(uint32_t m) { return (m >> 8) & 1; }
__device__ __forceinline__ uint32_t meta_kv(uint32_t m) { return (m >> 9) & 1; }
__device__ __forceinline__ uint32_t meta_iota(uint32_t m) { return (m >> 10) & 1; }
__device__ __forceinline__ uint32_t make_meta(uint32_t shift, uint32_t buf, uint32_t kv,
                                              uint32_t iota = 0) {
    return shift | (buf << 8) | (kv << 9) | (iota << 10);
}
__host__ __device__ __forceinline__ int class_of(const Seg& c, uint32_t local = 1) {
    if (c.len <= kTiny) return TINY;
    if (c.len <= kCapS) {
        if (((c.meta >> 9) & 1) && (c.meta & 0xFF) <= 8)
            return c.len <= 64 ? BIT2 : c.len <= 128 ? BIT4 : c.len <= 256 ? BIT8 : BIT16;
        return SMALL;
    }
    // > 512 with valid keys: one more digit pass is cheaper than a CTA-wide
    // sort (measured on c3's ~2048-member second-pass buckets); up to one
    // tile it runs inside one CTA (no histogram / scan kernels)
    if ((c.meta >> 9) & 1)
        return !local ? LARGE : c.len <= 2048 ? LOCALD2 : c.len <= kCapM ? LOCALD : LARGE;
    return c.len <= 1024 ? MED1K : c.len <= 2048 ? MED2K : c.len <= kCapM ? MEDIUM : LARGE;
}
__device__ __forceinline__ void emit(const Lists& out, const Seg& c) {
    const int k = class_of(c, out.local);
    out.seg[k][atomicAdd(out.cnt + k, 1u)] = c;
}

// ---------------------------------------------------------------------------
// Warp-level finish of a run of L <= 32 suffixes (lanes 0..L-1 hold the slots
// in slot order).  Sorts by key word `word`, then word+1, ... until no ties
// remain, entirely in registers.  Returns the lane's slot in final order.
// ---------------------------------------------------------------------------
// nlook (optional): accumulates (in a register) the key-word lookups
// (random text reads) made.
__device__ __forceinline__ uint32_t warp_finish(uint32_t slot, uint32_t L, uint32_t word,
                                                uint32_t key0, bool have_key, const Bufs& B,
                                                uint32_t group0 = 0, bool active0 = true,
                                                uint32_t* nlook = nullptr) {
    // Several independent runs may be packed into one call: lanes [g, g+len)
    // of each run carry group0 = g (its first lane); runs never mix.  A lane
    // that is not active (or not valid) is a group of its own.
    const uint32_t lane = threadIdx.x & 31;
    const bool valid = lane < L;
    bool active = valid && active0;
    uint32_t group = active ? group0 : lane;
    for (;;) {
        uint32_t key = 0;
        if (active) key = have_key ? key0 : key_of(B, slot, word);
        if (nlook && !have_key && active) ++*nlook;
        have_key = false;
        // group extents: [group, gend)
        const uint32_t starts = __ballot_sync(0xFFFFFFFFu, group == lane);
        const uint32_t above = lane == 31 ? 0u : (starts & (0xFFFFFFFEu << group) & ~((2u << lane) - 1u));
        const uint32_t gend = above ? (uint32_t)(__ffs(above) - 1) : 32u;
        const uint32_t W = __reduce_max_sync(0xFFFFFFFFu, gend - group);
        if (W <= 8) {
            // short runs (the usual case: pairs): stable rank inside the group
            // by comparing with the at most W-1 neighbours on each side, then
            // move slot and key to lane group+rank
            uint32_t rank = 0;
            for (uint32_t d = 1; d < W; ++d) {
                const uint32_t ku = __shfl_up_sync(0xFFFFFFFFu, key, d);
                const uint32_t kd = __shfl_down_sync(0xFFFFFFFFu, key, d);
                if (lane >= group + d && ku <= key) ++rank;
                if (lane + d < gend && kd < key) ++rank;
            }
            const uint32_t dest = group + rank;
            uint32_t ns = slot, nk = key;
            for (int d = -(int)W + 1; d < (int)W; ++d) {
                const uint32_t srcl = (uint32_t)((int)lane + d) & 31u;
                const uint32_t dd = __shfl_sync(0xFFFFFFFFu, dest, srcl);
                const uint32_t ss = __shfl_sync(0xFFFFFFFFu, slot, srcl);
                const uint32_t kk = __shfl_sync(0xFFFFFFFFu, key, srcl);
                if ((int)lane + d >= 0 && (int)lane + d < 32 && dd == lane) {
                    ns = ss;
                    nk = kk;
                }
            }
            slot = ns;
            key = nk;
        } else {
            unsigned long long comp;
            if (!valid) comp = ~0ull;
            else comp = ((unsigned long long)group << 37) | ((unsigned long long)key << 5) | lane;
#pragma unroll
            for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
                for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                    const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, comp, j);
                    const bool up = (lane & k) == 0;
                    const bool lower = (lane & j) == 0;
                    const unsigned long long mn = comp < other ? comp : other;
                    const unsigned long long mx = comp < other ? other : comp;
                    comp = (lower == up) ? mn : mx;
                }
            }
            slot = __shfl_sync(0xFFFFFFFFu, slot, (uint32_t)(comp & 31));
            key = (uint32_t)(comp >> 5);
        }
        // ties on this word with 14 real symbols continue on the next word
        const uint32_t kp = __shfl_up_sync(0xFFFFFFFFu, key, 1);
        const uint32_t kn = __shfl_down_sync(0xFFFFFFFFu, key, 1);
        const bool g_active = active;  // whole groups are active or not
        const bool eqp = g_active && lane > group && kp == key;
        const bool eqn = g_active && lane + 1 < gend && kn == key;
        active = (eqp || eqn) && ((key & 15u) == B.ksyms);
        const uint32_t st2 = __ballot_sync(0xFFFFFFFFu, !active || !eqp);
        group = active ? 31u - __clz(st2 & (0xFFFFFFFFu >> (31 - lane))) : lane;
        if (!__any_sync(0xFFFFFFFFu, active)) break;
        ++word;
    }
    return slot;
}

// ---------------------------------------------------------------------------
// Key word 0 of every slot of the block (the first MSD pass's keys): 16
// consecutive slots per thread share 3 text words and 2 terminator words;
// 64-byte vector stores.  Same encoding as suffix_key (common.cuh).
// ---------------------------------------------------------------------------
// Key word 0 of the 16 slots p0 .. p0+15 (p0 a multiple of 16 inside the
// packed text): 3 text words and 2 terminator words for all 16.
__device__ __forceinline__ void keys16(const uint32_t* __restrict__ text,
                                       const uint32_t* __restrict__ term, uint64_t p0,
                                       uint32_t (&k)[16]) {
    const uint64_t w = p0 >> 4;
    const uint32_t off = (uint32_t)(p0 & 15);
    const uint32_t t0 = __ldg(text + w), t1 = __ldg(text + w + 1), t2 = __ldg(text + w + 2);
    const uint64_t v01 = ((uint64_t)t0 << 32) | t1, v12 = ((uint64_t)t1 << 32) | t2;
    const uint64_t tb = p0 >> 5;
    const uint32_t toff = (uint32_t)(p0 & 31);
    const uint64_t T = ((uint64_t)__ldg(term + tb) << 32) | __ldg(term + tb + 1);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t o = off + j;
        const uint64_t v = o < 16 ? (v01 << (2 * o)) : (v12 << (2 * (o - 16)));
        uint32_t syms = (uint32_t)(v >> 36);
        uint32_t ended = (uint32_t)__clzll((long long)(T << (toff + j)));
        ended = ended > (uint32_t)kKeySyms ? (uint32_t)kKeySyms : ended;
        const uint32_t keep = 2 * ended;
        const uint32_t mask = keep == 0 ? 0u : (0x0FFFFFFFu & ~((1u << (28 - keep)) - 1u));
        k[j] = ((syms & mask) << 4) | ended;
    }
}

__global__ void keygen_kernel(const uint32_t* __restrict__ text, const uint32_t* __restrict__ term,
                              uint64_t base, uint32_t n, uint32_t* __restrict__ key) {
    const uint32_t ng = (n + 15) >> 4;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
        uint32_t k[16];
        keys16(text, term, base + 16ull * g, k);
        const uint32_t i0 = 16 * g;
        if (i0 + 16 <= n) {
            uint4* dst = reinterpret_cast<uint4*>(key + i0);
            __stcs(dst + 0, make_uint4(k[0], k[1], k[2], k[3]));
            __stcs(dst + 1, make_uint4(k[4], k[5], k[6], k[7]));
            __stcs(dst + 2, make_uint4(k[8], k[9], k[10], k[11]));
            __stcs(dst + 3, make_uint4(k[12], k[13], k[14], k[15]));
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (i0 + j < n) key[i0 + j] = k[j];
        }
    }
}

// Key word 0 of every slot with 3-bit symbols (sigma = 5), one slot per thread.
__global__ void keygen5_kernel(const uint32_t* __restrict__ text, const uint32_t* __restrict__ term,
                               const uint32_t* __restrict__ nbit, uint64_t base, uint32_t n,
                               uint32_t* __restrict__ key) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        key[i] = suffix_key5(text, term, nbit, base + i, 0);
}

// ---------------------------------------------------------------------------
// init / control
// ---------------------------------------------------------------------------
__global__ void init_kernel(uint32_t* __restrict__ sa0, uint32_t* __restrict__ saf, uint32_t n,
                            Lists in, Lists out, uint32_t* misc, Bufs B) {
    // a LARGE first segment reads its slots as "iota" (meta bit) and never
    // needs them materialised; smaller blocks go straight to the segment sorts
    if (n <= kCapM) {
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
             i += (uint64_t)gridDim.x * blockDim.x)
            sa0[i] = sa_entry(B, (uint32_t)i);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int c = 0; c < NCLASS; ++c) {
            in.cnt[c] = 0;
            out.cnt[c] = 0;
        }
        for (int c = 0; c < M_N; ++c) misc[c] = 0;
        if (n == 1) saf[0] = sa_entry(B, 0u);
        // a LARGE first segment gets its keys from the first histogram pass
        else if (n > 1) emit(in, Seg{0u, n, 0u, make_meta(24, 0, n > kCapM ? 0u : 1u, n > kCapM ? 1u : 0u)});
    }
}

// Consumed lists: the counts of the classes processed this round (mask) are
// zeroed; an unprocessed class keeps its segments for a later round.
__global__ void reset_counts_kernel(uint32_t* cnt, uint32_t* misc, uint32_t mask) {
    if (threadIdx.x < NCLASS && ((mask >> threadIdx.x) & 1u)) cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        misc[M_CHUNKS] = 0;
        misc[M_GROUPS] = 0;
    }
}

// ---------------------------------------------------------------------------
// LARGE: one stable 8-bit MSD digit pass
// ---------------------------------------------------------------------------
// Split each large segment into chunks (one CTA of the digit pass each) and
// the chunks into prefix groups of kGroup.  Chunks are kMinChunk..kChunk long,
// as many as keep every SM busy when few large segments are left.
__global__ void chunkify_kernel(Lists in, SegX* __restrict__ segx, Chunk* __restrict__ chunks,
                                Group* __restrict__ groups, uint32_t* misc) {
    const uint32_t n = in.cnt[LARGE];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    const uint32_t want = (148u * 8u + n - 1) / n;  // chunks per segment to fill the GPU
    for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        const Seg s = in.seg[LARGE][i];
        const uint32_t lo = (s.len + kChunk - 1) / kChunk;
        const uint32_t hi = (s.len + kMinChunk - 1) / kMinChunk;
        uint32_t nch = max(lo, min(hi, want));
        nch = nch > kMaxChunks ? kMaxChunks : nch;
        uint32_t clen = (s.len + nch - 1) / nch;
        // whole scatter tiles per chunk: a ragged last tile costs a full
        // tile's ranking and barriers (1 element per tile at 2^24/1024)
        if (clen > (uint32_t)kDigTile) clen = (clen + kDigTile - 1) / kDigTile * kDigTile;
        nch = (s.len + clen - 1) / clen;
        const uint32_t ngr = (nch + kGroup - 1) / kGroup;
        uint32_t base = 0, gbase = 0;
        if (lane == 0) {
            base = atomicAdd(misc + M_CHUNKS, nch);
            gbase = atomicAdd(misc + M_GROUPS, ngr);
            atomicAdd(misc + M_ACTIVE, s.len);
            segx[i] = SegX{base, nch, gbase, 0u};
        }
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        gbase = __shfl_sync(0xFFFFFFFFu, gbase, 0);
        for (uint32_t c = lane; c < nch; c += 32) {
            const uint32_t b = s.start + c * clen;
            const uint32_t e = min(b + clen, s.start + s.len);
            chunks[base + c] = Chunk{i, b, e, gbase + c / kGroup};
        }
        for (uint32_t g = lane; g < ngr; g += 32)
            groups[gbase + g] = Group{base + g * kGroup, min(kGroup, nch - g * kGroup)};
    }
}

#ifndef SB_HIST_MINB
#define SB_HIST_MINB 4
#endif
__global__ void __launch_bounds__(kDigNt, SB_HIST_MINB) digit_hist_kernel(Lists in, const Chunk* __restrict__ chunks,
                                                            const uint32_t* misc, Bufs B,
                                                            uint32_t* __restrict__ hist) {
    constexpr int NW = kDigNt / 32;
    __shared__ uint32_t h[NW][256];
    const uint32_t nch = misc[M_CHUNKS];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
        for (uint32_t i = tid; i < NW * 256; i += kDigNt) (&h[0][0])[i] = 0;
        __syncthreads();
        const Chunk ch = chunks[c];
        const Seg s = in.seg[LARGE][ch.seg];
        const uint32_t shift = meta_shift(s.meta);
        const uint32_t buf = meta_buf(s.meta);
        const bool kv = meta_kv(s.meta);
        const uint32_t* S = B.sa[buf];
        uint32_t* K = B.key[buf];
        if (!kv && meta_iota(s.meta) && s.word == 0 && !B.nbit) {
            // the block's first pass: key word 0 generated here from the packed
            // text (16 consecutive slots per thread, keys16) and written for the
            // scatter -- no separate key-generation pass
            for (uint32_t g = (ch.begin >> 4) + tid; g <= (ch.end - 1) >> 4; g += kDigNt) {
                uint32_t k[16];
                keys16(B.text, B.term, B.base + 16ull * g, k);
                const uint32_t i0 = 16 * g;
                if (i0 >= ch.begin && i0 + 16 <= ch.end) {
                    uint4* dst = reinterpret_cast<uint4*>(K + i0);
                    dst[0] = make_uint4(k[0], k[1], k[2], k[3]);
                    dst[1] = make_uint4(k[4], k[5], k[6], k[7]);
                    dst[2] = make_uint4(k[8], k[9], k[10], k[11]);
                    dst[3] = make_uint4(k[12], k[13], k[14], k[15]);
#pragma unroll
                    for (int j = 0; j < 16; ++j) atomicAdd(&h[warp][(k[j] >> shift) & 0xFFu], 1u);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const uint32_t p = i0 + j;
                        if (p >= ch.begin && p < ch.end) {
                            K[p] = k[j];
                            atomicAdd(&h[warp][(k[j] >> shift) & 0xFFu], 1u);
                        }
                    }
                }
            }
        } else if (kv) {
            // keys valid: 4 consecutive keys per thread per 16-byte load
            const uint32_t a0 = ch.begin & ~3u;
            for (uint32_t p0 = a0; p0 < ch.end; p0 += kDigNt * 4 * 2) {
                uint4 q[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const uint32_t p = p0 + (u * kDigNt + tid) * 4;
                    q[u] = p < ch.end ? __ldcs(reinterpret_cast<const uint4*>(K + p))
                                      : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const uint32_t p = p0 + (u * kDigNt + tid) * 4;
                    const uint32_t kk[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const bool in = p + v >= ch.begin && p + v < ch.end;
                        const uint32_t d = (kk[v] >> shift) & 0xFFu;
                        const uint32_t d0 = __shfl_sync(0xFFFFFFFFu, d, 0);
                        if (__all_sync(0xFFFFFFFFu, in && d == d0)) {
                            if (lane == 0) atomicAdd(&h[warp][d0], 32u);
                        } else if (in) {
                            atomicAdd(&h[warp][d], 1u);
                        }
                    }
                }
            }
        } else {
            constexpr int U = 8;
            for (uint32_t p0 = ch.begin; p0 < ch.end; p0 += kDigNt * U) {
                uint32_t key[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t p = p0 + u * kDigNt + tid;
                    key[u] = 0;
                    if (p < ch.end) {
                        const uint32_t sl = meta_iota(s.meta) ? p : __ldg(S + p);
                        key[u] = key_of(B, sl, s.word);
                        K[p] = key[u];
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t p = p0 + u * kDigNt + tid;
                    if (p < ch.end) atomicAdd(&h[warp][(key[u] >> shift) & 0xFFu], 1u);
                }
            }
        }
        __syncthreads();
        if (tid < 256) {
            uint32_t t = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) t += h[w][tid];
            hist[(size_t)c * 256 + tid] = t;
        }
        __syncthreads();
    }
}

// Exclusive prefix of the chunk histograms inside each group of <= kGroup
// chunks (one CTA per group, one thread per digit); gtot = group totals.
__global__ void __launch_bounds__(256) group_scan_kernel(const Group* __restrict__ groups,
                                                         const uint32_t* misc,
                                                         uint32_t* __restrict__ hist,
                                                         uint32_t* __restrict__ gtot) {
    const uint32_t ng = misc[M_GROUPS];
    const uint32_t d = threadIdx.x;
    for (uint32_t g = blockIdx.x; g < ng; g += gridDim.x) {
        const Group gr = groups[g];
        uint32_t v[kGroup];
#pragma unroll
        for (uint32_t b = 0; b < kGroup; ++b)
            v[b] = b < gr.nchunks ? hist[(size_t)(gr.first_chunk + b) * 256 + d] : 0u;
        uint32_t run = 0;
#pragma unroll
        for (uint32_t b = 0; b < kGroup; ++b) {
            if (b < gr.nchunks) hist[(size_t)(gr.first_chunk + b) * 256 + d] = run;
            run += v[b];
        }
        gtot[(size_t)g * 256 + d] = run;
    }
}

// Per segment: prefix over its groups (gtot -> exclusive group offsets),
// digit bases, sieve decisions and child segments.
__global__ void __launch_bounds__(256) digit_scan_kernel(Lists in, Lists out,
                                                         SegX* __restrict__ segx,
                                                         uint32_t* __restrict__ gtot,
                                                         uint32_t* __restrict__ dbase,
                                                         uint32_t ksyms) {
    __shared__ uint32_t wsum[8];
    __shared__ uint32_t ccount[NCLASS], cbase[NCLASS];
    __shared__ int all_one;
    const uint32_t n = in.cnt[LARGE];
    const uint32_t d = threadIdx.x, lane = d & 31, warp = d >> 5;
    for (uint32_t si = blockIdx.x; si < n; si += gridDim.x) {
        const Seg s = in.seg[LARGE][si];
        const SegX x = segx[si];
        const uint32_t ngr = (x.nchunks + kGroup - 1) / kGroup;
        uint32_t total = 0;
        for (uint32_t g0 = 0; g0 < ngr; g0 += 8) {
            uint32_t v[8];
#pragma unroll
            for (int b = 0; b < 8; ++b)
                v[b] = g0 + b < ngr ? gtot[(size_t)(x.group_base + g0 + b) * 256 + d] : 0u;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                if (g0 + b < ngr) gtot[(size_t)(x.group_base + g0 + b) * 256 + d] = total;
                total += v[b];
            }
        }
        if (d < NCLASS) ccount[d] = 0;
        if (d == 0) all_one = 0;
        uint32_t incl = total;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (total == s.len) all_one = 1;
        uint32_t excl = incl - total;
        for (uint32_t w = 0; w < warp; ++w) excl += wsum[w];
        __syncthreads();
        const uint32_t shift = meta_shift(s.meta);
        const uint32_t buf = meta_buf(s.meta);
        const bool resolved = (total == 1) || (shift == 0 && (d & 15u) < ksyms);
        uint32_t flag = 0;
        int cls = -1;
        Seg c;
        uint32_t local = 0;
        if (total > 0) {
            if (resolved) {
                flag = 0x80000000u;
            } else {
                const uint32_t cbuf = all_one ? buf : 1u - buf;
                const uint32_t ciota = all_one ? meta_iota(s.meta) : 0u;  // data not moved
                c.start = s.start + excl;
                c.len = total;
                if (shift == 0) {
                    c.word = s.word + 1;
                    c.meta = make_meta(24, cbuf, 0, ciota);
                } else {
                    c.word = s.word;
                    c.meta = make_meta(shift - 8, cbuf, 1, ciota);
                }
                cls = class_of(c, out.local);
                local = atomicAdd(&ccount[cls], 1u);
                if (all_one) segx[si].skip = 1;
            }
        }
        dbase[(size_t)si * 256 + d] = (s.start + excl) | flag;
        __syncthreads();
        if (d < NCLASS && ccount[d]) cbase[d] = atomicAdd(out.cnt + d, ccount[d]);
        __syncthreads();
        if (cls >= 0) out.seg[cls][cbase[cls] + local] = c;
        __syncthreads();
    }
}

// 4-byte async copy global -> shared, L2 evict-first (the scatter reads each
// key / slot once; the rank dictionary and g should keep L2)
__device__ __forceinline__ void cp_async4(uint32_t* dst, const uint32_t* src, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// A scatter tile: tile-local source pointers of one chunk.
struct Tile {
    uint32_t c, t0, end;  // chunk, first element, chunk end
};

// IPT items per thread (tile = kDigNt * IPT)
template <int IPT>
__global__ void __launch_bounds__(kDigNt, 2) digit_scatter_kernel(
    Lists in, const SegX* __restrict__ segx, const Chunk* __restrict__ chunks, const uint32_t* misc,
    const uint32_t* __restrict__ hist, const uint32_t* __restrict__ gtot,
    const uint32_t* __restrict__ dbase, Bufs B) {
    constexpr int NW = kDigNt / 32;
    constexpr int TILE = kDigNt * IPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* wcnt = reinterpret_cast<uint32_t*>(smem_raw);  // NW*256
    uint2* s_kv = reinterpret_cast<uint2*>(wcnt + NW * 256);  // TILE (key, slot)
    uint32_t* s_ink = reinterpret_cast<uint32_t*>(s_kv + TILE);  // TILE: next tile's keys
    uint32_t* s_ins = s_ink + TILE;                              // TILE: next tile's slots
    uint32_t* dstart = s_ins + TILE;                             // 257
    uint32_t* run_base = dstart + 260;                        // 256
    uint32_t* off = run_base + 256;                           // 256: run_base - dstart
    uint32_t* tmp = off + 256;                                // 32
    uint8_t* fin = reinterpret_cast<uint8_t*>(tmp + 32);      // 256
    const uint32_t nch = misc[M_CHUNKS];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t pol_ef;
#if SB_SCATTER_L2
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_ef));
#else
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_ef));
#endif

    // Tiles of this CTA's chunks in order; the next tile's keys (and slots)
    // are prefetched into shared memory with cp.async while the current one
    // is ranked.  Each thread copies exactly the elements it later reads, so
    // the prefetch needs no barrier.
    auto first_tile = [&](uint32_t c) -> Tile {
        for (; c < nch; c += gridDim.x) {
            const Chunk ch = chunks[c];
            if (!segx[ch.seg].skip) return Tile{c, ch.begin, ch.end};
        }
        return Tile{nch, 0u, 0u};
    };
    auto next_tile = [&](const Tile& t) -> Tile {
        if (t.t0 + TILE < t.end) return Tile{t.c, t.t0 + TILE, t.end};
        return first_tile(t.c + gridDim.x);
    };
    auto prefetch = [&](const Tile& t) {
        if (t.c >= nch) return;
        const Seg s = in.seg[LARGE][chunks[t.c].seg];
        const uint32_t buf = meta_buf(s.meta);
        const uint32_t tn = min((uint32_t)TILE, t.end - t.t0);
        const uint32_t* K = B.key[buf] + t.t0;
        const uint32_t* S = B.sa[buf] + t.t0;
        const bool iota = meta_iota(s.meta);
#pragma unroll
        for (int it = 0; it < IPT; ++it) {
            const uint32_t e = warp * (32 * IPT) + it * 32 + lane;
            if (e < tn) {
                cp_async4(s_ink + e, K + e, pol_ef);
                if (!iota) cp_async4(s_ins + e, S + e, pol_ef);
            }
        }
        cp_async_commit();
    };

    Tile cur = first_tile(blockIdx.x);
    prefetch(cur);
    uint32_t chunk_of_setup = ~0u;
    uint32_t shift = 0, buf = 0, word_of_setup = 0;
    bool iota = false;
    while (cur.c < nch) {
        if (cur.c != chunk_of_setup) {
            // new chunk: the previous chunk's write-out must be done with fin/run_base
            __syncthreads();
            const Chunk ch = chunks[cur.c];
            const Seg s = in.seg[LARGE][ch.seg];
            shift = meta_shift(s.meta);
            buf = meta_buf(s.meta);
            iota = meta_iota(s.meta);
            word_of_setup = s.word;
            if (tid < 256) {
                const uint32_t db = dbase[(size_t)ch.seg * 256 + tid];
                run_base[tid] = (db & 0x7FFFFFFFu) + gtot[(size_t)ch.group * 256 + tid] +
                                hist[(size_t)cur.c * 256 + tid];
                fin[tid] = (uint8_t)(db >> 31);
            }
            chunk_of_setup = cur.c;
        }
        uint32_t* S2 = B.sa[1 - buf];
        uint32_t* K2 = B.key[1 - buf];
        const uint32_t t0 = cur.t0;
        const uint32_t tn = min((uint32_t)TILE, cur.end - t0);
        uint32_t key[IPT], slot[IPT], dig[IPT], dest[IPT];
        cp_async_wait_all();
#pragma unroll
        for (int it = 0; it < IPT; ++it) {
            const uint32_t e = warp * (32 * IPT) + it * 32 + lane;
            const bool valid = e < tn;
            key[it] = valid ? s_ink[e] : 0u;
            slot[it] = valid ? (iota ? t0 + e : s_ins[e]) : 0u;
            dig[it] = valid ? ((key[it] >> shift) & 0xFFu) : 0x100u;
        }
        if (iota && B.smask != 0xFFFFFFFFu) {
            // generated slots get their B_int payload.  On key word 0 the
            // symbol before slot s is the top symbol of slot s-1's key and a
            // clamp of 0 marks s-1 as a terminator: the previous element's key
            // comes from the neighbouring lane (or the warp's previous tile
            // element), no text lookups.
            if (word_of_setup == 0) {
                const uint32_t e0 = warp * (32 * IPT);
                uint32_t carry = 0;
                if (lane == 0 && e0 < tn && t0 + e0 > 0) carry = B.key[buf][t0 + e0 - 1];
#pragma unroll
                for (int it = 0; it < IPT; ++it) {
                    const uint32_t up = __shfl_up_sync(0xFFFFFFFFu, key[it], 1);
                    const uint32_t last = __shfl_sync(0xFFFFFFFFu, key[it], 31);
                    const uint32_t pk = lane == 0 ? carry : up;
                    carry = last;
                    const uint32_t sl = slot[it];
                    uint32_t b;
                    if (sl == 0 || (pk & 15u) == 0) b = 4u;
                    else if (B.nbit) b = ((pk >> 28) & 7u) == 4u ? 5u : ((pk >> 28) & 7u);
                    else b = pk >> 30;
                    slot[it] = sl | (b << kPayloadShift);
                }
            } else {
#pragma unroll
                for (int it = 0; it < IPT; ++it) slot[it] = sa_entry(B, slot[it]);
            }
        }
        cur = next_tile(cur);
        prefetch(cur);
        block_rank<kDigNt, IPT>(dig, dest, wcnt, dstart, tmp);
        if (tid < 256) {
            off[tid] = run_base[tid] - dstart[tid];  // mod 2^32
            run_base[tid] += dstart[tid + 1] - dstart[tid];
        }
#pragma unroll
        for (int it = 0; it < IPT; ++it)
            if (dig[it] < 256) {
                s_kv[dest[it]] = make_uint2(key[it], slot[it]);
            }
        __syncthreads();
        // coalesced write-out: consecutive tile positions of one digit go to
        // consecutive global positions.  The next tile's block_rank barriers
        // order this loop's shared reads before their overwrite.
        for (uint32_t i = tid; i < tn; i += kDigNt) {
            const uint2 kv = s_kv[i];
            const uint32_t d = (kv.x >> shift) & 0xFFu;
            const uint32_t gp = off[d] + i;
            if (fin[d]) {
                SB_ASSERT(gp < B.n);
                __stcs(B.saf + gp, kv.y);
            } else {
#if SB_SCATTER_L2
                S2[gp] = kv.y;
                K2[gp] = kv.x;
#else
                __stcs(S2 + gp, kv.y);
                __stcs(K2 + gp, kv.x);
#endif
            }
        }
    }
}

template <int IPT>
constexpr size_t scatter_smem() {
    return (size_t)(kDigNt / 32) * 256 * 4 + 4 * (size_t)(kDigNt * IPT) * 4 + 260 * 4 +
           2 * 256 * 4 + 32 * 4 + 256 + 16;
}

// ---------------------------------------------------------------------------
// TINY: one warp per segment
// ---------------------------------------------------------------------------
constexpr uint32_t kTinyPerWarp = 32;  // list entries per warp, packed into shared calls

// Fast path for packed tiny segments whose unknown key bits fit in 16 (keys
// valid, shift <= 8): one u32 bitonic over the warp on (group, key bits, lane).
// Returns the lane's slot in sorted order; `tie` marks lanes that still tie on
// this word with 14 real symbols and `run` the first lane of their tie run.
__device__ __forceinline__ uint32_t warp_sort16(uint32_t slot, uint32_t L, uint32_t grp,
                                                uint32_t key, uint32_t rb, bool& tie,
                                                uint32_t& run, uint32_t ksyms) {
    const uint32_t lane = threadIdx.x & 31;
    const bool valid = lane < L;
    const uint32_t rmask = (1u << rb) - 1u;
    uint32_t v = valid ? (grp << 26) | ((key & rmask) << 5) | lane : 0xFFFFFFFFu;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
        {
            const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, v, k - 1);
            const bool lower = (lane & (uint32_t)(k >> 1)) == 0;
            v = lower ? min(v, o) : max(v, o);
        }
#pragma unroll
        for (int j = k >> 2; j > 0; j >>= 1) {
            const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, v, j);
            const bool lower = (lane & (uint32_t)j) == 0;
            v = lower ? min(v, o) : max(v, o);
        }
    }
    const uint32_t src = v & 31u;
    const uint32_t s2 = __shfl_sync(0xFFFFFFFFu, slot, src);
    const uint32_t k2 = __shfl_sync(0xFFFFFFFFu, key, src);
    const uint32_t hi = v >> 5;
    const uint32_t prv = __shfl_up_sync(0xFFFFFFFFu, hi, 1);
    const uint32_t nxt = __shfl_down_sync(0xFFFFFFFFu, hi, 1);
    const bool eqp = valid && lane > 0 && prv == hi;
    const bool eqn = valid && lane + 1 < L && nxt == hi;
    tie = (eqp || eqn) && ((k2 & 15u) == ksyms);
    const uint32_t starts = __ballot_sync(0xFFFFFFFFu, tie && !eqp);
    run = 31u - __clz(starts & (0xFFFFFFFFu >> (31 - lane)));
    return s2;
}

#ifndef SB_TINY_MINB
#define SB_TINY_MINB 5  // 48 registers: 5 CTAs per SM (c3 step -4.6 %, measured)
#endif
__global__ void __launch_bounds__(256, SB_TINY_MINB) tiny_kernel(Lists in, Bufs B, uint32_t* misc) {
    const uint32_t n = in.cnt[TINY];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    for (uint32_t i0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kTinyPerWarp; i0 < n;
         i0 += nw * kTinyPerWarp) {
        const uint32_t i1 = min(n, i0 + kTinyPerWarp);
        // pack consecutive segments into the 32 lanes; each lane remembers its
        // segment's output position, start word and key (a segment keeps its
        // lanes through the sort: the composite sorts by group first)
        uint32_t lb = 0, dst = 0, word = 0, key = 0, slot = 0, grp = 0, elems = 0, rb = 0;
        uint32_t bf = 0;
        bool mine = false, kv = false, fast = true;
        // all of the warp's list entries in one coalesced load (lane l holds
        // entry i0+l); the packing loop below broadcasts them with shuffles, so
        // it never waits on memory
        Seg mys = Seg{0u, 0u, 0u, 0u};
        if (lane < i1 - i0) mys = in.seg[TINY][i0 + lane];
        for (uint32_t i = i0; i <= i1; ++i) {
            Seg sg;
            if (i < i1) {
                const uint32_t src = i - i0;
                sg.start = __shfl_sync(0xFFFFFFFFu, mys.start, src);
                sg.len = __shfl_sync(0xFFFFFFFFu, mys.len, src);
                sg.word = __shfl_sync(0xFFFFFFFFu, mys.word, src);
                sg.meta = __shfl_sync(0xFFFFFFFFu, mys.meta, src);
            }
            if (i == i1 || lb + sg.len > 32) {
                if (lb) {
                    // the packed group's members, all loads in flight at once
                    // (per-segment loads serialised their latencies)
                    if (mine) {
                        slot = B.sa[bf][dst];
                        key = kv ? B.key[bf][dst] : 0u;
                    }
                    uint32_t r;
                    if (__all_sync(0xFFFFFFFFu, fast || lane >= lb)) {
                        bool tie;
                        uint32_t run;
                        r = warp_sort16(slot, lb, grp, key, rb, tie, run, B.ksyms);
                        // ties continue on word+1 (key words from the text)
                        if (__any_sync(0xFFFFFFFFu, tie))
                            r = warp_finish(r, lb, word + 1, 0u, false, B, run, tie);
                    } else {
                        r = warp_finish(slot, lb, word, key, kv, B, grp);
                    }
                    SB_ASSERT(!mine || dst < B.n);
                    if (mine) B.saf[dst] = r;
                }
                lb = 0;
                mine = false;
                fast = true;
                if (i == i1) break;
            }
            if (lane >= lb && lane < lb + sg.len) {
                const uint32_t e = lane - lb;
                bf = meta_buf(sg.meta);
                mine = true;
                dst = sg.start + e;
                word = sg.word;
                kv = meta_kv(sg.meta);
                grp = lb;
                rb = meta_shift(sg.meta) + 8;
                fast = kv && meta_shift(sg.meta) <= 8;
            }
            lb += sg.len;
            elems += sg.len;
        }
        if (lane == 0) atomicAdd(misc + M_ELEMS_T, elems);
    }
}

// ---------------------------------------------------------------------------
// LOCALD: the digit pass of one segment of 513..4096 members with valid keys,
// entirely in one CTA -- the segment is one tile, so the tile's stable ranks
// ARE the segment's digit histogram and offsets: no chunk / histogram / scan
// kernels, one read and one write of (key, slot).  Same outputs as the
// LARGE path: resolved buckets (one member, or equal keys that end inside
// the word) go to their final SA positions; buckets of 2..32 members are
// finished right here by the warps, as the TINY class would (a register sort
// of their remaining key bits, ties continued on the next words); the
// others become child segments, keyed on the next digit (or the next word
// at shift 0).
// ---------------------------------------------------------------------------
#ifndef SB_LD_MINB
#define SB_LD_MINB 4  // resident CTAs per SM of local_digit_kernel<256>
#endif
constexpr int kLocIpt = 8;

template <int NT>
constexpr size_t local_digit_smem() {
    return (size_t)(NT / 32) * 256 * 4 + 2 * (size_t)(NT * kLocIpt) * 8 + 260 * 4 + 32 * 4 + 256 +
           64;
}

// NT = 512: LOCALD (tile 4096); NT = 256: LOCALD2 (tile 2048)
template <int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? SB_LD_MINB : 1024 / NT) local_digit_kernel(Lists in, Lists out, Bufs B,
                                                                   uint32_t* misc) {
    constexpr int kLocNt = NT;
    constexpr uint32_t kTileL = NT * kLocIpt;
    constexpr int NWL = NT / 32;
    constexpr int DPW = 256 / NWL;  // digits per warp in the small-bucket finish (16 or 32)
    constexpr int CLS = NT == 512 ? LOCALD : LOCALD2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* wcnt = reinterpret_cast<uint32_t*>(smem_raw);                   // NW*256
    uint2* s_kv = reinterpret_cast<uint2*>(wcnt + (kLocNt / 32) * 256);       // tile: sorted
    uint2* s_in = s_kv + kTileL;                                              // tile: as loaded
    uint32_t* dstart = reinterpret_cast<uint32_t*>(s_in + kTileL);            // 257
    uint32_t* tmp = dstart + 260;                                             // 32
    uint8_t* fin = reinterpret_cast<uint8_t*>(tmp + 32);                      // 256
    __shared__ uint32_t ccount[NCLASS], cbase[NCLASS];
    const uint32_t n = in.cnt[CLS];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t nlook = 0;  // this thread's key-word lookups (algorithmic-byte count)
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    // the next segment's (key, slot) are fetched into s_in with cp.async
    // while this one is finished (each thread copies exactly the elements it
    // reads back: no barrier needed for the copies themselves)
    auto prefetch = [&](uint32_t si2) {
        if (si2 >= n) return;
        const Seg s2 = in.seg[CLS][si2];
        const uint32_t b2 = meta_buf(s2.meta);
        const bool io2 = meta_iota(s2.meta);
#pragma unroll
        for (int it = 0; it < kLocIpt; ++it) {
            const uint32_t e = warp * (32 * kLocIpt) + it * 32 + lane;
            if (e < s2.len) {
                cp_async4(&s_in[e].x, B.key[b2] + s2.start + e, pol);
                if (io2) s_in[e].y = sa_entry(B, s2.start + e);
                else cp_async4(&s_in[e].y, B.sa[b2] + s2.start + e, pol);
            }
        }
        cp_async_commit();
    };
    prefetch(blockIdx.x);
    for (uint32_t si = blockIdx.x; si < n; si += gridDim.x) {
        const Seg s = in.seg[CLS][si];
        const uint32_t shift = meta_shift(s.meta), buf = meta_buf(s.meta);
        // (key, slot) wait in shared memory while the digits are ranked
        // (registers hold only digits and ranks: no spills at 2 CTAs/SM)
        uint32_t dig[kLocIpt], dest[kLocIpt];
        cp_async_wait_all();
#pragma unroll
        for (int it = 0; it < kLocIpt; ++it) {
            const uint32_t e = warp * (32 * kLocIpt) + it * 32 + lane;
            const bool valid = e < s.len;
            const uint32_t key = valid ? s_in[e].x : 0u;
            dig[it] = valid ? ((key >> shift) & 0xFFu) : 0x100u;
        }
        if (tid < NCLASS) ccount[tid] = 0;
        block_rank<kLocNt, kLocIpt>(dig, dest, wcnt, dstart, tmp);
        // per digit: sieve decision and child segment (digit_scan's rules)
        int cls = -1;
        uint32_t local = 0;
        Seg c;
        if (tid < 256) {
            const uint32_t d = tid;
            const uint32_t total = dstart[d + 1] - dstart[d];
            const bool resolved = (total == 1) || (shift == 0 && (d & 15u) < B.ksyms);
            // 2..32 members, remaining key bits <= 16 (or the next word):
            // finished in this CTA below (fin = 2)
            const bool here = !resolved && total >= 2 && total <= 32 && shift <= 16;
            fin[d] = resolved ? 1 : here ? 2 : 0;
            if (total > 0 && !resolved && !here) {
                c.start = s.start + dstart[d];
                c.len = total;
                if (shift == 0) {
                    c.word = s.word + 1;
                    c.meta = make_meta(24, 1u - buf, 0);
                } else {
                    c.word = s.word;
                    c.meta = make_meta(shift - 8, 1u - buf, 1);
                }
                cls = class_of(c, out.local);
                local = atomicAdd(&ccount[cls], 1u);
            }
        }
#pragma unroll
        for (int it = 0; it < kLocIpt; ++it)
            if (dig[it] < 256) s_kv[dest[it]] = s_in[warp * (32 * kLocIpt) + it * 32 + lane];
        __syncthreads();
        prefetch(si + gridDim.x);  // s_in is free again
        if (tid < NCLASS && ccount[tid]) cbase[tid] = atomicAdd(out.cnt + tid, ccount[tid]);
        if (tid == 0) {
            atomicAdd(misc + M_ACTIVE, s.len);
            atomicAdd(misc + M_ACTIVE_LOC, s.len);
        }
        __syncthreads();
        if (cls >= 0) out.seg[cls][cbase[cls] + local] = c;
        // the small buckets: warp w takes digits [DPW*w, DPW*w + DPW) in
        // order and packs consecutive buckets into its 32 lanes (tiny_kernel's
        // scheme); lane q holds digit q's size and start, broadcast by shuffles
        {
            uint32_t my_tot = 0, my_start = 0;
            if (lane < (uint32_t)DPW) {
                const uint32_t d = warp * DPW + lane;
                my_start = dstart[d];
                my_tot = fin[d] == 2 ? dstart[d + 1] - my_start : 0u;
            }
            uint32_t todo = __ballot_sync(0xFFFFFFFFu, my_tot != 0);
            uint32_t lb = 0, dstp = 0, slot = 0, key = 0, grp = 0;
            bool mine = false;
            while (true) {
                const uint32_t q = todo ? (uint32_t)(__ffs(todo) - 1) : 32u;
                const uint32_t tot = q < 32 ? __shfl_sync(0xFFFFFFFFu, my_tot, q) : 0u;
                if (q == 32 || lb + tot > 32) {
                    if (lb) {
                        uint32_t r;
                        if (shift > 0) {
                            // the child's unknown key bits: [0, shift)
                            bool tie;
                            uint32_t run;
                            r = warp_sort16(slot, lb, grp, key, shift, tie, run, B.ksyms);
                            if (__any_sync(0xFFFFFFFFu, tie))
                                r = warp_finish(r, lb, s.word + 1, 0u, false, B, run, tie,
                                                &nlook);
                        } else {
                            r = warp_finish(slot, lb, s.word + 1, 0u, false, B, grp, true,
                                            &nlook);
                        }
                        SB_ASSERT(!mine || s.start + dstp < B.n);
                        if (mine) B.saf[s.start + dstp] = r;
                    }
                    lb = 0;
                    mine = false;
                    if (q == 32) break;
                }
                const uint32_t st0 = __shfl_sync(0xFFFFFFFFu, my_start, q);
                if (lane >= lb && lane < lb + tot) {
                    dstp = st0 + (lane - lb);
                    const uint2 kv = s_kv[dstp];
                    key = kv.x;
                    slot = kv.y;
                    grp = lb;
                    mine = true;
                }
                lb += tot;
                todo &= todo - 1;
            }
        }
        // write-out in segment order: finished buckets to the final SA, the
        // child segments' (key, slot) into the other buffer
        uint32_t* S2 = B.sa[1 - buf] + s.start;
        uint32_t* K2 = B.key[1 - buf] + s.start;
        for (uint32_t i = tid; i < s.len; i += kLocNt) {
            const uint2 kv = s_kv[i];
            const uint8_t f = fin[(kv.x >> shift) & 0xFFu];
            if (f == 1) {
                SB_ASSERT(s.start + i < B.n);
                __stcs(B.saf + s.start + i, kv.y);
            } else if (f == 0) {
                S2[i] = kv.y;
                K2[i] = kv.x;
            }
        }
        __syncthreads();
    }
    // one atomic per warp for the lookup count
    uint32_t w = nlook;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xFFFFFFFFu, w, o);
    if (lane == 0 && w) atomicAdd(misc + M_LOOKUPS, w);
}


// ---------------------------------------------------------------------------
// Common tail of the warp sorts: buf[0..L) holds the segment's (key word,
// slot) pairs in sorted order.  Write the final SA entries, then finish ties
// on this word with 14 real symbols: runs <= 32 are packed into shared
// warp_finish calls, longer runs become segments of the next word.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void warp_tail(const uint2* buf, const Seg& s, const Lists& out,
                                          const Bufs& B) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t L = s.len;
    const uint32_t nit = (L + 31) >> 5;
    const uint32_t bid = meta_buf(s.meta);
    for (uint32_t e = lane; e < L; e += 32) __stcs(B.saf + s.start + e, buf[e].y);
        uint32_t lb = 0, my_pos = 0, my_grp = 0;
        bool mine = false;
        for (uint32_t it = 0; it < nit; ++it) {
            const uint32_t e = it * 32 + lane;
            const uint32_t k = buf[e].x;
            const bool st = e < L && (e == 0 || buf[e - 1].x != k) && e + 1 < L &&
                            buf[e + 1].x == k && (k & 15u) == B.ksyms;
            uint32_t m = __ballot_sync(0xFFFFFFFFu, st);
            while (m) {
                const uint32_t l = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t rs = it * 32 + l;
                const uint32_t rk = buf[rs].x;
                uint32_t Lr = 0;
                for (uint32_t c = rs + 1;; c += 32) {
                    const uint32_t q = c + lane;
                    const bool eq = q < L && buf[q].x == rk;
                    const uint32_t ne = __ballot_sync(0xFFFFFFFFu, !eq);
                    if (ne) {
                        Lr = c + (__ffs(ne) - 1) - rs;
                        break;
                    }
                }
                if (Lr <= kTiny) {
                    if (lb + Lr > 32) {
                        uint32_t sl = mine ? buf[my_pos].y : 0u;
                        sl = warp_finish(sl, lb, s.word + 1, 0u, false, B, my_grp);
                        if (mine) B.saf[s.start + my_pos] = sl;
                        lb = 0;
                        mine = false;
                    }
                    if (lane >= lb && lane < lb + Lr) {
                        mine = true;
                        my_pos = rs + lane - lb;
                        my_grp = lb;
                    }
                    lb += Lr;
                } else {
                    for (uint32_t q = lane; q < Lr; q += 32) B.sa[bid][s.start + rs + q] = buf[rs + q].y;
                    if (lane == 0) emit(out, Seg{s.start + rs, Lr, s.word + 1, make_meta(24, bid, 0, 0)});
                }
            }
        }
        if (lb) {
            uint32_t sl = mine ? buf[my_pos].y : 0u;
            sl = warp_finish(sl, lb, s.word + 1, 0u, false, B, my_grp);
            if (mine) B.saf[s.start + my_pos] = sl;
        }
}

// ---------------------------------------------------------------------------
// BIT2..BIT16: one warp per segment, register bitonic network
// ---------------------------------------------------------------------------
// Ascending bitonic sort of N = 32*NIT values, lane-major (element e = lane*NIT
// + r lives in register v[r] of lane e/NIT).  Each merge stage starts with the
// "mirror" comparator e <-> e^(k-1), so every comparator sorts ascending and no
// direction selects are needed; strides below NIT stay in registers, larger
// ones are one shuffle per value.
template <int NIT>
__device__ __forceinline__ void warp_bitonic(uint32_t (&v)[NIT]) {
    constexpr int N = 32 * NIT;
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
        if (k <= NIT) {
#pragma unroll
            for (int r = 0; r < NIT; ++r) {
                const int q = r ^ (k - 1);
                if (r < q) {
                    const uint32_t a = v[r], b = v[q];
                    v[r] = min(a, b);
                    v[q] = max(a, b);
                }
            }
        } else {
            const int lm = k / NIT - 1;
            const bool lower = (lane & (uint32_t)(k / NIT / 2)) == 0;
            uint32_t o[NIT];
#pragma unroll
            for (int r = 0; r < NIT; ++r) o[r] = __shfl_xor_sync(0xFFFFFFFFu, v[NIT - 1 - r], lm);
#pragma unroll
            for (int r = 0; r < NIT; ++r) v[r] = lower ? min(v[r], o[r]) : max(v[r], o[r]);
        }
#pragma unroll
        for (int j = k >> 2; j > 0; j >>= 1) {
            if (j < NIT) {
#pragma unroll
                for (int r = 0; r < NIT; ++r) {
                    if ((r & j) == 0) {
                        const uint32_t a = v[r], b = v[r | j];
                        v[r] = min(a, b);
                        v[r | j] = max(a, b);
                    }
                }
            } else {
                const int lj = j / NIT;
                const bool lower = (lane & (uint32_t)lj) == 0;
#pragma unroll
                for (int r = 0; r < NIT; ++r) {
                    const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, v[r], lj);
                    v[r] = lower ? min(v[r], o) : max(v[r], o);
                }
            }
        }
    }
}

template <int NIT>
#ifndef SB_BIT_MINB
#define SB_BIT_MINB 5  // 48 registers: 5 CTAs per SM (c2 step -2.8 %, measured)
#endif
__global__ void __launch_bounds__(kWarpCta * 32, SB_BIT_MINB) bitonic_kernel(Lists in, Lists out, int cls,
                                                               Bufs B, uint32_t* misc) {
    constexpr int N = 32 * NIT;
    constexpr int IDXB = NIT == 2 ? 6 : NIT == 4 ? 7 : NIT == 8 ? 8 : 9;
    static_assert((1 << IDXB) == N, "index field");
    __shared__ uint2 s_buf[kWarpCta][N];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint2* buf = s_buf[wib];
    const uint32_t n = in.cnt[cls];
    const uint32_t nw = gridDim.x * kWarpCta;
    for (uint32_t si = blockIdx.x * kWarpCta + wib; si < n; si += nw) {
        const Seg s = in.seg[cls][si];
        const uint32_t L = s.len;
        const uint32_t bid = meta_buf(s.meta);
        const uint32_t rb = meta_shift(s.meta) + 8;  // unknown low key bits (<= 16)
        const uint32_t rmask = (1u << rb) - 1u;
        const uint32_t* S = B.sa[bid];
        const uint32_t* K = B.key[bid];
        if (lane == 0) atomicAdd(misc + M_ELEMS_B, L);
        const uint32_t top = __ldg(K + s.start) & ~rmask;
        uint32_t v[NIT];
#pragma unroll
        for (int r = 0; r < NIT; ++r) {
            const uint32_t e = lane * NIT + r;
            v[r] = e < L ? (((__ldcs(K + s.start + e) & rmask) << IDXB) | e) : 0xFFFFFFFFu;
        }
        warp_bitonic<NIT>(v);
        // sorted order is lane-major (element e = lane*NIT + r); ties on this
        // word (equal keys with 14 real symbols) are found in registers
        uint32_t* sl32 = reinterpret_cast<uint32_t*>(buf);  // N slots in sorted order
        uint32_t* tl = sl32 + N;                            // compacted tie list
        uint32_t k16[NIT];
#pragma unroll
        for (int r = 0; r < NIT; ++r) {
            const uint32_t e = lane * NIT + r;
            k16[r] = v[r] >> IDXB;
            if (e < L) sl32[e] = __ldcs(S + s.start + (v[r] & (N - 1)));
        }
        const uint32_t nxt0 = __shfl_down_sync(0xFFFFFFFFu, k16[0], 1);
        uint32_t eqn = 0;  // bit r: element e ties with e+1
#pragma unroll
        for (int r = 0; r < NIT; ++r) {
            const uint32_t e = lane * NIT + r;
            const uint32_t nk = r + 1 < NIT ? k16[r + 1] : nxt0;
            if (e + 1 < L && nk == k16[r] && (k16[r] & 15u) == B.ksyms) eqn |= 1u << r;
        }
        const uint32_t lastn = __shfl_up_sync(0xFFFFFFFFu, eqn >> (NIT - 1), 1) & (lane > 0 ? 1u : 0u);
        const uint32_t eqp = ((eqn << 1) | lastn) & ((1u << NIT) - 1u);  // bit r: ties with e-1
        const uint32_t tb = eqn | eqp;
        __syncwarp();
        for (uint32_t e = lane; e < L; e += 32) __stcs(B.saf + s.start + e, sl32[e]);
        if (__any_sync(0xFFFFFFFFu, tb != 0)) {
            // compact the tied elements (sorted order kept; bit 31 = run start)
            const uint32_t c = __popc(tb);
            uint32_t x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            const uint32_t T = __shfl_sync(0xFFFFFFFFu, x, 31);
            uint32_t w = x - c;
#pragma unroll
            for (int r = 0; r < NIT; ++r)
                if ((tb >> r) & 1u)
                    tl[w++] = (lane * NIT + r) | ((v[r] & (N - 1)) << 16) |
                              (((eqp >> r) & 1u) ? 0u : 0x80000000u);
            __syncwarp();
            // batches of whole runs through warp_finish on the next word
            for (uint32_t b = 0; b < T;) {
                const uint32_t j = b + lane;
                const uint32_t te = j < T ? tl[j] : 0u;
                const uint32_t starts = __ballot_sync(0xFFFFFFFFu, j < T && (te >> 31));
                const bool full_fit = b + 32 >= T || (tl[b + 32] >> 31);
                uint32_t nb = full_fit ? min(32u, T - b) : (starts & ~1u) ? 31u - __clz(starts & ~1u) : 0u;
                if (nb == 0) {
                    // one run longer than 32: a segment of the next round
                    uint32_t Lr = 32;
                    for (;;) {
                        const uint32_t q = b + Lr + lane;
                        const bool st = q >= T || (tl[q] >> 31);
                        const uint32_t bl = __ballot_sync(0xFFFFFFFFu, st);
                        if (bl) {
                            Lr += __ffs(bl) - 1;
                            break;
                        }
                        Lr += 32;
                    }
                    const uint32_t rs = tl[b] & 0xFFFFu;
                    for (uint32_t q = lane; q < Lr; q += 32) B.sa[bid][s.start + rs + q] = sl32[rs + q];
                    if (lane == 0) emit(out, Seg{s.start + rs, Lr, s.word + 1, make_meta(24, bid, 0, 0)});
                    b += Lr;
                    continue;
                }
                const uint32_t e = te & 0xFFFFu;
                const uint32_t grp = 31u - __clz(starts & (0xFFFFFFFFu >> (31 - lane)));
                uint32_t sl = lane < nb ? sl32[e] : 0u;
                sl = warp_finish(sl, nb, s.word + 1, 0u, false, B, grp);
                __syncwarp();
                SB_ASSERT(lane >= nb || (e < L && s.start + e < B.n));
                if (lane < nb) B.saf[s.start + e] = sl;
                b += nb;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// SMALL: one warp per segment, LSD radix sort in registers
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWarpCta * 32) warp_sort_kernel(Lists in, Lists out, Bufs B,
                                                                 uint32_t* misc) {
    __shared__ uint32_t s_cnt[kWarpCta][256];
    __shared__ uint2 s_buf[kWarpCta][kCapS];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint32_t* cnt = s_cnt[wib];
    uint2* buf = s_buf[wib];
    const uint32_t n = in.cnt[SMALL];
    const uint32_t nw = gridDim.x * kWarpCta;
    for (uint32_t si = blockIdx.x * kWarpCta + wib; si < n; si += nw) {
        const Seg s = in.seg[SMALL][si];
        const uint32_t L = s.len;
        const uint32_t nit = (L + 31) >> 5;
        const uint32_t bid = meta_buf(s.meta);
        const bool kv = meta_kv(s.meta);
        const uint32_t* S = B.sa[bid];
        if (lane == 0) atomicAdd(misc + M_ELEMS_S, L);
        uint32_t key[kIpl], slot[kIpl], rank[kIpl];
#pragma unroll
        for (int it = 0; it < kIpl; ++it) {
            key[it] = 0xFFFFFFFFu;  // padding sorts last (stably after every real key)
            slot[it] = 0;
            const uint32_t e = it * 32 + lane;
            if ((uint32_t)it < nit && e < L) {
                slot[it] = S[s.start + e];
                key[it] = kv ? B.key[bid][s.start + e] : key_of(B, slot[it], s.word);
            }
        }
        const uint32_t top = kv ? meta_shift(s.meta) : 24u;
        for (uint32_t sh = 0; sh <= top; sh += 8) {
            const uint32_t d0 = (__shfl_sync(0xFFFFFFFFu, key[0], 0) >> sh) & 0xFFu;
            bool same = true;
#pragma unroll
            for (int it = 0; it < kIpl; ++it)
                if ((uint32_t)it < nit && it * 32 + lane < L) same &= ((key[it] >> sh) & 0xFFu) == d0;
            if (__all_sync(0xFFFFFFFFu, same)) continue;
#pragma unroll
            for (int j = 0; j < 8; ++j) cnt[lane * 8 + j] = 0;
            __syncwarp();
#pragma unroll
            for (int it = 0; it < kIpl; ++it) {
                if ((uint32_t)it < nit) {
                    const uint32_t d = (key[it] >> sh) & 0xFFu;
                    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
                    const uint32_t leader = __ffs(peers) - 1;
                    uint32_t b = 0;
                    if (lane == leader) {
                        b = cnt[d];
                        cnt[d] = b + __popc(peers);
                    }
                    b = __shfl_sync(0xFFFFFFFFu, b, leader);
                    rank[it] = b + __popc(peers & lanemask_lt());
                    __syncwarp();
                }
            }
            {
                uint32_t v[8], sum = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    v[j] = cnt[lane * 8 + j];
                    sum += v[j];
                }
                uint32_t incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= (uint32_t)o) incl += y;
                }
                uint32_t run = incl - sum;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    cnt[lane * 8 + j] = run;
                    run += v[j];
                }
            }
            __syncwarp();
#pragma unroll
            for (int it = 0; it < kIpl; ++it) {
                if ((uint32_t)it < nit) {
                    const uint32_t d = (key[it] >> sh) & 0xFFu;
                    buf[cnt[d] + rank[it]] = make_uint2(key[it], slot[it]);
                }
            }
            __syncwarp();
#pragma unroll
            for (int it = 0; it < kIpl; ++it) {
                if ((uint32_t)it < nit) {
                    const uint2 v = buf[it * 32 + lane];
                    key[it] = v.x;
                    slot[it] = v.y;
                }
            }
            __syncwarp();
        }
        // final order out; stash (key, slot) for the tie scan
#pragma unroll
        for (int it = 0; it < kIpl; ++it) {
            const uint32_t e = it * 32 + lane;
            if ((uint32_t)it < nit) buf[e] = make_uint2(key[it], slot[it]);
        }
        __syncwarp();
        warp_tail(buf, s, out, B);
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// MEDIUM: one CTA per segment, LSD radix in shared memory
// ---------------------------------------------------------------------------
// Ascending bitonic sort of N = 8*NT values over the CTA (element e = 8*tid + r
// in register v[r]): strides < 8 in registers, < 256 by warp shuffles, larger
// ones through shared memory xs[N] -- a handful of block barriers in all.
template <int NT>
__device__ __forceinline__ void block_bitonic(uint32_t (&v)[8], uint32_t* xs) {
    constexpr int N = 8 * NT;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
        if (k <= 8) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int q = r ^ (k - 1);
                if (r < q) {
                    const uint32_t a = v[r], b = v[q];
                    v[r] = min(a, b);
                    v[q] = max(a, b);
                }
            }
        } else if (k <= 256) {
            const int lm = k / 8 - 1;
            const bool lower = (lane & (uint32_t)(k / 16)) == 0;
            uint32_t o[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) o[r] = __shfl_xor_sync(0xFFFFFFFFu, v[7 - r], lm);
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = lower ? min(v[r], o[r]) : max(v[r], o[r]);
        } else {
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 8; ++r) xs[8 * tid + r] = v[r];
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint32_t e = 8 * tid + r;
                const uint32_t o = xs[e ^ (uint32_t)(k - 1)];
                v[r] = (e & (uint32_t)(k / 2)) == 0 ? min(v[r], o) : max(v[r], o);
            }
        }
#pragma unroll
        for (int j = k >> 2; j > 0; j >>= 1) {
            if (j < 8) {
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    if ((r & j) == 0) {
                        const uint32_t a = v[r], b = v[r | j];
                        v[r] = min(a, b);
                        v[r | j] = max(a, b);
                    }
                }
            } else if (j < 256) {
                const int lj = j / 8;
                const bool lower = (lane & (uint32_t)lj) == 0;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, v[r], lj);
                    v[r] = lower ? min(v[r], o) : max(v[r], o);
                }
            } else {
                __syncthreads();
#pragma unroll
                for (int r = 0; r < 8; ++r) xs[8 * tid + r] = v[r];
                __syncthreads();
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const uint32_t e = 8 * tid + r;
                    const uint32_t o = xs[e ^ (uint32_t)j];
                    v[r] = (e & (uint32_t)j) == 0 ? min(v[r], o) : max(v[r], o);
                }
            }
        }
    }
    __syncthreads();
}

template <int CAP, int NT>
constexpr size_t local_smem() {
    return (size_t)CAP * 16 + (size_t)(NT / 32) * 256 * 4 + 260 * 4 + 32 * 4 + (CAP / 2) * 8 + 64;
}

template <int CAP, int NT>
__global__ void __launch_bounds__(NT) local_kernel(Lists in, Lists out, int cls, Bufs B,
                                                    uint32_t* misc) {
    constexpr int IPT = CAP / NT;
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* const keyA0 = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* const slotA0 = keyA0 + CAP;
    uint32_t* const keyB0 = slotA0 + CAP;
    uint32_t* const slotB0 = keyB0 + CAP;
    uint32_t* wcnt = slotB0 + CAP;          // NW*256
    uint32_t* dstart = wcnt + NW * 256;     // 257
    uint32_t* tmp = dstart + 260;           // 32
    uint2* runs = reinterpret_cast<uint2*>(tmp + 32);  // CAP/2
    __shared__ uint32_t n_runs;
    __shared__ int same_digit;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t n = in.cnt[cls];
    for (uint32_t si = blockIdx.x; si < n; si += gridDim.x) {
        uint32_t *keyA = keyA0, *slotA = slotA0, *keyB = keyB0, *slotB = slotB0;
        const Seg s = in.seg[cls][si];
        const uint32_t len = s.len;
        const uint32_t buf = meta_buf(s.meta);
        const bool kv = meta_kv(s.meta);
        uint32_t* S = B.sa[buf];
        if (tid == 0) {
            atomicAdd(misc + M_ELEMS_M, len);
            n_runs = 0;
        }
        for (uint32_t i = tid; i < len; i += NT) {
            const uint32_t sl = S[s.start + i];
            slotA[i] = sl;
            keyA[i] = kv ? B.key[buf][s.start + i] : key_of(B, sl, s.word);
        }
        __syncthreads();
        const uint32_t top = kv ? meta_shift(s.meta) : 24u;
        if (kv && top <= 8) {
            // <= 16 unknown key bits: one block bitonic sort of packed
            // (key bits << 12 | index) values (index = slot order, so stable)
            static_assert(CAP <= 4096 && IPT == 8, "block bitonic packing");
            const uint32_t rb = top + 8, rmask = (1u << rb) - 1u;
            const uint32_t hi = keyA[0] & ~rmask;
            uint32_t v[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint32_t e = 8 * tid + r;
                v[r] = e < len ? (((keyA[e] & rmask) << 12) | e) : 0xFFFFFFFFu;
            }
            block_bitonic<NT>(v, keyB);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint32_t e = 8 * tid + r;
                if (e < len) {
                    keyB[e] = hi | (v[r] >> 12);
                    slotB[e] = slotA[v[r] & 0xFFFu];
                }
            }
            __syncthreads();
            uint32_t* t;
            t = keyA; keyA = keyB; keyB = t;
            t = slotA; slotA = slotB; slotB = t;
        }
        // LSD passes over the digits not yet known to be equal
        for (uint32_t sh = 0; sh <= top && !(kv && top <= 8); sh += 8) {
            if (tid == 0) same_digit = 1;
            __syncthreads();
            const uint32_t d0 = (keyA[0] >> sh) & 0xFFu;
            bool same = true;
            for (uint32_t i = tid; i < len; i += NT) same &= ((keyA[i] >> sh) & 0xFFu) == d0;
            if (!same) same_digit = 0;
            __syncthreads();
            if (same_digit) continue;
            uint32_t dig[IPT], dest[IPT];
#pragma unroll
            for (int it = 0; it < IPT; ++it) {
                const uint32_t e = warp * (32 * IPT) + it * 32 + lane;
                dig[it] = e < len ? ((keyA[e] >> sh) & 0xFFu) : 0x100u;
            }
            block_rank<NT, IPT>(dig, dest, wcnt, dstart, tmp);
#pragma unroll
            for (int it = 0; it < IPT; ++it) {
                if (dig[it] < 256) {
                    const uint32_t e = warp * (32 * IPT) + it * 32 + lane;
                    keyB[dest[it]] = keyA[e];
                    slotB[dest[it]] = slotA[e];
                }
            }
            __syncthreads();
            uint32_t* t;
            t = keyA; keyA = keyB; keyB = t;
            t = slotA; slotA = slotB; slotB = t;
        }
        // write the order; collect tied runs (equal word, 14 real symbols)
        for (uint32_t i = tid; i < len; i += NT) {
            SB_ASSERT(s.start + i < B.n);
            B.saf[s.start + i] = slotA[i];
            const uint32_t k = keyA[i];
            const bool starts = (i == 0 || keyA[i - 1] != k) && i + 1 < len && keyA[i + 1] == k &&
                                (k & 15u) == B.ksyms;
            if (starts) {
                uint32_t L = 2;
                while (i + L < len && keyA[i + L] == k) ++L;
                runs[atomicAdd(&n_runs, 1u)] = make_uint2(i, L);
            }
        }
        __syncthreads();
        const uint32_t nr = n_runs;
        for (uint32_t r = warp; r < nr; r += NW) {
            const uint2 rr = runs[r];
            if (rr.y <= kTiny) {
                uint32_t sl = lane < rr.y ? slotA[rr.x + lane] : 0u;
                sl = warp_finish(sl, rr.y, s.word + 1, 0u, false, B);
                if (lane < rr.y) B.saf[s.start + rr.x + lane] = sl;
            } else {
                for (uint32_t q = lane; q < rr.y; q += 32) S[s.start + rr.x + q] = slotA[rr.x + q];
                if (lane == 0) emit(out, Seg{s.start + rr.x, rr.y, s.word + 1, make_meta(24, buf, 0, 0)});
            }
        }
        __syncthreads();
    }
}

__global__ void strip_payload_kernel(uint32_t* sa, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        sa[i] &= (1u << kPayloadShift) - 1u;
}

}  // namespace sortk

using namespace sortk;

cudaError_t sort_reserve(SortScratch& ws, uint32_t n_suf, const SortOpts& opts) {
    Profiler dummy;
    (void)dummy;
    return sort_block(dummy, nullptr, ws, nullptr, nullptr, 0, n_suf, nullptr, nullptr, true, opts,
                      nullptr);
}

cudaError_t sort_block(Profiler& prof, cudaStream_t s, SortScratch& ws, const uint32_t* text,
                       const uint32_t* term, uint64_t slot_base, uint32_t n_suf,
                       uint32_t* d_sa_final, SortStats* st, bool reserve_only,
                       const SortOpts& opts, const uint32_t* nbit) {
    if (n_suf == 0) return cudaSuccess;
    const size_t n = n_suf;
    const size_t cap[NCLASS] = {n / 2 + 1,   n / 33 + 1,   n / 65 + 1,   n / 129 + 1,
                                n / 257 + 1, n / 33 + 1,   n / 513 + 1,  n / 1025 + 1,
                                n / 2049 + 1, n / (kCapS + 1) + 1,   // LARGE: > 512 (kv, small blocks)
                                n / 2049 + 1,                        // LOCALD: 2049..4096 (kv)
                                n / (kCapS + 1) + 1};                // LOCALD2: 513..2048 (kv)
    const size_t max_large = cap[LARGE];
    const size_t max_chunks = n / kMinChunk + max_large + 1;
    uint32_t *sa0, *sa1, *k0, *k1, *hist, *ctr;
    SB_CHECK(ensure(ws.sa0, n, &sa0));
    SB_CHECK(ensure(ws.sa1, n, &sa1));
    SB_CHECK(ensure(ws.k0, n, &k0));
    SB_CHECK(ensure(ws.k1, n, &k1));
    size_t list_elems = 0;
    for (int c = 0; c < NCLASS; ++c) list_elems += cap[c];
    Seg *la, *lb;
    SB_CHECK(ensure(ws.segs_a, list_elems, &la));
    SB_CHECK(ensure(ws.segs_b, list_elems, &lb));
    SegX* segx;
    uint32_t* dbase;
    Chunk* chunks;
    SB_CHECK(ensure(ws.small_a, max_large, &segx));
    SB_CHECK(ensure(ws.small_b, max_large * 256, &dbase));
    SB_CHECK(ensure(ws.chunks, max_chunks, &chunks));
    SB_CHECK(ensure(ws.hist, max_chunks * 256, &hist));
    const size_t max_groups = max_chunks;  // <= one group per chunk
    uint32_t* gtot;
    Group* groups;
    SB_CHECK(ensure(ws.gtot, max_groups * 256, &gtot));
    SB_CHECK(ensure(ws.groups, max_groups, &groups));
    SB_CHECK(ensure(ws.ctr, 2 * NCLASS + M_N + 8, &ctr));
    uint32_t* misc = ctr + 2 * NCLASS;
    Lists A, Bl;
    {
        size_t off = 0;
        for (int c = 0; c < NCLASS; ++c) {
            A.seg[c] = la + off;
            Bl.seg[c] = lb + off;
            off += cap[c];
        }
        A.cnt = ctr;
        Bl.cnt = ctr + NCLASS;
        // the one-CTA digit pass pays on large blocks (c3: the ~2048-member
        // third level); smaller blocks (c2) keep the global digit passes
        static const uint64_t local_min =
            getenv("SETBWTE_LOCAL_MIN") ? (uint64_t)atoll(getenv("SETBWTE_LOCAL_MIN")) : (1ull << 25);
        A.local = Bl.local = (uint64_t)n >= local_min ? 1u : 0u;
    }
    if (reserve_only) return cudaSuccess;
    Bufs B;
    B.sa[0] = sa0;
    B.sa[1] = sa1;
    B.key[0] = k0;
    B.key[1] = k1;
    B.saf = d_sa_final;
    B.text = text;
    B.term = term;
    B.base = slot_base;
    B.smask = sa_slot_mask(n_suf, opts.payload_limit);
    B.n = n_suf;
    B.nbit = nbit;
    B.ksyms = nbit ? (uint32_t)kKeySyms5 : (uint32_t)kKeySyms;

    // (set on every call: cheap, per device, and safe from several host threads)
    constexpr size_t sm_m = local_smem<kCapM, kNtM>();
    constexpr size_t sm_m1 = local_smem<1024, 128>();
    constexpr size_t sm_m2 = local_smem<2048, 256>();
    SB_CHECK(cudaFuncSetAttribute(local_kernel<1024, 128>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_m1));
    SB_CHECK(cudaFuncSetAttribute(local_kernel<2048, 256>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_m2));
    constexpr size_t sm_d = scatter_smem<kDigIpt>();
    constexpr size_t sm_ld = local_digit_smem<512>();
    constexpr size_t sm_ld2 = local_digit_smem<256>();
    SB_CHECK(cudaFuncSetAttribute(local_digit_kernel<512>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_ld));
    SB_CHECK(cudaFuncSetAttribute(local_digit_kernel<256>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_ld2));
    SB_CHECK(cudaFuncSetAttribute(local_kernel<kCapM, kNtM>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_m));
    SB_CHECK(cudaFuncSetAttribute(digit_scatter_kernel<kDigIpt>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_d));

    if (n <= kCapM && !nbit) {
        SB_LAUNCH(prof, s, "sort_keygen", 4.375 * n, n,
                  keygen_kernel<<<grid_for((n + 15) / 16, 256, 148u * 16u), 256, 0, s>>>(
                      text, term, slot_base, n_suf, k0));
        SB_CHECK(cudaGetLastError());
    } else if (n <= kCapM) {
        SB_LAUNCH(prof, s, "sort_keygen", 4.5 * n, n,
                  keygen5_kernel<<<grid_for(n, 256, 148u * 16u), 256, 0, s>>>(
                      text, term, nbit, slot_base, n_suf, k0));
        SB_CHECK(cudaGetLastError());
    }
    SB_LAUNCH(prof, s, "sort_init", n <= kCapM ? 4.0 * n : 0.0, n,
              init_kernel<<<n <= kCapM ? grid_for(n, 256) : 1u, 256, 0, s>>>(sa0, d_sa_final, n_suf, A, Bl, misc, B));
    SB_CHECK(cudaGetLastError());
    uint32_t h_cnt[NCLASS] = {0}, h_oth[NCLASS] = {0};  // counts of in / out
    if (n > 1) h_cnt[class_of(Seg{0u, (uint32_t)n, 0u, 24u | (1u << 9)}, A.local)] = 1;
    Lists in = A, out = Bl;
    uint32_t prev_active = 0;
    uint32_t h_misc[M_N] = {0};
    // one round: the kernels of every class with a (recorded or read-back)
    // non-zero count, the consumed counts reset, the lists swapped
    auto run_round = [&](const uint32_t* cnt) -> cudaError_t {
        uint32_t mask = 0;
        for (int c = 0; c < NCLASS; ++c)
            if (cnt[c]) mask |= 1u << c;
        {
            const int cls[4] = {BIT2, BIT4, BIT8, BIT16};
            const char* nm[4] = {"sort_bitonic64", "sort_bitonic128", "sort_bitonic256",
                                 "sort_bitonic512"};
            for (int q = 0; q < 4; ++q) {
                const uint32_t c = cnt[cls[q]];
                if (!c) continue;
                const unsigned grid = grid_for((uint64_t)c * 32, kWarpCta * 32, 148u * 16u);
                switch (q) {
                    case 0: SB_LAUNCH(prof, s, nm[q], 0, 0, bitonic_kernel<2><<<grid, kWarpCta * 32, 0, s>>>(in, out, BIT2, B, misc)); break;
                    case 1: SB_LAUNCH(prof, s, nm[q], 0, 0, bitonic_kernel<4><<<grid, kWarpCta * 32, 0, s>>>(in, out, BIT4, B, misc)); break;
                    case 2: SB_LAUNCH(prof, s, nm[q], 0, 0, bitonic_kernel<8><<<grid, kWarpCta * 32, 0, s>>>(in, out, BIT8, B, misc)); break;
                    default: SB_LAUNCH(prof, s, nm[q], 0, 0, bitonic_kernel<16><<<grid, kWarpCta * 32, 0, s>>>(in, out, BIT16, B, misc)); break;
                }
                SB_CHECK(cudaGetLastError());
            }
        }
        if (cnt[TINY]) {
            SB_LAUNCH(prof, s, "sort_tiny", 0, 0,
                      tiny_kernel<<<grid_for(((uint64_t)cnt[TINY] + kTinyPerWarp - 1) / kTinyPerWarp * 32,
                                             256, 148u * 16u), 256, 0,
                                    s>>>(in, B, misc));
            SB_CHECK(cudaGetLastError());
        }
        if (cnt[SMALL]) {
            SB_LAUNCH(prof, s, "sort_small", 0, 0,
                      warp_sort_kernel<<<grid_for((uint64_t)cnt[SMALL] * 32, kWarpCta * 32,
                                                  148u * 8u),
                                         kWarpCta * 32, 0, s>>>(in, out, B, misc));
            SB_CHECK(cudaGetLastError());
        }
        if (cnt[MED1K]) {
            SB_LAUNCH(prof, s, "sort_medium", 0, 0,
                      (local_kernel<1024, 128><<<std::min<uint32_t>(cnt[MED1K], 148u * 12u), 128,
                                                  sm_m1, s>>>(in, out, MED1K, B, misc)));
            SB_CHECK(cudaGetLastError());
        }
        if (cnt[MED2K]) {
            SB_LAUNCH(prof, s, "sort_medium", 0, 0,
                      (local_kernel<2048, 256><<<std::min<uint32_t>(cnt[MED2K], 148u * 6u), 256,
                                                  sm_m2, s>>>(in, out, MED2K, B, misc)));
            SB_CHECK(cudaGetLastError());
        }
        // algorithmic bytes: the digit pass's read + write of (key, slot) per
        // member (16 B, added with the round's active count below)
        static const unsigned g_loc2 = getenv("SETBWTE_LOC_GRID") ? (unsigned)atoi(getenv("SETBWTE_LOC_GRID")) : 148u * 4u * 4u;
        if (cnt[LOCALD]) {
            SB_LAUNCH(prof, s, "sort_local_digit", 0, 0,
                      (local_digit_kernel<512><<<std::min<uint32_t>(cnt[LOCALD], 148u * 2u * 4u),
                                                 512, sm_ld, s>>>(in, out, B, misc)));
            SB_CHECK(cudaGetLastError());
        }
        if (cnt[LOCALD2]) {
            SB_LAUNCH(prof, s, "sort_local_digit", 0, 0,
                      (local_digit_kernel<256><<<std::min<uint32_t>(cnt[LOCALD2], g_loc2),
                                                 256, sm_ld2, s>>>(in, out, B, misc)));
            SB_CHECK(cudaGetLastError());
        }
        if (cnt[MEDIUM]) {
            SB_LAUNCH(prof, s, "sort_medium", 0, 0,
                      (local_kernel<kCapM, kNtM><<<std::min<uint32_t>(cnt[MEDIUM], 148u * 3u),
                                                   kNtM, sm_m, s>>>(in, out, MEDIUM, B, misc)));
            SB_CHECK(cudaGetLastError());
        }
        if (cnt[LARGE]) {
            SB_LAUNCH(prof, s, "sort_chunkify", 0, 0,
                      chunkify_kernel<<<grid_for((uint64_t)cnt[LARGE] * 32, 128), 128, 0, s>>>(
                          in, segx, chunks, groups, misc));
            SB_CHECK(cudaGetLastError());
            static const unsigned g_dig = getenv("SETBWTE_DIG_GRID") ? (unsigned)atoi(getenv("SETBWTE_DIG_GRID")) : 148u * 8u;
            SB_LAUNCH(prof, s, "digit_hist", 0, 0,
                      digit_hist_kernel<<<g_dig, kDigNt, 0, s>>>(in, chunks, misc, B, hist));
            SB_CHECK(cudaGetLastError());
            SB_LAUNCH(prof, s, "digit_scan", 0, 0,
                      group_scan_kernel<<<148u * 8u, 256, 0, s>>>(groups, misc, hist, gtot));
            SB_CHECK(cudaGetLastError());
            SB_LAUNCH(prof, s, "digit_scan", 0, 0,
                      digit_scan_kernel<<<std::min<uint32_t>(cnt[LARGE], 148u * 8u), 256, 0, s>>>(
                          in, out, segx, gtot, dbase, B.ksyms));
            SB_CHECK(cudaGetLastError());
            SB_LAUNCH(prof, s, "digit_scatter", 0, 0,
                      (digit_scatter_kernel<kDigIpt><<<g_dig, kDigNt, sm_d, s>>>(
                          in, segx, chunks, misc, hist, gtot, dbase, B)));
            SB_CHECK(cudaGetLastError());
        }
        SB_LAUNCH(prof, s, "sort_ctl", 0, 0,
                  reset_counts_kernel<<<1, 32, 0, s>>>(in.cnt, misc, mask));
        SB_CHECK(cudaGetLastError());
        std::swap(in, out);
        return cudaSuccess;
    };
    // one read-back of both count lists and misc (contiguous in ctr); a
    // pageable destination makes the copy return when the data is here (its
    // in-driver wait measured faster than pinned memory + a stream sync)
    auto read_back = [&]() -> cudaError_t {
        uint32_t h_all[2 * NCLASS + M_N];
        {
            TraceScope tr(TR_SORT_READBACK);
            SB_CHECK(cudaMemcpyAsync(h_all, ctr, sizeof(h_all), cudaMemcpyDeviceToHost, s));
            SB_CHECK(cudaStreamSynchronize(s));
        }
        memcpy(h_cnt, h_all + (in.cnt - ctr), sizeof(h_cnt));
        memcpy(h_oth, h_all + (out.cnt - ctr), sizeof(h_oth));
        memcpy(h_misc, h_all + 2 * NCLASS, sizeof(h_misc));
        if (h_misc[M_ACTIVE] != prev_active) {
            if (st) {
                st->active_per_pass.push_back(h_misc[M_ACTIVE] - prev_active);
                st->digit_passes++;
            }
            prev_active = h_misc[M_ACTIVE];
        }
        return cudaSuccess;
    };
    // replay a recorded launch pattern (no read-backs), then finish host-driven
    SortPattern* pat = opts.pattern;
    bool replayable = false;
    std::vector<std::vector<uint32_t>> rounds;
    if (pat && n >= (1u << 20)) {
        std::lock_guard<std::mutex> lk(pat->mu);
        if (!pat->rounds.empty() && pat->n + pat->n / 16 >= n && n + n / 16 >= pat->n) {
            rounds = pat->rounds;
            replayable = true;
        }
    }
    if (replayable) {
        for (const std::vector<uint32_t>& r : rounds) SB_CHECK(run_round(r.data()));
        SB_CHECK(read_back());
        if (st) st->replayed++;
    }
    std::vector<std::vector<uint32_t>> rec;
    uint32_t extra = 0;  // host-driven rounds after a replay
    for (;;) {
        uint32_t any_in = 0, any_out = 0;
        for (int c = 0; c < NCLASS; ++c) {
            any_in |= h_cnt[c];
            any_out |= h_oth[c];
        }
        if (!any_in && !any_out) break;
        if (!any_in) {
            // only carried-over segments left (a replayed round skipped their
            // class): they sit in the other list
            std::swap(in, out);
            std::swap(h_cnt, h_oth);
            continue;
        }
        if (!replayable) rec.emplace_back(h_cnt, h_cnt + NCLASS);
        else {
            if (st) st->after_replay++;
            ++extra;
        }
        SB_CHECK(run_round(h_cnt));
        SB_CHECK(read_back());
    }
    if (pat && !replayable && n >= (1u << 20)) {
        std::lock_guard<std::mutex> lk(pat->mu);
        if (pat->rounds.empty()) {
            pat->n = n;
            pat->rounds = rec;
            pat->misses = 0;
        }
    } else if (pat && replayable) {
        // a stale pattern (blocks of another read-length mix): re-record it
        // after two consecutive replays that needed extra host-driven rounds
        std::lock_guard<std::mutex> lk(pat->mu);
        pat->misses = extra > 1 ? pat->misses + 1 : 0;
        if (pat->misses >= 2) {
            pat->rounds.clear();
            pat->n = 0;
            pat->misses = 0;
        }
    }
    const uint64_t act_local = h_misc[M_ACTIVE];
    if (st) st->rounds++;
    // algorithmic bytes: a digit pass reads/writes the
    // (slot, key) pair -- histogram 8 B, scatter 16 B per active element; the
    // local sorts read (slot, key) and write the final SA entry (12 B/element).
    const uint64_t act_loc = h_misc[M_ACTIVE_LOC];
    prof.add_bytes("digit_hist", 8.0 * (act_local - act_loc), act_local - act_loc);
    prof.add_bytes("digit_scatter", 16.0 * (act_local - act_loc), act_local - act_loc);
    // + the key-word lookups of the in-place finish: two random 32-byte
    // sectors each (a text word pair and a terminator word pair), counted at
    // sector granularity like ComputeRanks' Blk reads
    prof.add_bytes("sort_local_digit", 16.0 * act_loc + 64.0 * h_misc[M_LOOKUPS], act_loc);
    prof.add_bytes("sort_tiny", 12.0 * h_misc[M_ELEMS_T], h_misc[M_ELEMS_T]);
    prof.add_bytes("sort_small", 12.0 * h_misc[M_ELEMS_S], h_misc[M_ELEMS_S]);
    prof.add_bytes("sort_medium", 12.0 * h_misc[M_ELEMS_M], h_misc[M_ELEMS_M]);
    prof.add_bytes("sort_bitonic", 12.0 * h_misc[M_ELEMS_B], h_misc[M_ELEMS_B]);
    return cudaSuccess;
}

cudaError_t launch_strip_payload(cudaStream_t s, uint32_t* sa, uint32_t n, uint64_t limit) {
    if (n == 0 || !sa_payload(n, limit)) return cudaSuccess;
    sortk::strip_payload_kernel<<<grid_for(n, 256), 256, 0, s>>>(sa, n);
    return cudaGetLastError();
}

}  // namespace setbwte
