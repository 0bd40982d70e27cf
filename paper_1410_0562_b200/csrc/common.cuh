// common.cuh -- shared device-side layouts and helpers of libsetbwte.so.
//
// Layouts:
//
// * Packed slot text.  An append of m strings is laid out in "slots":
//   string j occupies slots slot_off[j] .. slot_off[j+1]-1 with
//   slot_off[j] = offsets[j] + j, its last slot being the terminator
//   (string-major layout of Alg.2, reading R2).  `text` holds 2 bits
//   per slot, 16 slots per u32, BIG-endian inside the word (slot t of a word
//   sits at bits 31-2t..30-2t) so that 14 consecutive symbols are one shift
//   away from a 28-bit big-endian key.  Terminator slots hold code 0.
//   `term` holds 1 bit per slot (1 = terminator), 32 per u32, big-endian.
//   Both arrays carry two words of zero padding.
//
// * Rank dictionary of B_ext (the "occurrence counters" of Sec.5):
//   per 64 symbols one 32-byte Blk = u16 cnt[4] (occurrences of each code in
//   the enclosing 2^16-symbol superblock before this Blk) + three 64-bit
//   planes lo/hi (code bits) and dol ('$' flag; '$' stores code 0).  Per
//   superblock, u64 sb[4] = occurrences of each code before the superblock.
//   rank(c,i) = sb[i>>16][c] + blk[i>>6].cnt[c]
//             + popc(match_c(lo,hi) & ~dol & ((1<<(i&63))-1)).
//   n/64+1 Blks and n/2^16+1 superblocks are stored so that i = n is valid.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace setbwte {

struct __align__(32) Blk {
    uint16_t cnt[4];
    uint64_t lo;
    uint64_t hi;
    uint64_t dol;
};
static_assert(sizeof(Blk) == 32, "Blk must be one 32-byte sector");

constexpr int kSbShift = 16;                 // superblock = 2^16 symbols
constexpr int kBlkPerSb = 1 << (kSbShift - 6);  // 1024 Blks per superblock
constexpr int kKeySyms = 14;                 // symbols per 32-bit key word (reading R6)

// ---- packed text access ----------------------------------------------------

__device__ __forceinline__ uint32_t text_sym(const uint32_t* __restrict__ text, uint64_t p) {
    return (text[p >> 4] >> (30 - 2 * (uint32_t)(p & 15))) & 3u;
}

__device__ __forceinline__ bool term_bit(const uint32_t* __restrict__ term, uint64_t p) {
    return (term[p >> 5] >> (31 - (uint32_t)(p & 31))) & 1u;
}

// Key word d of the suffix starting at global slot p (Sec.3 P:88 "long integer
// keys made of multiple 32-bit words"; encoding = reading R6):
//   bits 31..4 : the 14 symbols at slots q..q+13, q = p + 14d, 2 bits each,
//                symbols at and after the first terminator replaced by code 0
//   bits  3..0 : number of real symbols before the first terminator in the
//                window, clamped to 14.
// Comparing key words is comparing the suffixes window by window with a
// terminator below every symbol; equal keys with a clamp < 14 mean identical
// suffixes (ties then go by string index = slot order).
__device__ __forceinline__ uint32_t suffix_key(const uint32_t* __restrict__ text,
                                               const uint32_t* __restrict__ term, uint64_t p,
                                               uint32_t d) {
    const uint64_t q = p + (uint64_t)kKeySyms * d;
    const uint64_t w = q >> 4;
    const uint32_t t = (uint32_t)(q & 15);
    const uint64_t v = ((uint64_t)__ldg(text + w) << 32) | __ldg(text + w + 1);
    uint32_t syms = (uint32_t)((v << (2 * t)) >> 36);  // 28 bits, slot q at the top
    const uint64_t tw = q >> 5;
    const uint32_t tt = (uint32_t)(q & 31);
    const uint64_t u = (((uint64_t)__ldg(term + tw) << 32) | __ldg(term + tw + 1)) << tt;
    uint32_t ended = (uint32_t)__clzll((long long)u);
    ended = ended > (uint32_t)kKeySyms ? (uint32_t)kKeySyms : ended;
    const uint32_t keep = 2 * ended;  // bits of real symbols to keep (from the top)
    const uint32_t mask = keep == 0 ? 0u : (0x0FFFFFFFu & ~((1u << (28 - keep)) - 1u));
    syms &= mask;
    return (syms << 4) | ended;
}

// ---- sigma = 5 (the fifth, largest symbol c_5, e.g. N of "ACGTN"; SPEC S:31,
// P:28 Sec.2) ---------------------------------------------------------------
// The packed text keeps its 2-bit plane; a third 1-bit-per-slot plane `nbit`
// (big-endian, like `term`) marks the slots holding code 4, whose 2-bit code
// is 0.  Key words then carry 3-bit symbols: 9 per word (kKeySyms5).
constexpr int kKeySyms5 = 9;

__device__ __forceinline__ uint32_t text_sym5(const uint32_t* __restrict__ text,
                                              const uint32_t* __restrict__ nbit, uint64_t p) {
    return term_bit(nbit, p) ? 4u : text_sym(text, p);
}

// Key word d of the suffix at slot p with 3-bit symbols (sigma = 5):
//   bit 31     : 0
//   bits 30..4 : the 9 symbols at slots q..q+8, q = p + 9d, 3 bits each
//                (codes 0..4), symbols at and after the first terminator 0
//   bits  3..0 : real symbols before the first terminator in the window,
//                clamped to 9.
// Same order argument as suffix_key (reading R6).
__device__ __forceinline__ uint32_t suffix_key5(const uint32_t* __restrict__ text,
                                                const uint32_t* __restrict__ term,
                                                const uint32_t* __restrict__ nbit, uint64_t p,
                                                uint32_t d) {
    const uint64_t q = p + (uint64_t)kKeySyms5 * d;
    const uint64_t w = q >> 4;
    const uint32_t t = (uint32_t)(q & 15);
    const uint64_t v = (((uint64_t)__ldg(text + w) << 32) | __ldg(text + w + 1)) << (2 * t);
    const uint64_t tw = q >> 5;
    const uint32_t tt = (uint32_t)(q & 31);
    const uint64_t u = (((uint64_t)__ldg(term + tw) << 32) | __ldg(term + tw + 1)) << tt;
    const uint64_t nn = (((uint64_t)__ldg(nbit + tw) << 32) | __ldg(nbit + tw + 1)) << tt;
    uint32_t ended = (uint32_t)__clzll((long long)u);
    ended = ended > (uint32_t)kKeySyms5 ? (uint32_t)kKeySyms5 : ended;
    uint32_t syms = 0;
#pragma unroll
    for (int k = 0; k < kKeySyms5; ++k) {
        const uint32_t c = (uint32_t)(v >> (62 - 2 * k)) & 3u;
        const uint32_t isn = (uint32_t)(nn >> (63 - k)) & 1u;
        syms = (syms << 3) | (isn ? 4u : c);
    }
    const uint32_t keep = 3 * ended;  // bits of real symbols to keep (from the top)
    const uint32_t mask = keep == 0 ? 0u : (0x07FFFFFFu & ~((1u << (27 - keep)) - 1u));
    syms &= mask;
    return (syms << 4) | ended;
}

// The N plane of B_ext's dictionary (sigma = 5), beside the Blk array: per
// 64 symbols the plane of code-4 symbols and their count since the enclosing
// superblock; per superblock u64 nsb = code-4 symbols before it.  In the Blk
// itself a code-4 symbol is stored like '$' (dol = 1, code 0), so the four
// Blk counters and match_plane() never see it; '$' is dol & ~n.
struct __align__(16) NBlk {
    uint64_t n;
    uint32_t cnt;
    uint32_t pad;
};
static_assert(sizeof(NBlk) == 16, "NBlk is 16 bytes");

// rank(c_5, i): code-4 symbols in B_ext[0, i)
__device__ __forceinline__ uint64_t dict_rank_n(const NBlk* __restrict__ nblk,
                                                const uint64_t* __restrict__ nsb, uint64_t i) {
    const NBlk* b = nblk + (i >> 6);
    uint64_t n, cw;
    asm("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(n), "=l"(cw) : "l"(b));
    const uint64_t mask = (1ull << (i & 63)) - 1ull;
    return __ldg(nsb + (i >> kSbShift)) + (uint32_t)cw + (uint64_t)__popcll(n & mask);
}

// ---- rank dictionary ---------------------------------------------------------

__device__ __forceinline__ uint64_t match_plane(uint32_t c, uint64_t lo, uint64_t hi, uint64_t dol) {
    const uint64_t a = (c & 1u) ? lo : ~lo;
    const uint64_t b = (c & 2u) ? hi : ~hi;
    return a & b & ~dol;
}

// The Blk array of B_ext, possibly split into shards held by different
// handles / GPUs (NEXT-3): shard q holds Blks [first[q], first[q+1]).  P = 1
// is the ordinary single array.  Device pointers of other shards are peer
// (UVA) pointers: reads of a remote shard go over NVLink.
constexpr int kMaxShards = 8;
struct Dict {
    const Blk* ptr[kMaxShards];
    uint64_t first[kMaxShards];
    int P;
};
__host__ __device__ inline Dict make_dict(const Blk* p) {
    Dict d;
    for (int q = 0; q < kMaxShards; ++q) {
        d.ptr[q] = nullptr;
        d.first[q] = ~0ull;
    }
    d.ptr[0] = p;
    d.first[0] = 0;
    d.P = 1;
    return d;
}
__device__ __forceinline__ const Blk* dict_blk(const Dict& d, uint64_t b) {
    int q = 0;
    for (int r = 1; r < d.P; ++r) {
        if (b < d.first[r]) break;
        q = r;
    }
    return d.ptr[q] + (b - d.first[q]);
}

__device__ __forceinline__ const Blk* blk_at(const Blk* p, uint64_t b) { return p + b; }
__device__ __forceinline__ const Blk* blk_at(const Dict& d, uint64_t b) { return dict_blk(d, b); }

// rank(c, i, B_ext) for a real symbol code c (Eq.(2)) -- one 32-byte Blk
// sector plus one superblock counter.
__device__ __forceinline__ uint64_t dict_rank(const Blk* __restrict__ blk,
                                              const uint64_t* __restrict__ sb, uint32_t c,
                                              uint64_t i) {
    const Blk* b = blk + (i >> 6);
    const uint64_t base = __ldg(sb + ((i >> kSbShift) << 2) + c);
    // the whole 32-byte Blk (one sector) in one 256-bit load
    uint64_t w0, w1, w2, w3;
    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
        : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3)
        : "l"(b));
    const uint32_t r = (uint32_t)((w0 >> (16 * c)) & 0xFFFFu);
    const uint64_t mask = (1ull << (i & 63)) - 1ull;
    return base + r + (uint64_t)__popcll(match_plane(c, w1, w2, w3) & mask);
}

__device__ __forceinline__ uint64_t dict_rank(const Dict& d, const uint64_t* __restrict__ sb,
                                              uint32_t c, uint64_t i) {
    const Blk* b = dict_blk(d, i >> 6);
    const uint64_t base = __ldg(sb + ((i >> kSbShift) << 2) + c);
    uint64_t w0, w1, w2, w3;
    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
        : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3)
        : "l"(b));
    const uint32_t r = (uint32_t)((w0 >> (16 * c)) & 0xFFFFu);
    const uint64_t mask = (1ull << (i & 63)) - 1ull;
    return base + r + (uint64_t)__popcll(match_plane(c, w1, w2, w3) & mask);
}

}  // namespace setbwte
