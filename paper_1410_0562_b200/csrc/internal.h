// internal.h -- host-side runtime pieces shared by the .cu files of
// libsetbwte.so (not part of the C-ABI; see include/setbwte.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace setbwte {

// A user device allocator (setbwte_set_allocator); empty = cudaMalloc/cudaFree.
struct Allocator {
    void* (*alloc)(size_t, void*) = nullptr;
    void (*free_)(void*, void*) = nullptr;
    void* ctx = nullptr;
};

// Growth-only device buffer (contents are NOT preserved on growth).  `owner`
// points at the handle's allocator slot (read at every growth); `fr`/`fctx`
// remember how the current allocation must be released.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    const Allocator* owner = nullptr;
    void (*fr)(void*, void*) = nullptr;
    void* fctx = nullptr;
};

cudaError_t ensure_bytes(DevBuf& b, size_t bytes);

template <class T>
inline cudaError_t ensure(DevBuf& b, size_t count, T** out) {
    cudaError_t e = ensure_bytes(b, count * sizeof(T) + 64);
    *out = static_cast<T*>(b.p);
    return e;
}

// Per-kernel accounting: launch counts always; CUDA-event time when profiling.
struct KStat {
    uint64_t launches = 0;
    double ms = 0.0;
    double bytes = 0.0;   // algorithmic bytes
    uint64_t units = 0;   // the unit the bytes are counted per (suffixes, LF steps, ...)
};

struct Profiler {
    bool on = false;
    std::string only;  // when set, only launches of this kernel name are timed
    struct Rec {
        std::string name;
        cudaEvent_t a, b;
        cudaStream_t s;
    };
    std::vector<Rec> pending;
    // mode 3 (timeline): every launch's start and end, ms after `ref` (an
    // event the append records on the main stream first; not owned here)
    bool tl = false;
    cudaEvent_t ref = nullptr;
    struct TL {
        std::string name;
        uint64_t stream;
        float t0, t1;
    };
    std::vector<TL> timeline;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, KStat> k;
    uint64_t total_launches = 0;

    cudaEvent_t get_event();
    void begin(const char* name, cudaStream_t s, double bytes, uint64_t units, cudaEvent_t* ev);
    void end(const char* name, cudaStream_t s, cudaEvent_t a);
    cudaError_t resolve();  // after a stream sync: accumulate event times
    void add_bytes(const char* name, double bytes, uint64_t units) {
        KStat& ks = k[name];
        ks.bytes += bytes;
        ks.units += units;
    }
    void reset();
    ~Profiler();
};

// Launch helper: counts the launch and brackets it with events when profiling.
#define SB_LAUNCH(prof, stream, name, bytes, units, ...)                    \
    do {                                                                    \
        cudaEvent_t _ev = nullptr;                                          \
        (prof).begin(name, stream, (double)(bytes), (uint64_t)(units), &_ev); \
        __VA_ARGS__;                                                        \
        (prof).end(name, stream, _ev);                                      \
    } while (0)

// Device-side bounds checks of the debug build (tools/variant.sh dbg ...
// "-DSB_DEBUG"): a failed check prints and traps, so the launch fails loudly.
#ifdef SB_DEBUG
#define SB_ASSERT(cond)                                                               \
    do {                                                                              \
        if (!(cond)) {                                                                \
            printf("SB_ASSERT failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);      \
            __trap();                                                                 \
        }                                                                             \
    } while (0)
#else
#define SB_ASSERT(cond) \
    do {                \
    } while (0)
#endif

#define SB_CHECK(expr)                             \
    do {                                           \
        cudaError_t _e = (expr);                   \
        if (_e != cudaSuccess) return _e;          \
    } while (0)

inline unsigned grid_for(uint64_t n, unsigned threads, unsigned cap = 148u * 32u) {
    uint64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// ---------------------------------------------------------------------------
// Stage launchers (each file documents its kernels).
// ---------------------------------------------------------------------------

// pack.cu -- A0: validate + pack an append (Alg.1; layout in common.cuh).
struct Packed {
    uint32_t* text;       // 2-bit slot text
    uint32_t* term;       // terminator bitmap
    uint32_t* nbit = nullptr;  // sigma = 5: code-4 bitmap (common.cuh), else null
    uint64_t* slot_off;   // m+1 slot offsets (slot_off[j] = offsets[j] + j)
    uint32_t* gfirst;     // string owning slot 32g, per 32-slot group
    uint64_t n_slots;
};
cudaError_t launch_pack(Profiler& prof, cudaStream_t s, const uint8_t* d_bytes,
                        const uint64_t* d_off, uint64_t m, uint64_t n_bytes,
                        const uint8_t* d_code_of, Packed pk, unsigned long long* d_err_pos,
                        int* d_bad_offsets);
// The two halves of launch_pack, so an append can pack block by block as its
// bytes arrive: slot offsets + group map + CSR check, then the 32-slot groups
// [g_begin, g_end).
cudaError_t launch_pack_prepare(Profiler& prof, cudaStream_t s, const uint64_t* d_off, uint64_t m,
                                uint64_t n_bytes, Packed pk, int* d_bad_offsets);
cudaError_t launch_pack_range(Profiler& prof, cudaStream_t s, const uint8_t* d_bytes,
                              uint64_t m, uint64_t n_bytes, const uint8_t* d_code_of, Packed pk,
                              uint64_t g_begin, uint64_t g_end, unsigned long long* d_err_pos);
// Greedy block partition (reading R8): blocks end at the first
// string boundary where the block holds >= M suffixes.  Writes K+1 pairs
// (string index, slot offset) into d_bounds and K into *d_k.
cudaError_t launch_partition(Profiler& prof, cudaStream_t s, const uint64_t* d_slot_off,
                             uint64_t m, uint64_t M, uint64_t* d_bounds, uint64_t* d_k);

// Split strings [j0, j1) into `parts` contiguous slices balanced by suffix
// count: out[r] = first string of slice r, out[parts] = j1, then
// out[parts+1+r] = slot_off[out[r]] (the slices' slot boundaries).
cudaError_t launch_slices(Profiler& prof, cudaStream_t s, const uint64_t* d_slot_off,
                          uint64_t j0, uint64_t j1, int parts, uint64_t* d_out);
// The same for each of the K blocks of a partition (d_bounds as written by
// launch_partition): 2*(parts+1) values per block, block after block.
cudaError_t launch_slices_blocks(Profiler& prof, cudaStream_t s, const uint64_t* d_slot_off,
                                 const uint64_t* d_bounds, uint64_t K, int parts,
                                 uint64_t* d_out);

// sort.cu -- A1 ConstructSA (Sec.3).
struct SortScratch {
    DevBuf sa0, sa1, k0, k1, segs_a, segs_b, small_a, small_b, chunks, hist, ctr, gtot, groups;
    void free_all();
    std::vector<DevBuf*> bufs();
};
struct SortStats {
    uint64_t digit_passes = 0;
    uint64_t rounds = 0;
    std::vector<uint64_t> active_per_pass;  // elements entering each digit pass
    uint64_t replayed = 0;      // blocks sorted by replaying a recorded launch pattern
    uint64_t after_replay = 0;  // host-driven rounds that had to follow a replay
};
struct SortOpts;
cudaError_t sort_reserve(SortScratch& ws, uint32_t n_suf, const SortOpts& opts);
// SA payload: while a block has fewer than 2^29 suffixes, every SA entry the
// sort moves is (slot | b << 29) with b = the block's B_int symbol of that
// suffix (2-bit code, or 4 for '$', Alg.1), attached when the slot is
// generated.  The gather then reads B_int with the SA entry instead of two
// random text lookups.
constexpr uint32_t kPayloadShift = 29;
// (limit: the handle's option "sa_payload"; 0 switches the payload off)
constexpr uint64_t kPayloadLimit = 1ull << kPayloadShift;
__host__ __device__ inline bool sa_payload(uint64_t n_suf, uint64_t limit = kPayloadLimit) {
    return n_suf < limit && n_suf < kPayloadLimit;
}
__host__ __device__ inline uint32_t sa_slot_mask(uint64_t n_suf, uint64_t limit = kPayloadLimit) {
    return sa_payload(n_suf, limit) ? (1u << kPayloadShift) - 1u : 0xFFFFFFFFu;
}
cudaError_t launch_strip_payload(cudaStream_t s, uint32_t* sa, uint32_t n, uint64_t limit);
// per-handle sort options (setbwte_set_option "sa_payload")
// The launch pattern of one host-driven sort (per round: the segment count of
// every size class), recorded once per handle from a block of >= 2^20
// suffixes and replayed for blocks of about the same size without reading
// counts back between rounds (the kernels read the real counts on the device;
// a class the pattern skips keeps its segments for a later round).  One
// read-back at the end decides whether host-driven rounds must follow.
struct SortPattern {
    std::mutex mu;
    uint32_t n = 0;                                   // block size it was recorded on
    std::vector<std::vector<uint32_t>> rounds;        // NCLASS counts per round
    uint32_t misses = 0;  // consecutive replays that needed host-driven rounds after it
    void drop() {
        std::lock_guard<std::mutex> lk(mu);
        rounds.clear();
        n = 0;
        misses = 0;
    }
};
struct SortOpts {
    uint64_t payload_limit = kPayloadLimit;
    SortPattern* pattern = nullptr;  // launch-pattern replay (null: every round host-driven)
};

cudaError_t sort_block(Profiler& prof, cudaStream_t s, SortScratch& ws, const uint32_t* text,
                       const uint32_t* term, uint64_t slot_base, uint32_t n_suf,
                       uint32_t* d_sa_final, SortStats* st, bool reserve_only = false,
                       const SortOpts& opts = SortOpts(), const uint32_t* nbit = nullptr);

// sigma = 5 (common.cuh NBlk): the text's code-4 plane and the dictionary's
// N plane + superblock counts, for the kernels that read them.
struct N5Dict {
    const uint32_t* nbit = nullptr;
    const NBlk* nblk = nullptr;
    const uint64_t* nsb = nullptr;
};
// ... and what Insert reads / writes of it.
struct N5Ins {
    const NBlk* in = nullptr;    // B_ext's N plane (n_in symbols; null when empty)
    NBlk* out = nullptr;         // B_ext-new's N plane
    uint64_t* ntot = nullptr;    // per output superblock code-4 total (scratch)
    uint64_t* nsb_out = nullptr; // B_ext-new's N superblock counters
};

// ranks.cu -- A3 ComputeRanks (Lemma 1, Alg.2) and the
// fused A2/A4 extraction + gather (Alg.1).
cudaError_t launch_compute_ranks(Profiler& prof, cudaStream_t s, const uint32_t* text,
                                 const uint64_t* slot_off, uint64_t j0, uint64_t j1,
                                 uint64_t slot_base, const Dict& blk, const uint64_t* sb,
                                 const uint64_t* d_C, uint64_t m_ext, uint64_t n_steps, void* g,
                                 int gw, uint8_t* bslot = nullptr, bool bing = false,
                                 const N5Dict* n5 = nullptr, bool one_wave = false);
// g / pos element width gw = 4 (u32, index < 2^32 symbols) or 8 (u64).
// Blocks without the SA payload get B_int from ComputeRanks: bslot (one byte
// per slot) with u32 g, or bing = the top byte of each u64 g.
// With sb_start != NULL also writes sb_start[0..nsb] (superblock slices of pos).
cudaError_t launch_merge_ranks(Profiler& prof, cudaStream_t s, const Blk* oblk, const uint64_t* osb,
                               const uint64_t* oC, uint64_t m_o, uint64_t n_o, const Blk* hblk,
                               const uint64_t* hsb, const uint64_t* hC, uint64_t init, void* gsa,
                               int gw);
cudaError_t launch_merge_pos(Profiler& prof, cudaStream_t s, const Blk* oblk, uint64_t n_o,
                             const void* gsa, void* pos, int gw, uint8_t* bint, uint64_t* sb_start,
                             uint64_t nsb);
cudaError_t launch_gather(Profiler& prof, cudaStream_t s, const uint32_t* text,
                          const uint32_t* term, uint64_t slot_base, const uint32_t* sa,
                          const void* g, uint32_t n_suf, void* pos, int gw, uint8_t* bint,
                          uint64_t* sb_start = nullptr, uint64_t nsb = 0,
                          const uint8_t* bslot = nullptr, uint64_t payload_limit = kPayloadLimit,
                          bool bing = false, const uint32_t* nbit = nullptr);

// gather.cu -- the g -> g_sa gather in bucketed passes (L2-local g reads).
struct GatherScratch {
    uint32_t* slot;  // n: SA slots partitioned by bucket
    void* gval;      // n x gw: g of those slots
    uint32_t* rows;  // 256 x tiles + 256: per-tile bucket offsets, bucket sizes
};
// scratch bytes for a block of n suffixes (GatherScratch carved from one buffer)
size_t gather_scratch_bytes(uint32_t n, int gw);
// log2 of the slots per bucket, or 0 = use the plain gather; mode 0 off,
// 1 auto (g larger than L2), 2 forced (tests)
uint32_t gather_buckets_shift(uint32_t n, int gw, int mode);
cudaError_t launch_gather_bucketed(Profiler& prof, cudaStream_t s, const uint32_t* text,
                                   const uint32_t* term, uint64_t slot_base, const uint32_t* sa,
                                   const void* g, uint32_t n_suf, void* pos, int gw,
                                   uint8_t* bint, uint64_t* sb_start, uint64_t nsb,
                                   const uint8_t* bslot, uint64_t payload_limit, bool bing,
                                   const uint32_t* nbit, uint32_t shift,
                                   const GatherScratch& ws);

// insert.cu -- A5 Insert + dictionary rebuild (Alg.1, Sec.5).
cudaError_t launch_insert(Profiler& prof, cudaStream_t s, const Dict& in_blk, uint64_t n_in,
                          const void* pos, int gw, const uint8_t* bint, uint64_t n_ins,
                          Blk* out_blk, uint64_t* out_sb, uint64_t* sb_tot,
                          const uint64_t* sb_start, uint64_t m_new, uint64_t* d_C,
                          const N5Ins* n5 = nullptr);
// Insert restricted to output superblocks [sb_begin, sb_end) (host tier)
// and the closing superblock scan.
cudaError_t launch_insert_range(Profiler& prof, cudaStream_t s, const Dict& in_blk, uint64_t n_in,
                                const void* pos, int gw, const uint8_t* bint, uint64_t n_ins,
                                Blk* out_blk, uint64_t* sb_tot, const uint64_t* sb_start,
                                uint64_t sb_begin, uint64_t sb_end, const N5Ins* n5 = nullptr);
cudaError_t launch_sb_scan(Profiler& prof, cudaStream_t s, const uint64_t* sb_tot, uint64_t nsb,
                           uint64_t* out_sb, uint64_t m_new, uint64_t* d_C);
cudaError_t launch_rank_batch(Profiler& prof, cudaStream_t s, const Dict& blk, const uint64_t* sb,
                              uint64_t n, const uint8_t* code_of, const uint8_t* c,
                              const uint64_t* k, uint64_t q, uint64_t* out,
                              const N5Dict* n5 = nullptr);
cudaError_t launch_count(Profiler& prof, cudaStream_t s, const Dict& blk, const uint64_t* sb,
                         uint64_t n, const uint64_t* d_C, const uint8_t* code_of,
                         const uint8_t* pat, const uint64_t* poff, uint64_t q, uint64_t* out,
                         const N5Dict* n5 = nullptr);
cudaError_t launch_decode(Profiler& prof, cudaStream_t s, const Dict& blk, uint64_t n,
                          const uint8_t* sym_ascii, uint8_t* out, const NBlk* nblk = nullptr);
// Debug/export: SA + B_int ASCII of a sorted block.
cudaError_t launch_bint_ascii(Profiler& prof, cudaStream_t s, const uint8_t* bint,
                              uint32_t n_suf, const uint8_t* sym_ascii, uint8_t* out);

// Host-side wait tracing (env SETBWTE_TRACE=1): wall time spent in each kind
// of host wait, summed over all threads, printed to stderr after each append.
enum TraceId { TR_SORT_READBACK, TR_MEMINFO, TR_APPEND_SYNC, TR_VALIDATE, TR_RANK_WAIT,
               TR_LANE_JOIN, TR_FINAL_SYNC, TR_TOTAL, TR_N };
bool trace_on();
void trace_add(int id, uint64_t ns);
void trace_dump();
struct TraceScope {
    int id;
    std::chrono::steady_clock::time_point t0;
    explicit TraceScope(int i) : id(i), t0(std::chrono::steady_clock::now()) {}
    ~TraceScope() {
        if (trace_on())
            trace_add(id, (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                              std::chrono::steady_clock::now() - t0).count());
    }
};

}  // namespace setbwte
