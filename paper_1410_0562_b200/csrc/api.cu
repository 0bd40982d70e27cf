// api.cu -- the host runtime behind include/setbwte.h: the handle, the
// per-append stage sequence of Algorithm 1 on one CUDA stream, the
// ping-pong B_ext dictionary, error state and statistics.
#include <ctype.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>
#include <sys/mman.h>

#include "internal.h"
#include "setbwte.h"

using namespace setbwte;

// ---------------------------------------------------------------------------
// DevBuf / Profiler
// ---------------------------------------------------------------------------
namespace setbwte {

static cudaError_t release(DevBuf& b) {
    cudaError_t e = cudaSuccess;
    if (b.p && b.fr) {
        // a user allocator does not order its free against our streams (a
        // caching allocator may hand the block out again at once): drain first
        e = cudaDeviceSynchronize();
        b.fr(b.p, b.fctx);
    } else if (b.p) {
        e = cudaFree(b.p);  // synchronises implicitly
    }
    b.p = nullptr;
    b.cap = 0;
    b.fr = nullptr;
    b.fctx = nullptr;
    return e;
}

cudaError_t ensure_bytes(DevBuf& b, size_t bytes) {
    if (bytes <= b.cap && b.p) return cudaSuccess;
    if (b.p) {
        cudaError_t e = release(b);
        if (e != cudaSuccess) return e;
    }
    size_t cap = bytes + bytes / 4;  // 1.25x headroom against regrowth
    const Allocator* al = b.owner;
    if (al && al->alloc) {
        b.p = al->alloc(cap, al->ctx);
        if (!b.p) return cudaErrorMemoryAllocation;
        b.fr = al->free_;
        b.fctx = al->ctx;
        // a caching allocator may return a block whose previous owner still
        // has work queued on the allocator's stream, which our streams do not
        // wait for: drain before the library writes it
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return e;
    } else {
        cudaError_t e = cudaMalloc(&b.p, cap);
        if (e != cudaSuccess) {
            b.p = nullptr;
            return e;
        }
    }
    b.cap = cap;
    return cudaSuccess;
}

static void free_buf(DevBuf& b) { release(b); }

std::vector<DevBuf*> SortScratch::bufs() {
    return {&sa0, &sa1, &k0, &k1, &segs_a, &segs_b, &small_a, &small_b, &chunks, &hist,
            &ctr, &gtot, &groups};
}

void SortScratch::free_all() {
    for (DevBuf* b : bufs()) free_buf(*b);
}

static std::atomic<uint64_t> g_trace_ns[TR_N], g_trace_cnt[TR_N];

bool trace_on() {
    static const bool on = getenv("SETBWTE_TRACE") && atoi(getenv("SETBWTE_TRACE")) > 0;
    return on;
}

void trace_add(int id, uint64_t ns) {
    g_trace_ns[id] += ns;
    g_trace_cnt[id] += 1;
}

void trace_dump() {
    if (!trace_on()) return;
    static const char* names[TR_N] = {"sort_readback", "meminfo", "append_sync", "validate",
                                      "rank_wait", "lane_join", "final_sync", "total"};
    fprintf(stderr, "[setbwte trace]");
    for (int i = 0; i < TR_N; ++i) {
        fprintf(stderr, " %s=%.2fms/%llu", names[i], g_trace_ns[i].exchange(0) / 1e6,
                (unsigned long long)g_trace_cnt[i].exchange(0));
    }
    fprintf(stderr, "\n");
}

cudaEvent_t Profiler::get_event() {
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void Profiler::begin(const char* name, cudaStream_t s, double bytes, uint64_t units,
                     cudaEvent_t* ev) {
    KStat& ks = k[name];
    ks.launches++;
    ks.bytes += bytes;
    ks.units += units;
    total_launches++;
    if (on && (only.empty() || only == name)) {
        *ev = get_event();
        cudaEventRecord(*ev, s);
    }
}

void Profiler::end(const char* name, cudaStream_t s, cudaEvent_t a) {
    if (on && a) {
        cudaEvent_t b = get_event();
        cudaEventRecord(b, s);
        pending.push_back(Rec{name, a, b, s});
    }
}

cudaError_t Profiler::resolve() {
    cudaError_t err = cudaSuccess;
    for (Rec& r : pending) {
        float ms = 0.f;
        cudaError_t e = cudaEventElapsedTime(&ms, r.a, r.b);
        if (e == cudaSuccess) k[r.name].ms += ms; else err = e;
        if (tl && ref && e == cudaSuccess) {
            float t0 = 0.f, t1 = 0.f;
            if (cudaEventElapsedTime(&t0, ref, r.a) == cudaSuccess &&
                cudaEventElapsedTime(&t1, ref, r.b) == cudaSuccess)
                timeline.push_back(TL{r.name, (uint64_t)(uintptr_t)r.s, t0, t1});
        }
        pool.push_back(r.a);
        pool.push_back(r.b);
    }
    pending.clear();
    return err;
}

void Profiler::reset() {
    for (Rec& r : pending) {
        pool.push_back(r.a);
        pool.push_back(r.b);
    }
    pending.clear();
    k.clear();
    timeline.clear();
    total_launches = 0;
}

Profiler::~Profiler() {
    for (Rec& r : pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

}  // namespace setbwte

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (setbwte_set_comm).  A communicator must be used
// with the NCCL instance that created it: libnccl.so.2 already loaded into
// the process (e.g. by PyTorch) is taken first (RTLD_NOLOAD), else the
// system's.  The library therefore has no link-time NCCL dependency.
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
    bool ok = false;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclCommCount) comm_count = nullptr;
    decltype(&ncclCommUserRank) comm_user_rank = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) return a;
        a.group_start = (decltype(a.group_start))dlsym(lib, "ncclGroupStart");
        a.group_end = (decltype(a.group_end))dlsym(lib, "ncclGroupEnd");
        a.broadcast = (decltype(a.broadcast))dlsym(lib, "ncclBroadcast");
        a.comm_count = (decltype(a.comm_count))dlsym(lib, "ncclCommCount");
        a.comm_user_rank = (decltype(a.comm_user_rank))dlsym(lib, "ncclCommUserRank");
        a.error_string = (decltype(a.error_string))dlsym(lib, "ncclGetErrorString");
        a.ok = a.group_start && a.group_end && a.broadcast && a.comm_count && a.comm_user_rank;
        return a;
    }();
    return api;
}
}  // namespace

// ---------------------------------------------------------------------------
// Handle
// ---------------------------------------------------------------------------
struct DevErr {
    unsigned long long err_pos;
    int bad_offsets;
    int pad;
};

struct setbwte_s {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;       // main stream (user's, or own_stream)
    static constexpr int kMaxLanes = 4;
    cudaStream_t lane_stream[kMaxLanes] = {};  // ConstructSA of upcoming blocks, one per sort lane
    cudaStream_t copy_stream = nullptr;   // packing of an append's bytes, block by block
    cudaStream_t h2d_stream = nullptr;    // H2D of host input, in chunks (starts before the partition)
    std::vector<cudaEvent_t> ev_chunk;    // per H2D chunk: its bytes are on the device
    std::vector<cudaEvent_t> ev_packed;   // per block: its slots (and the next block's first group) packed
    DevErr* derr_host = nullptr;          // pinned landing spot for the validation result
    cudaEvent_t ev_start = nullptr, ev_sorted[kMaxLanes] = {}, ev_used[kMaxLanes] = {};
    Profiler prof;
    bool failed = false;

    // alphabet
    char alpha[6] = {0};
    int sigma = 0;
    uint8_t code_of[256];
    DevBuf d_code_of, d_sym;

    // the index: B_ext as a rank dictionary, ping-pong (reading: Sec.5)
    uint64_t n = 0, m = 0;
    DevBuf blk[2], sb[2];
    DevBuf nblk[2], nsb[2], ntot;  // sigma = 5: the N plane (common.cuh NBlk), ping-pong
    int cur = 0;
    DevBuf d_C, sb_tot;

    // append scratch
    DevBuf in_bytes, in_off, text, term, nbit, slot_off, gfirst, bounds, err, small;
    DevBuf saf, g, pos, bint, outbuf, bslot, gtmp;
    SortScratch sort[kMaxLanes];  // sort[0] also serves the inline (sort_lanes = 0) path
    Allocator user_alloc;         // setbwte_set_allocator (empty: cudaMalloc)

    // options
    uint64_t M = 1ull << 24;
    int sort_lanes = -1;   // host sort lanes; 0 = no pipelining (every stage on the main stream);
                           // -1 = automatic (lanes_for)
    uint64_t lanes_checked_suf = 0;  // largest block the lane count was checked against free memory
    int lanes_checked_nl = 0;        // ... and the lane count that fitted
    uint64_t hbm_budget = ~0ull;  // max bytes of B_ext dictionary kept in HBM

    // host tier: B_ext's dictionary in pinned, mapped
    // host memory (zero-copy for ComputeRanks / queries), rewritten in place
    // by Insert through HBM staging, top superblock range first
    bool host_tier = false;
    Blk* hdict = nullptr;       // host pointer (mmap'd, registered mapped + portable)
    Blk* hdict_dev = nullptr;   // device alias
    uint64_t hdict_cap = 0;     // capacity in Blks
    size_t hdict_bytes = 0;     // bytes mapped
    // the host Insert's read-ahead pipeline: staging H2D / write-back D2H
    cudaStream_t tier_in = nullptr, tier_out = nullptr;
    cudaEvent_t ev_staged[2] = {}, ev_merged[2] = {}, ev_written[2] = {};
    DevBuf stage_in, stage_out;
    std::vector<uint64_t> h_sb_start;

    // reverse orientation: the strings of the running call go BEFORE
    // every string already indexed, so a new terminator is the smallest suffix
    bool prepending = false;
    // the running append started on an empty index: a failure after its first
    // Insert empties the index again instead of failing the handle
    bool started_empty = false;

    // data-parallel ComputeRanks (and, with insert_split, Insert by output range)
    int rank = 0, world = 1;
    bool insert_split = false;
    bool sort_split = false;  // rank (k mod P) sorts block k, SA_int shared (NEXT-1 / C3)
    // NEXT-3: B_ext sharded by output superblock range across the ranks;
    // every rank keeps only its shard (ping-pong) and reads the others'
    // through their device pointers (peer / UVA)
    bool sharded = false;
    DevBuf shard_buf[2], shard_ptrs;
    int shard_cur = 0;
    bool shard_ipc = false;  // ranks are separate processes: exchange CUDA IPC handles
    std::vector<std::pair<uint64_t, void*>> ipc_open[kMaxShards];  // peer address -> opened mapping
    std::vector<void*> shard_retired;  // outgrown shard allocations (freed at destroy)
    Dict shard_dict = make_dict(nullptr);
    SortOpts sopt;                           // option "sa_payload"
    SortPattern sort_pattern;                // recorded launch pattern (sopt.pattern)
    int g_width = 0;                         // option "g_width": 0 auto, 8 = always u64
    int gather_mode = 0;                     // option "gather_buckets": 0 off, 1 auto, 2 forced
    setbwte_allgather_fn allgather = nullptr;
    void* allgather_ctx = nullptr;
    ncclComm_t nccl = nullptr;       // setbwte_set_comm: exchanges run in-library on NCCL
    bool force_exchange = false;     // option "force_exchange" (test hook: exchange at world 1)
    // per block of the running append, this rank partition's string / slot
    // boundaries for ComputeRanks: (world+1) string indices then (world+1)
    // slot offsets (computed on the device, read back once per append)
    std::vector<uint64_t> blk_slices;

    // diagnostics
    uint64_t err_pos = 0;
    uint8_t err_byte = 0;
    uint64_t last_blocks = 0, last_bases = 0, last_m = 0;
    SortStats sstats;
    std::string stats_json;
};

namespace {

setbwte_status from_cuda(setbwte_t h, cudaError_t e) {
    if (e == cudaSuccess) return SETBWTE_OK;
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) return SETBWTE_E_NOMEM;
    if (h) h->failed = true;
    return SETBWTE_E_CUDA;
}

// A failing CUDA call: with SETBWTE_DEBUG set in the environment, its error
// and source line go to stderr (the C ABI itself only returns E_CUDA / E_NOMEM).
#define API_CHECK(h, expr)                                                          \
    do {                                                                            \
        cudaError_t _e = (expr);                                                    \
        if (_e != cudaSuccess) {                                                    \
            if (getenv("SETBWTE_DEBUG"))                                            \
                fprintf(stderr, "setbwte: %s at api.cu:%d\n", cudaGetErrorString(_e), \
                        __LINE__);                                                  \
            return from_cuda((h), _e);                                              \
        }                                                                           \
    } while (0)

#define API_ENTER(h)                                          \
    do {                                                      \
        if (!(h)) return SETBWTE_E_INVALID_ARG;               \
        if ((h)->failed) return SETBWTE_E_STATE;              \
        cudaError_t _d = cudaSetDevice((h)->device);          \
        if (_d != cudaSuccess) return from_cuda((h), _d);     \
    } while (0)

struct PackOut {
    Packed pk;
    uint64_t n_bytes = 0;
};

// Validate + pack an append whose inputs are already on the device.
setbwte_status pack_input(setbwte_t h, const uint8_t* d_bytes, const uint64_t* d_off, uint64_t m,
                          PackOut* out) {
    uint64_t n_bytes = 0;
    API_CHECK(h, cudaMemcpyAsync(&n_bytes, d_off + m, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                 h->stream));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    const uint64_t n_slots = n_bytes + m;
    const uint64_t n_groups = (n_slots + 31) / 32;
    Packed pk;
    pk.n_slots = n_slots;
    API_CHECK(h, ensure(h->text, 2 * n_groups + 8, &pk.text));
    API_CHECK(h, ensure(h->term, n_groups + 8, &pk.term));
    if (h->sigma == 5) API_CHECK(h, ensure(h->nbit, n_groups + 8, &pk.nbit));
    API_CHECK(h, ensure(h->slot_off, m + 2, &pk.slot_off));
    API_CHECK(h, ensure(h->gfirst, n_groups + 2, &pk.gfirst));
    DevErr* derr;
    API_CHECK(h, ensure(h->err, 1, &derr));
    DevErr init{~0ull, 0, 0};
    API_CHECK(h, cudaMemcpyAsync(derr, &init, sizeof(init), cudaMemcpyHostToDevice, h->stream));
    API_CHECK(h, launch_pack(h->prof, h->stream, d_bytes, d_off, m, n_bytes,
                             (const uint8_t*)h->d_code_of.p, pk, &derr->err_pos,
                             &derr->bad_offsets));
    DevErr res;
    API_CHECK(h, cudaMemcpyAsync(&res, derr, sizeof(res), cudaMemcpyDeviceToHost, h->stream));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    if (res.bad_offsets) return SETBWTE_E_INVALID_ARG;
    if (res.err_pos != ~0ull) {
        h->err_pos = res.err_pos;
        uint8_t b = 0;
        API_CHECK(h, cudaMemcpy(&b, d_bytes + res.err_pos, 1, cudaMemcpyDeviceToHost));
        h->err_byte = b;
        return SETBWTE_E_INVALID_CHAR;
    }
    out->pk = pk;
    out->n_bytes = n_bytes;
    return SETBWTE_OK;
}

// Dictionary accessors for the current B_ext.
inline const Blk* cur_blk(setbwte_t h) {
    return h->host_tier ? h->hdict_dev : (const Blk*)h->blk[h->cur].p;
}
inline const uint64_t* cur_sb(setbwte_t h) { return (const uint64_t*)h->sb[h->cur].p; }
// sigma = 5: the N plane of the current B_ext (and the text's code-4 plane)
inline N5Dict cur_n5(setbwte_t h, const uint32_t* nbit = nullptr) {
    N5Dict d;
    d.nbit = nbit;
    d.nblk = (const NBlk*)h->nblk[h->cur].p;
    d.nsb = (const uint64_t*)h->nsb[h->cur].p;
    return d;
}
// The current B_ext Blks as a (possibly sharded) Dict.
inline Dict cur_dict(setbwte_t h) { return h->sharded ? h->shard_dict : make_dict(cur_blk(h)); }

// B_ext's dictionary (4 bits/symbol) larger than ~half the L2: ComputeRanks'
// LF walk is DRAM-bound rather than L2-latency-bound.
// (Not the host tier: its zero-copy walk is PCIe-latency-bound and wants every
// read in flight it can get.)
inline bool dict_beyond_l2(setbwte_t h) { return !h->host_tier && (h->n >> 1) > (64ull << 20); }

// True when the running appends split ComputeRanks across ranks.
inline bool partitioned(setbwte_t h) { return h->world > 1 || h->force_exchange; }

// The one exchange step of the data-parallel path: an
// all-gather-v in place.  buf is a DEVICE buffer holding the concatenation of
// every rank's slice (bytes_per_rank[r] bytes for rank r, in rank order);
// this rank's slice is queued on the main stream; afterwards (in stream order)
// every slice is filled.  With a communicator (setbwte_set_comm) it is one
// NCCL group of `world` in-place broadcasts (root r sends slice r) on the main
// stream -- no host synchronisation; else the setbwte_set_partition callback.
setbwte_status exchange(setbwte_t h, void* buf, const uint64_t* bytes_per_rank) {
    if (h->nccl) {
        const NcclApi& nc = nccl_api();
        if (!nc.ok) return SETBWTE_E_NCCL;
        ncclResult_t r = nc.group_start();
        uint64_t off = 0;
        for (int q = 0; q < h->world && r == ncclSuccess; ++q) {
            if (bytes_per_rank[q]) {
                char* p = static_cast<char*>(buf) + off;
                r = nc.broadcast(p, p, bytes_per_rank[q], ncclUint8, q, h->nccl, h->stream);
            }
            off += bytes_per_rank[q];
        }
        const ncclResult_t r2 = nc.group_end();
        if (r != ncclSuccess || r2 != ncclSuccess) {
            if (getenv("SETBWTE_DEBUG") && nc.error_string)
                fprintf(stderr, "setbwte: NCCL %s\n", nc.error_string(r != ncclSuccess ? r : r2));
            return SETBWTE_E_NCCL;
        }
        return SETBWTE_OK;
    }
    if (h->world <= 1) return SETBWTE_OK;  // force_exchange without a communicator: nothing to do
    if (!h->allgather) return SETBWTE_E_STATE;
    if (h->allgather(buf, bytes_per_rank, h->world, (void*)h->stream, h->allgather_ctx) != 0)
        return SETBWTE_E_STATE;
    return SETBWTE_OK;
}

// ComputeRanks for strings [j0, j1) of a packed append, into g (block-local
// slots starting at slot_base).  With world > 1, only this rank's slice is
// computed and the slices are exchanged (exchange()).  `slices` (optional):
// the block's precomputed partition, (world+1) string indices then (world+1)
// slot offsets; without it the partition is computed and read back here.
setbwte_status compute_ranks_for(setbwte_t h, const Packed& pk, uint64_t j0, uint64_t j1,
                                 uint64_t slot_base, uint64_t n_suf, void* g, int gw,
                                 uint8_t* bslot = nullptr, bool bing = false,
                                 const uint64_t* slices = nullptr) {
    if (h->n == 0) {
        // empty B_ext: every suffix has rank 0
        API_CHECK(h, cudaMemsetAsync(g, 0, n_suf * gw, h->stream));
        return SETBWTE_OK;
    }
    const N5Dict n5 = cur_n5(h, pk.nbit);
    const N5Dict* n5p = h->sigma == 5 ? &n5 : nullptr;
    if (!partitioned(h)) {
        API_CHECK(h, launch_compute_ranks(h->prof, h->stream, pk.text, pk.slot_off, j0, j1,
                                          slot_base, cur_dict(h), cur_sb(h),
                                          (const uint64_t*)h->d_C.p, h->prepending ? 0 : h->m,
                                          n_suf - (j1 - j0), g, gw, bslot, bing, n5p,
                                          dict_beyond_l2(h)));
        return SETBWTE_OK;
    }
    // data-parallel over strings: balanced slices by suffix count
    const int P = h->world;
    std::vector<uint64_t> own;
    if (!slices) {
        // one-off call (setbwte_compute_ranks): partition and read back here
        uint64_t* d_sl;
        API_CHECK(h, ensure(h->small, 2 * (size_t)P + 8, &d_sl));
        API_CHECK(h, launch_slices(h->prof, h->stream, pk.slot_off, j0, j1, P, d_sl));
        own.resize(2 * (P + 1));
        API_CHECK(h, cudaMemcpyAsync(own.data(), d_sl, sizeof(uint64_t) * 2 * (P + 1),
                                     cudaMemcpyDeviceToHost, h->stream));
        API_CHECK(h, cudaStreamSynchronize(h->stream));
        slices = own.data();
    }
    const uint64_t* sl = slices;               // string boundaries
    const uint64_t* slot_of = slices + P + 1;  // their slot offsets
    const uint64_t a = sl[h->rank], b = sl[h->rank + 1];
    const uint64_t steps = (slot_of[h->rank + 1] - slot_of[h->rank]) - (b - a);
    API_CHECK(h, launch_compute_ranks(h->prof, h->stream, pk.text, pk.slot_off, a, b, slot_base,
                                      cur_dict(h), cur_sb(h), (const uint64_t*)h->d_C.p,
                                      h->prepending ? 0 : h->m, steps, g, gw, nullptr,
                                      false, n5p, dict_beyond_l2(h)));
    std::vector<uint64_t> bytes(P);
    for (int r = 0; r < P; ++r) bytes[r] = (uint64_t)gw * (slot_of[r + 1] - slot_of[r]);
    return exchange(h, g, bytes.data());
}

// Algorithm 1 for one block of strings [j0, j1) occupying slots
// [S0, S1) of the packed append, split in two stages on two streams so that
// ConstructSA of block k+1 (sort stream) overlaps ComputeRanks / gather /
// Insert of block k (main stream): the sort has no B_ext dependency
// (the paper's stage pipeline P:190-191).
struct BlockDesc {
    uint64_t j0, j1, S0, S1;
    uint64_t ev;  // index of the ev_packed event after which its slots are packed
    uint64_t id;  // block index in the append (h->blk_slices)
};

// Pinned mapped host buffer for the dictionary with >= nblk Blks, keeping
// the first keep_blks of the current content.  Capacity grows 1.5x, so the
// host memory stays <= 1.5 x 4 bits/symbol = 6 bits = 3 n log(sigma) for
// sigma = 4 -- at EVERY instant: the buffer is an anonymous
// mapping that grows with mremap (the kernel moves the page mappings; no
// second buffer and no copy), registered with CUDA as mapped memory.
static void host_dict_free(setbwte_t h) {
    if (!h->hdict) return;
    cudaHostUnregister(h->hdict);
    munmap(h->hdict, h->hdict_bytes);
    h->hdict = nullptr;
    h->hdict_dev = nullptr;
    h->hdict_cap = 0;
    h->hdict_bytes = 0;
}

setbwte_status host_reserve(setbwte_t h, uint64_t nblk, const Blk* src, bool src_dev,
                            uint64_t keep_blks) {
    const uint64_t cap = std::max<uint64_t>(nblk + nblk / 2, 1024);
    const size_t bytes = ((size_t)cap * sizeof(Blk) + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);
    // nothing may read the old mapping while it moves
    API_CHECK(h, cudaDeviceSynchronize());
    void* p = nullptr;
    if (h->hdict && !src_dev) {
        // grow in place (keep_blks of the old content travel with the pages)
        API_CHECK(h, cudaHostUnregister(h->hdict));
        p = mremap(h->hdict, h->hdict_bytes, bytes, MREMAP_MAYMOVE);
        if (p == MAP_FAILED) {
            // the old mapping is intact: register it again and report
            cudaHostRegister(h->hdict, h->hdict_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
            return SETBWTE_E_NOMEM;
        }
    } else {
        host_dict_free(h);
        p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p == MAP_FAILED) return SETBWTE_E_NOMEM;
    }
    h->hdict = (Blk*)p;
    h->hdict_bytes = bytes;
    madvise(p, bytes, MADV_HUGEPAGE);
    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        munmap(p, bytes);
        h->hdict = nullptr;
        h->hdict_bytes = 0;
        h->hdict_cap = 0;
        // a grown mapping took the dictionary's content with it
        if (keep_blks && !src_dev) h->failed = true;
        return from_cuda(h, e);
    }
    void* pd = nullptr;
    API_CHECK(h, cudaHostGetDevicePointer(&pd, p, 0));
    if (keep_blks && src_dev)
        API_CHECK(h, cudaMemcpyAsync(p, src, keep_blks * sizeof(Blk), cudaMemcpyDeviceToHost,
                                     h->stream));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    h->hdict_dev = (Blk*)pd;
    h->hdict_cap = cap;
    return SETBWTE_OK;
}

// Insert with B_ext in host memory: output superblocks in chunks from the top
// down; each chunk's external input range is staged into HBM, merged, and
// written back in place.  A chunk writes [O0, O1) and reads external symbols
// [E0, E1) with E1 <= O1 = the first output symbol of the chunk above it
// (an output index is never below its input index), so no write-back of a
// higher chunk touches an input symbol of a lower one.  So the staging H2D of the next (lower)
// chunk runs while this chunk merges and writes back: a read-ahead pipeline
// on three streams with double-buffered staging (the one extra Blk a stage
// reads past E1 only feeds bits the merge never uses).
setbwte_status host_insert(setbwte_t h, const void* pos, int gw, const uint8_t* bint,
                           uint64_t n_suf, uint64_t* osb, uint64_t* tot, uint64_t* sb_start,
                           uint64_t m_new) {
    const uint64_t n_in = h->n, n_out = n_in + n_suf;
    const uint64_t nblk = (n_out >> 6) + 1, nsb = (n_out >> kSbShift) + 1;
    if (!h->hdict || h->hdict_cap < nblk) {
        setbwte_status st = host_reserve(h, nblk, h->hdict, false, h->hdict ? (n_in >> 6) + 1 : 0);
        if (st != SETBWTE_OK) return st;
    }
    h->h_sb_start.resize(nsb + 1);
    API_CHECK(h, cudaMemcpyAsync(h->h_sb_start.data(), sb_start, (nsb + 1) * sizeof(uint64_t),
                                 cudaMemcpyDeviceToHost, h->stream));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    constexpr uint64_t CS = 1024;  // superblocks per chunk (2^26 symbols, 32 MB of Blks)
    Blk *sin, *sout;
    // two staging buffers of each kind
    API_CHECK(h, ensure(h->stage_in, 2 * (CS * kBlkPerSb + 8), &sin));
    API_CHECK(h, ensure(h->stage_out, 2 * (CS * kBlkPerSb + 8), &sout));
    const uint64_t nin_blk = n_in ? (n_in >> 6) + 1 : 0;
    // the pipeline starts after everything queued on the main stream
    API_CHECK(h, cudaEventRecord(h->ev_start, h->stream));
    API_CHECK(h, cudaStreamWaitEvent(h->tier_in, h->ev_start, 0));
    API_CHECK(h, cudaStreamWaitEvent(h->tier_out, h->ev_start, 0));
    int q = 0;
    for (int64_t c = (int64_t)((nsb - 1) / CS); c >= 0; --c, ++q) {
        const int b = q & 1;
        Blk* si = sin + b * (CS * kBlkPerSb + 8);
        Blk* so = sout + b * (CS * kBlkPerSb + 8);
        const uint64_t sa = (uint64_t)c * CS, sbe = std::min(nsb, sa + CS);
        const uint64_t O0 = sa << kSbShift, Oe = std::min(sbe << kSbShift, n_out);
        const uint64_t E0 = O0 - h->h_sb_start[sa];
        const uint64_t E1 = std::min(n_in, Oe - h->h_sb_start[sbe]);
        uint64_t bE0 = 0, bE1 = 0;
        // stage the chunk's input once the merge two chunks back released si
        if (q >= 2) API_CHECK(h, cudaStreamWaitEvent(h->tier_in, h->ev_merged[b], 0));
        if (E1 > E0) {
            bE0 = E0 >> 6;
            bE1 = std::min(((E1 - 1) >> 6) + 2, nin_blk);
            API_CHECK(h, cudaMemcpyAsync(si, h->hdict + bE0, (bE1 - bE0) * sizeof(Blk),
                                         cudaMemcpyHostToDevice, h->tier_in));
        }
        API_CHECK(h, cudaEventRecord(h->ev_staged[b], h->tier_in));
        // merge once staged and once the write-back two chunks back released so
        API_CHECK(h, cudaStreamWaitEvent(h->stream, h->ev_staged[b], 0));
        if (q >= 2) API_CHECK(h, cudaStreamWaitEvent(h->stream, h->ev_written[b], 0));
        API_CHECK(h, launch_insert_range(h->prof, h->stream, make_dict(si - bE0), n_in, pos, gw,
                                         bint, n_suf, so - (sa << (kSbShift - 6)), tot, sb_start,
                                         sa, sbe));
        API_CHECK(h, cudaEventRecord(h->ev_merged[b], h->stream));
        // write back
        const uint64_t b0 = sa << (kSbShift - 6), b1 = std::min(sbe << (kSbShift - 6), nblk);
        API_CHECK(h, cudaStreamWaitEvent(h->tier_out, h->ev_merged[b], 0));
        API_CHECK(h, cudaMemcpyAsync(h->hdict + b0, so, (b1 - b0) * sizeof(Blk),
                                     cudaMemcpyDeviceToHost, h->tier_out));
        API_CHECK(h, cudaEventRecord(h->ev_written[b], h->tier_out));
    }
    // the main stream joins the write-backs (later kernels read the host dictionary)
    API_CHECK(h, cudaEventRecord(h->ev_start, h->tier_out));
    API_CHECK(h, cudaStreamWaitEvent(h->stream, h->ev_start, 0));
    API_CHECK(h, launch_sb_scan(h->prof, h->stream, tot, nsb, osb, m_new, (uint64_t*)h->d_C.p));
    return SETBWTE_OK;
}

// Output buffers of one Insert of n_ins symbols (HBM or host tier).
struct InsertBufs {
    Blk* ob = nullptr;
    uint64_t *osb = nullptr, *tot = nullptr, *sb_start = nullptr;
    uint64_t nsb = 0;
};

setbwte_status insert_prepare(setbwte_t h, uint64_t n_ins, InsertBufs* ib) {
    const uint64_t n_out = h->n + n_ins;
    const uint64_t nblk = (n_out >> 6) + 1;
    ib->nsb = (n_out >> kSbShift) + 1;
    const int nxt = 1 - h->cur;
    if (h->sigma == 5) {
        // the N plane: ping-pong like the Blks, per-superblock totals as scratch
        if (nblk * sizeof(Blk) > h->hbm_budget) return SETBWTE_E_UNSUPPORTED;  // no host tier
        NBlk* nb;
        uint64_t* ns;
        API_CHECK(h, ensure(h->nblk[nxt], nblk, &nb));
        API_CHECK(h, ensure(h->nsb[nxt], ib->nsb + 8, &ns));
        API_CHECK(h, ensure(h->ntot, ib->nsb + 8, &ns));
    }
    if (!h->host_tier && !h->sharded && nblk * sizeof(Blk) > h->hbm_budget) {
        // the dictionary outgrows its HBM budget: move B_ext to the host tier
        // (after this block's ComputeRanks, which still reads the HBM copy)
        setbwte_status st2 = host_reserve(h, nblk, cur_blk(h), true, h->n ? (h->n >> 6) + 1 : 0);
        if (st2 != SETBWTE_OK) return st2;
        h->host_tier = true;
        free_buf(h->blk[0]);
        free_buf(h->blk[1]);
    }
    if (!h->host_tier && !h->sharded) API_CHECK(h, ensure(h->blk[nxt], nblk, &ib->ob));
    API_CHECK(h, ensure(h->sb[nxt], ib->nsb * 4, &ib->osb));
    API_CHECK(h, ensure(h->sb_tot, ib->nsb * 5 + 8, &ib->tot));  // totals + sb_start
    ib->sb_start = ib->tot + 4 * (ib->nsb + 1);
    return SETBWTE_OK;
}

// B_ext := Insert(B_int, g_sa, B_ext) with pos / B_int / sb_start ready.
setbwte_status insert_finish(setbwte_t h, const InsertBufs& ib, const void* pos, int gw,
                             const uint8_t* bint, uint64_t n_ins, uint64_t m_add) {
    const uint64_t m_new = h->m + m_add;
    if (h->host_tier) {
        setbwte_status st = host_insert(h, pos, gw, bint, n_ins, ib.osb, ib.tot, ib.sb_start, m_new);
        if (st != SETBWTE_OK) return st;
    } else if (h->sharded) {
        // NEXT-3: rank r merges output superblocks [nsb*r/P, nsb*(r+1)/P) into
        // its own new shard (reading the old B_ext from every shard); only the
        // superblock totals and the shard pointers are exchanged -- no rank
        // holds the whole dictionary
        const uint64_t n_out = h->n + n_ins;
        const uint64_t nblk = (n_out >> 6) + 1;
        const uint64_t P = (uint64_t)h->world;
        std::vector<uint64_t> tot_bytes(P);
        for (uint64_t r = 0; r < P; ++r)
            tot_bytes[r] = (ib.nsb * (r + 1) / P - ib.nsb * r / P) * 4 * sizeof(uint64_t);
        const uint64_t a = ib.nsb * h->rank / P, b = ib.nsb * (h->rank + 1) / P;
        const uint64_t fb = std::min(a * kBlkPerSb, nblk);
        const uint64_t own = std::min(b * kBlkPerSb, nblk) - fb;
        Blk* shard;
        {
            // grow without freeing: with CUDA IPC, peers may still map the old
            // allocation (freed at destroy), and a freed-and-reused range
            // cannot be re-imported while mapped
            DevBuf& sbuf = h->shard_buf[1 - h->shard_cur];
            const size_t need = (own + 8) * sizeof(Blk);
            if (sbuf.cap < need) {
                if (sbuf.p) h->shard_retired.push_back(sbuf.p);
                sbuf.p = nullptr;
                sbuf.cap = 0;
                const size_t cap = need + need / 2;
                API_CHECK(h, cudaMalloc(&sbuf.p, cap));
                sbuf.cap = cap;
            }
            shard = static_cast<Blk*>(sbuf.p);
        }
        API_CHECK(h, launch_insert_range(h->prof, h->stream, cur_dict(h), h->n, pos, gw, bint, n_ins,
                                         shard - a * kBlkPerSb, ib.tot, ib.sb_start, a, b));
        // every rank's (first Blk, shard address): a device pointer when the
        // ranks share an address space (shard_dict = 1), a CUDA IPC handle of
        // the shard allocation when they are separate processes (= 2)
        struct ShardEntry {
            uint64_t first, ptr;
            cudaIpcMemHandle_t ipc;
        };
        ShardEntry* d_ent;
        API_CHECK(h, ensure(h->shard_ptrs, P + 1, &d_ent));
        ShardEntry mine{};
        mine.first = fb;
        mine.ptr = (uint64_t)(uintptr_t)shard;
        if (h->shard_ipc) API_CHECK(h, cudaIpcGetMemHandle(&mine.ipc, shard));
        API_CHECK(h, cudaMemcpyAsync(d_ent + h->rank, &mine, sizeof(mine), cudaMemcpyHostToDevice,
                                     h->stream));
        std::vector<uint64_t> ent_bytes(P, sizeof(ShardEntry));
        setbwte_status xs = exchange(h, ib.tot, tot_bytes.data());
        if (xs == SETBWTE_OK) xs = exchange(h, d_ent, ent_bytes.data());
        if (xs != SETBWTE_OK) return xs;
        API_CHECK(h, launch_sb_scan(h->prof, h->stream, ib.tot, ib.nsb, ib.osb, m_new,
                                    (uint64_t*)h->d_C.p));
        std::vector<ShardEntry> all(P);
        API_CHECK(h, cudaMemcpyAsync(all.data(), d_ent, sizeof(ShardEntry) * P,
                                     cudaMemcpyDeviceToHost, h->stream));
        API_CHECK(h, cudaStreamSynchronize(h->stream));
        Dict d = make_dict(nullptr);
        d.P = (int)P;
        for (uint64_t r = 0; r < P; ++r) {
            d.first[r] = all[r].first;
            const Blk* ptr = reinterpret_cast<const Blk*>((uintptr_t)all[r].ptr);
            if (h->shard_ipc && (int)r != h->rank) {
                // open each peer allocation once, keyed by its address in the
                // peer (allocations are never freed before destroy)
                auto& cache = h->ipc_open[r];
                void* opened = nullptr;
                for (auto& kv : cache)
                    if (kv.first == all[r].ptr) opened = kv.second;
                if (!opened) {
                    API_CHECK(h, cudaIpcOpenMemHandle(&opened, all[r].ipc,
                                                      cudaIpcMemLazyEnablePeerAccess));
                    cache.push_back({all[r].ptr, opened});
                }
                ptr = reinterpret_cast<const Blk*>(opened);
            }
            d.ptr[r] = ptr;
        }
        h->shard_dict = d;
        h->shard_cur = 1 - h->shard_cur;
    } else if (partitioned(h) && h->insert_split && (h->allgather || h->nccl) && h->sigma != 5) {
        // Insert split by output range: rank r merges output
        // superblocks [nsb*r/P, nsb*(r+1)/P) only; the new dictionary's Blks and
        // the superblock totals are then all-gathered (slices in rank order),
        // and every rank scans the totals itself.
        const uint64_t n_out = h->n + n_ins;
        const uint64_t nblk = (n_out >> 6) + 1;
        const uint64_t P = (uint64_t)h->world;
        std::vector<uint64_t> blk_bytes(P), tot_bytes(P);
        for (uint64_t r = 0; r < P; ++r) {
            const uint64_t a = ib.nsb * r / P, b = ib.nsb * (r + 1) / P;
            const uint64_t ba = std::min(a * kBlkPerSb, nblk), bb = std::min(b * kBlkPerSb, nblk);
            blk_bytes[r] = (bb - ba) * sizeof(Blk);
            tot_bytes[r] = (b - a) * 4 * sizeof(uint64_t);
        }
        const uint64_t a = ib.nsb * h->rank / P, b = ib.nsb * (h->rank + 1) / P;
        API_CHECK(h, launch_insert_range(h->prof, h->stream, cur_dict(h), h->n, pos, gw, bint, n_ins,
                                         ib.ob, ib.tot, ib.sb_start, a, b));
        setbwte_status xs = exchange(h, ib.ob, blk_bytes.data());
        if (xs == SETBWTE_OK) xs = exchange(h, ib.tot, tot_bytes.data());
        if (xs != SETBWTE_OK) return xs;
        API_CHECK(h, launch_sb_scan(h->prof, h->stream, ib.tot, ib.nsb, ib.osb, m_new,
                                    (uint64_t*)h->d_C.p));
    } else {
        N5Ins n5;
        if (h->sigma == 5) {
            const int nxt = 1 - h->cur;
            n5.in = (const NBlk*)h->nblk[h->cur].p;
            n5.out = (NBlk*)h->nblk[nxt].p;
            n5.ntot = (uint64_t*)h->ntot.p;
            n5.nsb_out = (uint64_t*)h->nsb[nxt].p;
        }
        API_CHECK(h, launch_insert(h->prof, h->stream, cur_dict(h), h->n, pos, gw, bint, n_ins, ib.ob,
                                   ib.osb, ib.tot, ib.sb_start, m_new, (uint64_t*)h->d_C.p,
                                   h->sigma == 5 ? &n5 : nullptr));
    }
    h->cur = 1 - h->cur;
    h->n += n_ins;
    h->m = m_new;
    return SETBWTE_OK;
}

// ComputeRanks, B_int + g_sa gather, Insert; on the main stream.
setbwte_status rank_insert_stage(setbwte_t h, const Packed& pk, const BlockDesc& b,
                                 const uint32_t* saf) {
    const uint64_t n_suf = b.S1 - b.S0;
    // g / pos width: u32 while every position of the new B_ext fits
    const int gw = (h->n + n_suf) < (1ull << 32) && h->g_width != 8 ? 4 : 8;
    uint64_t* g = (uint64_t*)h->g.p;
    uint64_t* pos = (uint64_t*)h->pos.p;
    uint8_t* bint = (uint8_t*)h->bint.p;
    // blocks too large for the SA payload: ComputeRanks records B_int per
    // slot (single-rank ComputeRanks over a non-empty index only)
    // (with u64 g, B_int goes into g's top byte instead: bing)
    uint8_t* bslot = nullptr;
    bool bing = false;
    if (!sa_payload(n_suf, h->sopt.payload_limit) && h->n != 0 && !partitioned(h)) {
        if (gw == 8) bing = true;
        else API_CHECK(h, ensure(h->bslot, n_suf + 8, &bslot));
    }
    // g := ComputeRanks(S_jk, B_ext)
    const uint64_t* slices =
        partitioned(h) ? h->blk_slices.data() + b.id * 2 * (uint64_t)(h->world + 1) : nullptr;
    setbwte_status st =
        compute_ranks_for(h, pk, b.j0, b.j1, b.S0, n_suf, g, gw, bslot, bing, slices);
    if (st != SETBWTE_OK) return st;
    InsertBufs ib;
    st = insert_prepare(h, n_suf, &ib);
    if (st != SETBWTE_OK) return st;
    // B_int := B(S_jk, SA_int), g_sa / pos and the superblock
    // slices of pos, fused
    const uint32_t gshift = gather_buckets_shift((uint32_t)n_suf, gw, h->gather_mode);
    if (gshift) {
        // g larger than L2: the bucketed gather (gather.cu)
        uint8_t* gt;
        API_CHECK(h, ensure(h->gtmp, gather_scratch_bytes((uint32_t)n_suf, gw), &gt));
        GatherScratch ws;
        ws.slot = reinterpret_cast<uint32_t*>(gt);
        ws.gval = gt + ((4 * n_suf + 255) & ~255ull);
        ws.rows = reinterpret_cast<uint32_t*>(gt + ((4 * n_suf + 255) & ~255ull) +
                                              ((gw * n_suf + 255) & ~255ull));
        API_CHECK(h, launch_gather_bucketed(h->prof, h->stream, pk.text, pk.term, b.S0, saf, g,
                                            (uint32_t)n_suf, pos, gw, bint, ib.sb_start, ib.nsb,
                                            bslot, h->sopt.payload_limit, bing, pk.nbit, gshift,
                                            ws));
    } else {
        API_CHECK(h, launch_gather(h->prof, h->stream, pk.text, pk.term, b.S0, saf, g,
                                   (uint32_t)n_suf, pos, gw, bint, ib.sb_start, ib.nsb, bslot,
                                   h->sopt.payload_limit, bing, pk.nbit));
    }
    return insert_finish(h, ib, pos, gw, bint, n_suf, b.j1 - b.j0);
}

void build_stats(setbwte_t h);

// BWT merge (NEXT-4): h := h followed by the strings of o, from o's BWT alone.
setbwte_status merge_impl(setbwte_t h, setbwte_t o) {
    h->prof.reset();
    h->sstats = SortStats();
    h->last_blocks = o->n ? 1 : 0;
    h->last_bases = o->n - o->m;
    h->last_m = o->m;
    if (o->n == 0) {
        build_stats(h);
        return SETBWTE_OK;
    }
    API_CHECK(h, cudaStreamSynchronize(o->stream));
    const uint64_t n_o = o->n;
    const int gw = (h->n + n_o) < (1ull << 32) && h->g_width != 8 ? 4 : 8;
    uint64_t *g, *pos;
    uint8_t* bint;
    API_CHECK(h, ensure(h->g, n_o, &g));
    API_CHECK(h, ensure(h->pos, n_o, &pos));
    API_CHECK(h, ensure(h->bint, n_o, &bint));
    API_CHECK(h, launch_merge_ranks(h->prof, h->stream, cur_blk(o), cur_sb(o),
                                    (const uint64_t*)o->d_C.p, o->m, n_o,
                                    h->n ? cur_blk(h) : nullptr, h->n ? cur_sb(h) : nullptr,
                                    (const uint64_t*)h->d_C.p, h->m, g, gw));
    InsertBufs ib;
    setbwte_status st = insert_prepare(h, n_o, &ib);
    if (st != SETBWTE_OK) return st;
    API_CHECK(h, launch_merge_pos(h->prof, h->stream, cur_blk(o), n_o, g, pos, gw, bint,
                                  ib.sb_start, ib.nsb));
    st = insert_finish(h, ib, pos, gw, bint, n_o, o->m);
    if (st != SETBWTE_OK) return st;
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    API_CHECK(h, h->prof.resolve());
    build_stats(h);
    return SETBWTE_OK;
}

// sort_split (NEXT-1 across GPUs, C3): block k was sorted on rank k mod P
// only; its SA_int reaches every rank through the allgather callback (a
// one-contributor all-gather = a broadcast), queued on the main stream.
setbwte_status share_sa(setbwte_t h, const BlockDesc& b, size_t k, uint32_t* saf) {
    if (!h->sort_split || !partitioned(h)) return SETBWTE_OK;
    std::vector<uint64_t> bytes(h->world, 0);
    bytes[k % (size_t)h->world] = 4 * (b.S1 - b.S0);
    // the slices are laid out in rank order: the owner's starts at offset 0
    // only if every earlier rank contributes 0 bytes, which holds here
    return exchange(h, saf, bytes.data());
}

// Run Algorithm 1 over all blocks with the two-stage pipeline.
// Run Algorithm 1 over all blocks.  ConstructSA has no B_ext dependency, so
// two host threads ("sort lanes", one CUDA stream each) sort blocks k+1 and
// k+2 ahead while the calling thread runs ComputeRanks / gather / Insert of
// block k on the main stream in block order.  The sort's round trips to the
// host (segment counts) are then hidden behind the other lanes' kernels.
struct SortLane {
    cudaStream_t stream = nullptr;
    SortScratch* ws = nullptr;
    Profiler prof;
    SortStats st;
    uint32_t* saf = nullptr;
    cudaEvent_t ev_sorted = nullptr;
};

// An append failed after some of its blocks were inserted.  On an index the
// append started empty there is nothing to roll back to but the empty index:
// reset it (unless a sticky CUDA error already failed the handle); otherwise
// the handle is failed.  Either way the recorded sort launch pattern is
// dropped (it may come from the failed call's blocks).
void fail_partial(setbwte_t h) {
    h->sort_pattern.drop();
    if (h->started_empty && !h->failed) {
        if (cudaStreamSynchronize(h->stream) == cudaSuccess &&
            cudaMemsetAsync(h->d_C.p, 0, 8 * sizeof(uint64_t), h->stream) == cudaSuccess &&
            cudaStreamSynchronize(h->stream) == cudaSuccess) {
            h->n = 0;
            h->m = 0;
            h->cur = 0;
            return;
        }
        cudaGetLastError();
    }
    h->failed = true;
}

// Sort lanes of an append whose largest block has max_suf suffixes: the
// option's value, or automatically 3 for blocks below 2^26 suffixes and 2
// from there (measured, alternated runs: c2's 2^24-suffix blocks 6.25 vs
// 6.64 ms per step with 3 vs 2 lanes; c3's 2^27 185.1 vs 186.0 ms and c4's
// 2^30 795 vs 871 ms with 2 vs 3 -- three large sorts at once contend more
// than they overlap).
int lanes_for(setbwte_t h, uint64_t max_suf) {
    if (h->sort_lanes >= 0) return h->sort_lanes;
    return max_suf >= (1ull << 26) ? 2 : 3;
}

// validate(): called on the main thread before the first Insert (the index is
// untouched until then); a non-OK status aborts the append.
setbwte_status run_blocks(setbwte_t h, const Packed& pk, const std::vector<BlockDesc>& blocks,
                          const std::function<setbwte_status()>& validate) {
    const size_t K = blocks.size();
    if (K == 0) return SETBWTE_OK;
    uint64_t max_suf = 0, total = 0;
    for (const BlockDesc& b : blocks) {
        max_suf = std::max(max_suf, b.S1 - b.S0);
        total += b.S1 - b.S0;
    }
    int NL = std::max(1, std::min<int>({lanes_for(h, max_suf), (int)K, setbwte_s::kMaxLanes}));
    if (NL > 1 && (max_suf > h->lanes_checked_suf || NL > h->lanes_checked_nl)) {
        // each lane owns a sort scratch (~30 B per suffix of the largest
        // block): keep the lanes within half of the free device memory.
        // Queried only when the scratch may grow: cudaMemGetInfo measured
        // up to 10 ms while other streams of the process are busy.
        size_t free_b = 0, total_b = 0;
        TraceScope tr(TR_MEMINFO);
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            const double per_lane = 30.0 * (double)max_suf;
            while (NL > 1 && per_lane * NL > 0.5 * (double)free_b) --NL;
        }
        h->lanes_checked_suf = max_suf;
        h->lanes_checked_nl = NL;
    } else if (NL > 1) {
        NL = std::min(NL, h->lanes_checked_nl);
    }
    // reserve everything up front: a cudaFree/cudaMalloc mid-loop would
    // serialise the streams
    uint32_t* saf2;
    uint64_t* tmp;
    uint8_t* tb;
    API_CHECK(h, ensure(h->saf, (size_t)NL * (max_suf + 32) + 64, &saf2));  // one SA_int per lane
    API_CHECK(h, ensure(h->g, max_suf, &tmp));
    API_CHECK(h, ensure(h->pos, max_suf, &tmp));
    API_CHECK(h, ensure(h->bint, max_suf, &tb));
    for (int l = 0; l < NL; ++l) API_CHECK(h, sort_reserve(h->sort[l], (uint32_t)max_suf, h->sopt));
    const uint64_t n_final = h->n + total;
    API_CHECK(h, ensure(h->sb_tot, ((n_final >> kSbShift) + 1) * 5 + 8, &tmp));
    SortLane lanes[setbwte_s::kMaxLanes];
    for (int l = 0; l < NL; ++l) {
        lanes[l].stream = h->sort_lanes == 0 ? h->stream : h->lane_stream[l];
        lanes[l].ws = &h->sort[l];
        lanes[l].saf = saf2 + l * (max_suf + 32);
        lanes[l].ev_sorted = h->ev_sorted[l];
        lanes[l].prof.on = h->prof.on;
        lanes[l].prof.only = h->prof.only;
        lanes[l].prof.tl = h->prof.tl;
        lanes[l].prof.ref = h->prof.ref;
    }
    if (h->sort_lanes == 0) {
        // no pipelining: every stage of every block in order on the calling
        // thread and the main stream (what per-launch profiling needs: no
        // other thread can enqueue between a launch and its events)
        for (size_t k = 0; k < K; ++k) {
            API_CHECK(h, cudaStreamWaitEvent(h->stream, h->ev_packed[blocks[k].ev], 0));
            if (k == 0) {
                setbwte_status st0 = validate();
                if (st0 != SETBWTE_OK) return st0;
            }
            if (!h->sort_split || (int)(k % (size_t)h->world) == h->rank)
                API_CHECK(h, sort_block(h->prof, h->stream, h->sort[0], pk.text, pk.term,
                                        blocks[k].S0, (uint32_t)(blocks[k].S1 - blocks[k].S0),
                                        saf2, &h->sstats, false, h->sopt, pk.nbit));
            setbwte_status st1 = share_sa(h, blocks[k], k, saf2);
            if (st1 == SETBWTE_OK) st1 = rank_insert_stage(h, pk, blocks[k], saf2);
            if (st1 != SETBWTE_OK) {
                if (k > 0) fail_partial(h);
                return st1;
            }
        }
        return SETBWTE_OK;
    }
    // the sort lanes start after everything queued on the main stream so far
    API_CHECK(h, cudaEventRecord(h->ev_start, h->stream));
    for (int l = 0; l < NL; ++l) API_CHECK(h, cudaStreamWaitEvent(lanes[l].stream, h->ev_start, 0));

    std::mutex mu;
    std::condition_variable cv;
    std::vector<char> sorted(K, 0), used(K, 0);
    cudaError_t lane_err = cudaSuccess;
    bool abort = false;
    auto lane_main = [&](int l) {
        SortLane& L = lanes[l];
        cudaError_t e = cudaSetDevice(h->device);
        for (size_t k = l; k < K && e == cudaSuccess; k += NL) {
            // this block's slots and the group straddling into the next block
            e = cudaStreamWaitEvent(L.stream, h->ev_packed[blocks[k].ev], 0);
            if (e != cudaSuccess) break;
            if (k >= (size_t)NL) {
                // SA_int buffer of this lane is free once block k-NL's gather ran
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return used[k - NL] || abort; });
                if (abort) break;
                lk.unlock();
                e = cudaStreamWaitEvent(L.stream, h->ev_used[l], 0);
                if (e != cudaSuccess) break;
            }
            // sort_split: rank (k mod P) sorts block k; the others receive its SA_int
            const bool mine = !h->sort_split || (int)(k % (size_t)h->world) == h->rank;
            if (mine)
                e = sort_block(L.prof, L.stream, *L.ws, pk.text, pk.term, blocks[k].S0,
                               (uint32_t)(blocks[k].S1 - blocks[k].S0), L.saf, &L.st, false,
                               h->sopt, pk.nbit);
            if (e == cudaSuccess) e = cudaEventRecord(L.ev_sorted, L.stream);
            std::lock_guard<std::mutex> lk(mu);
            if (e != cudaSuccess) {
                lane_err = e;
                abort = true;
            } else {
                sorted[k] = 1;
            }
            cv.notify_all();
        }
    };
    std::vector<std::thread> threads;
    for (int l = 0; l < NL; ++l) threads.emplace_back(lane_main, l);

    setbwte_status st;
    {
        TraceScope tr(TR_VALIDATE);
        st = validate();
    }
    if (st != SETBWTE_OK) {
        std::lock_guard<std::mutex> lk(mu);
        abort = true;
        cv.notify_all();
    }
    for (size_t k = 0; k < K && st == SETBWTE_OK; ++k) {
        {
            TraceScope tr(TR_RANK_WAIT);
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return sorted[k] || abort; });
            if (abort) break;
        }
        const int l = (int)(k % NL);
        cudaError_t e = cudaStreamWaitEvent(h->stream, lanes[l].ev_sorted, 0);
        if (e != cudaSuccess) {
            st = from_cuda(h, e);
        } else {
            st = share_sa(h, blocks[k], k, lanes[l].saf);
            if (st == SETBWTE_OK) st = rank_insert_stage(h, pk, blocks[k], lanes[l].saf);
            if (st == SETBWTE_OK) {
                e = cudaEventRecord(h->ev_used[l], h->stream);
                if (e != cudaSuccess) st = from_cuda(h, e);
            }
        }
        std::lock_guard<std::mutex> lk(mu);
        if (st != SETBWTE_OK) {
            if (k > 0) fail_partial(h);  // a partially applied append cannot be rolled back
            abort = true;
            cv.notify_all();
            break;
        }
        used[k] = 1;
        cv.notify_all();
    }
    {
        TraceScope tr(TR_LANE_JOIN);
        for (std::thread& t : threads) t.join();
    }
    if (st == SETBWTE_OK && lane_err != cudaSuccess) {
        st = from_cuda(h, lane_err);
        if (h->n != 0) fail_partial(h);
    }
    // the main stream joins the sort lanes; their statistics merge into the handle's
    for (int l = 0; l < NL; ++l) {
        API_CHECK(h, cudaEventRecord(h->ev_start, lanes[l].stream));
        API_CHECK(h, cudaStreamWaitEvent(h->stream, h->ev_start, 0));
        API_CHECK(h, cudaStreamSynchronize(lanes[l].stream));
        API_CHECK(h, lanes[l].prof.resolve());
        for (auto& kv : lanes[l].prof.k) {
            KStat& d = h->prof.k[kv.first];
            d.launches += kv.second.launches;
            d.ms += kv.second.ms;
            d.bytes += kv.second.bytes;
            d.units += kv.second.units;
        }
        h->prof.total_launches += lanes[l].prof.total_launches;
        h->prof.timeline.insert(h->prof.timeline.end(), lanes[l].prof.timeline.begin(),
                                lanes[l].prof.timeline.end());
        h->sstats.digit_passes += lanes[l].st.digit_passes;
        h->sstats.rounds += lanes[l].st.rounds;
        h->sstats.replayed += lanes[l].st.replayed;
        h->sstats.after_replay += lanes[l].st.after_replay;
        h->sstats.active_per_pass.insert(h->sstats.active_per_pass.end(),
                                         lanes[l].st.active_per_pass.begin(),
                                         lanes[l].st.active_per_pass.end());
    }
    return st;
}

void build_stats(setbwte_t h) {
    std::string s = "{";
    char buf[512];
    snprintf(buf, sizeof(buf),
             "\"n\": %llu, \"m\": %llu, \"blocks\": %llu, \"bases\": %llu, \"strings\": %llu, "
             "\"launches\": %llu, \"profile\": %d, \"block_suffixes\": %llu, "
             "\"host_tier\": %d, \"host_dict_bytes\": %llu, ",
             (unsigned long long)h->n, (unsigned long long)h->m,
             (unsigned long long)h->last_blocks, (unsigned long long)h->last_bases,
             (unsigned long long)h->last_m, (unsigned long long)h->prof.total_launches,
             h->prof.on ? 1 : 0, (unsigned long long)h->M, h->host_tier ? 1 : 0,
             (unsigned long long)(h->hdict_cap * sizeof(Blk)));
    s += buf;
    s += "\"sort\": {\"digit_passes\": " + std::to_string(h->sstats.digit_passes) +
         ", \"replayed_blocks\": " + std::to_string(h->sstats.replayed) +
         ", \"rounds_after_replay\": " + std::to_string(h->sstats.after_replay) +
         ", \"active_per_pass\": [";
    for (size_t i = 0; i < h->sstats.active_per_pass.size(); ++i) {
        if (i) s += ", ";
        s += std::to_string(h->sstats.active_per_pass[i]);
    }
    s += "]}, \"kernels\": {";
    bool first = true;
    for (auto& kv : h->prof.k) {
        if (!first) s += ", ";
        first = false;
        snprintf(buf, sizeof(buf),
                 "\"%s\": {\"launches\": %llu, \"ms\": %.6f, \"bytes\": %.1f, \"units\": %llu}",
                 kv.first.c_str(), (unsigned long long)kv.second.launches, kv.second.ms,
                 kv.second.bytes, (unsigned long long)kv.second.units);
        s += buf;
    }
    s += "}";
    if (h->prof.tl) {
        // mode 3: [kernel, stream, start ms, end ms] per launch, from the append's start
        s += ", \"timeline\": [";
        for (size_t i = 0; i < h->prof.timeline.size(); ++i) {
            const Profiler::TL& t = h->prof.timeline[i];
            snprintf(buf, sizeof(buf), "%s[\"%s\", %llu, %.4f, %.4f]", i ? ", " : "",
                     t.name.c_str(), (unsigned long long)t.stream, t.t0, t.t1);
            s += buf;
        }
        s += "]";
    }
    s += "}";
    h->stats_json = s;
}

// One append (Algorithm 1 over its blocks).  Host input (host_bytes != NULL):
// the bytes travel in chunks on the H2D stream and each block is packed
// as soon as its bytes are on the device, so sorting starts while later blocks
// are still in flight; the whole input is validated before the first Insert
// (all-or-nothing).  Device input: d_bytes already holds everything.
setbwte_status append_impl(setbwte_t h, const uint8_t* host_bytes, const uint64_t* host_off,
                           const uint8_t* d_bytes, const uint64_t* d_off, uint64_t m,
                           uint64_t n_bytes, bool prepend = false) {
    h->prof.reset();
    if (h->prof.tl && h->prof.ref) API_CHECK(h, cudaEventRecord(h->prof.ref, h->stream));
    h->sstats = SortStats();
    h->last_blocks = 0;
    h->last_bases = 0;
    h->last_m = m;
    if (m == 0) {
        build_stats(h);
        return SETBWTE_OK;
    }
    if (m >= 0xFFFFFFFFull) return SETBWTE_E_UNSUPPORTED;  // u32 string ids in the packer
    if (n_bytes == ~0ull) {
        API_CHECK(h, cudaMemcpyAsync(&n_bytes, d_off + m, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                     h->stream));
        API_CHECK(h, cudaStreamSynchronize(h->stream));
    }
    const uint64_t n_slots = n_bytes + m;
    const uint64_t n_groups = (n_slots + 31) / 32;
    Packed pk;
    pk.n_slots = n_slots;
    API_CHECK(h, ensure(h->text, 2 * n_groups + 8, &pk.text));
    API_CHECK(h, ensure(h->term, n_groups + 8, &pk.term));
    if (h->sigma == 5) API_CHECK(h, ensure(h->nbit, n_groups + 8, &pk.nbit));
    API_CHECK(h, ensure(h->slot_off, m + 2, &pk.slot_off));
    API_CHECK(h, ensure(h->gfirst, n_groups + 2, &pk.gfirst));
    DevErr* derr;
    API_CHECK(h, ensure(h->err, 1, &derr));
    // host input: the bytes start travelling now, in chunks, while the
    // offsets are checked and the blocks partitioned (they do not depend on
    // either); each block's packing waits for the chunks covering it
    // chunks of n/32, between 16 and 64 MB: the first block starts after its
    // first chunk (~1 ms at PCIe speed) instead of after 1/8 of the input
    static const uint64_t max_chunk =
        getenv("SETBWTE_H2D_CHUNK_MB") ? (uint64_t)atoll(getenv("SETBWTE_H2D_CHUNK_MB")) << 20
                                       : 64ull << 20;
    const uint64_t chunk =
        std::max<uint64_t>(16ull << 20, std::min<uint64_t>(max_chunk, (n_bytes + 31) / 32));
    const uint64_t n_chunks = host_bytes && n_bytes ? (n_bytes + chunk - 1) / chunk : 0;
    if (n_chunks) {
        while (h->ev_chunk.size() < n_chunks) {
            cudaEvent_t ev;
            API_CHECK(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            h->ev_chunk.push_back(ev);
        }
        API_CHECK(h, cudaEventRecord(h->ev_start, h->stream));  // the buffer is free
        API_CHECK(h, cudaStreamWaitEvent(h->h2d_stream, h->ev_start, 0));
        for (uint64_t c = 0; c < n_chunks; ++c) {
            const uint64_t b0 = c * chunk, b1 = std::min(n_bytes, b0 + chunk);
            API_CHECK(h, cudaMemcpyAsync(const_cast<uint8_t*>(d_bytes) + b0, host_bytes + b0, b1 - b0,
                                         cudaMemcpyHostToDevice, h->h2d_stream));
            API_CHECK(h, cudaEventRecord(h->ev_chunk[c], h->h2d_stream));
        }
    }
    *h->derr_host = DevErr{~0ull, 0, 0};
    API_CHECK(h, cudaMemcpyAsync(derr, h->derr_host, sizeof(DevErr), cudaMemcpyHostToDevice,
                                 h->stream));
    API_CHECK(h, launch_pack_prepare(h->prof, h->stream, d_off, m, n_bytes, pk, &derr->bad_offsets));
    // partition into blocks of >= M suffixes
    uint64_t* d_bounds;
    API_CHECK(h, ensure(h->bounds, 2 * (m + 2) + 2, &d_bounds));
    uint64_t* d_k = d_bounds + 2 * (m + 2);
    API_CHECK(h, launch_partition(h->prof, h->stream, pk.slot_off, m, h->M, d_bounds, d_k));
    // one round trip for K, the CSR check and (usually all of) the bounds
    uint64_t K = 0;
    const uint64_t pre = std::min<uint64_t>(m + 1, 1024);  // bounds pairs read speculatively
    std::vector<uint64_t> bounds(2 * pre);
    API_CHECK(h, cudaMemcpyAsync(&K, d_k, sizeof(K), cudaMemcpyDeviceToHost, h->stream));
    API_CHECK(h, cudaMemcpyAsync(h->derr_host, derr, sizeof(DevErr), cudaMemcpyDeviceToHost,
                                 h->stream));
    API_CHECK(h, cudaMemcpyAsync(bounds.data(), d_bounds, sizeof(uint64_t) * 2 * pre,
                                 cudaMemcpyDeviceToHost, h->stream));
    {
        TraceScope tr(TR_APPEND_SYNC);
        API_CHECK(h, cudaStreamSynchronize(h->stream));
    }
    // an early return must not leave H2D copies reading the caller's buffer
    auto abort_with = [&](setbwte_status st) {
        cudaStreamSynchronize(h->h2d_stream);
        return st;
    };
    if (h->derr_host->bad_offsets) return abort_with(SETBWTE_E_INVALID_ARG);
    if (K + 1 > pre) {
        bounds.resize(2 * (K + 1));
        API_CHECK(h, cudaMemcpyAsync(bounds.data(), d_bounds, sizeof(uint64_t) * 2 * (K + 1),
                                     cudaMemcpyDeviceToHost, h->stream));
        API_CHECK(h, cudaStreamSynchronize(h->stream));
    }
    for (uint64_t b = 0; b < K; ++b) {
        if (bounds[2 * b + 3] - bounds[2 * b + 1] >= (1ull << 31))
            return abort_with(SETBWTE_E_UNSUPPORTED);
    }
    h->last_bases = n_bytes;
    h->last_blocks = K;
    std::vector<BlockDesc> blocks(K);
    for (uint64_t b = 0; b < K; ++b)
        blocks[b] = BlockDesc{bounds[2 * b], bounds[2 * b + 2], bounds[2 * b + 1], bounds[2 * b + 3],
                              std::min(b + 1, K - 1), b};
    if (partitioned(h)) {
        // every block's ComputeRanks partition across the ranks, computed on
        // the device and read back once here: the per-block exchange then
        // needs no host synchronisation
        const uint64_t per = 2 * (uint64_t)(h->world + 1);
        uint64_t* d_sl;
        API_CHECK(h, ensure(h->small, K * per + 8, &d_sl));
        API_CHECK(h, launch_slices_blocks(h->prof, h->stream, pk.slot_off, d_bounds, K, h->world,
                                          d_sl));
        h->blk_slices.resize(K * per);
        API_CHECK(h, cudaMemcpyAsync(h->blk_slices.data(), d_sl, K * per * sizeof(uint64_t),
                                     cudaMemcpyDeviceToHost, h->stream));
        API_CHECK(h, cudaStreamSynchronize(h->stream));
    }
    // packing, block by block on the pack ("copy") stream, each after its chunks;
    // with sort_lanes = 0 (no pipelining: the profiled step) on the main stream,
    // so every launch is timed alone
    cudaStream_t ps = h->sort_lanes == 0 ? h->stream : h->copy_stream;
    while (h->ev_packed.size() < K) {
        cudaEvent_t ev;
        API_CHECK(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        h->ev_packed.push_back(ev);
    }
    API_CHECK(h, cudaEventRecord(h->ev_start, h->stream));
    API_CHECK(h, cudaStreamWaitEvent(ps, h->ev_start, 0));
    uint64_t waited = 0;  // chunks the pack stream already waits for
    for (uint64_t k = 0; k < K; ++k) {
        if (n_chunks) {
            // the block's bytes, plus the staging window its last pack warp
            // reads beyond them (< 1104 bytes)
            const uint64_t last = std::min(n_bytes, host_off[blocks[k].j1] + 2048);
            const uint64_t need = std::min(n_chunks, (last + chunk - 1) / chunk);
            for (; waited < need; ++waited)
                API_CHECK(h, cudaStreamWaitEvent(ps, h->ev_chunk[waited], 0));
        }
        const uint64_t g0 = k == 0 ? 0 : blocks[k].S0 >> 5;
        const uint64_t g1 = k + 1 < K ? blocks[k + 1].S0 >> 5 : n_groups;
        API_CHECK(h, launch_pack_range(h->prof, ps, d_bytes, m, n_bytes,
                                       (const uint8_t*)h->d_code_of.p, pk, g0, g1, &derr->err_pos));
        API_CHECK(h, cudaEventRecord(h->ev_packed[k], ps));
    }
    API_CHECK(h, cudaMemcpyAsync(h->derr_host, derr, sizeof(DevErr), cudaMemcpyDeviceToHost,
                                 ps));
    auto validate = [&]() -> setbwte_status {
        cudaError_t e = cudaStreamSynchronize(ps);
        if (e != cudaSuccess) return from_cuda(h, e);
        const uint64_t ep = h->derr_host->err_pos;
        if (ep == ~0ull) return SETBWTE_OK;
        h->err_pos = ep;
        uint8_t byte = 0;
        if (host_bytes) {
            byte = host_bytes[ep];
        } else {
            e = cudaMemcpy(&byte, d_bytes + ep, 1, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return from_cuda(h, e);
        }
        h->err_byte = byte;
        return SETBWTE_E_INVALID_CHAR;
    };
    // reverse orientation: the last block first, each one prepended to the
    // index (its strings precede every string indexed so far)
    std::vector<BlockDesc> order(blocks);
    if (prepend) std::reverse(order.begin(), order.end());
    h->prepending = prepend;
    // An empty index has nothing to roll back: the first Insert need not wait
    // for the whole input to be on the device and validated (with host input,
    // the last chunk arrives ~2 ms into a c2 call).  A bad byte found at the
    // end empties the index again.
    const bool defer = h->n == 0 && !h->sharded && !h->host_tier;  // plain HBM index only
    h->started_empty = defer;
    setbwte_status st = run_blocks(h, pk, order,
                                   defer ? std::function<setbwte_status()>(
                                               []() { return SETBWTE_OK; })
                                         : std::function<setbwte_status()>(validate));
    h->prepending = false;
    h->started_empty = false;
    if (defer && st == SETBWTE_OK) {
        st = validate();
        if (st == SETBWTE_E_INVALID_CHAR) {
            h->sort_pattern.drop();
            API_CHECK(h, cudaStreamSynchronize(h->stream));
            h->n = 0;
            h->m = 0;
            h->cur = 0;
            API_CHECK(h, cudaMemset(h->d_C.p, 0, 8 * sizeof(uint64_t)));
        }
    }
    // the main stream joins the copy stream (the bytes buffer is reused later)
    API_CHECK(h, cudaEventRecord(h->ev_start, ps));
    API_CHECK(h, cudaStreamWaitEvent(h->stream, h->ev_start, 0));
    if (st != SETBWTE_OK) return st;
    {
        TraceScope tr(TR_FINAL_SYNC);
        API_CHECK(h, cudaStreamSynchronize(h->stream));
    }
    API_CHECK(h, h->prof.resolve());
    build_stats(h);
    return SETBWTE_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* setbwte_strerror(setbwte_status s) {
    switch (s) {
        case SETBWTE_OK: return "ok";
        case SETBWTE_E_INVALID_ARG: return "invalid argument";
        case SETBWTE_E_INVALID_CHAR: return "invalid character";
        case SETBWTE_E_OUT_OF_RANGE: return "position out of range";
        case SETBWTE_E_NOMEM: return "out of memory";
        case SETBWTE_E_CUDA: return "CUDA error";
        case SETBWTE_E_UNSUPPORTED: return "unsupported";
        case SETBWTE_E_STATE: return "handle in failed state";
        case SETBWTE_E_NCCL: return "NCCL unavailable or an NCCL call failed";
    }
    return "unknown status";
}

// Every growth buffer of the handle that may come from a user allocator.  The
// shard buffers do not: CUDA IPC (shard_dict = 2) needs cudaMalloc'd bases.
static std::vector<DevBuf*> pooled_bufs(setbwte_t h) {
    std::vector<DevBuf*> v = {&h->d_code_of, &h->d_sym, &h->blk[0], &h->blk[1], &h->sb[0],
                              &h->sb[1], &h->d_C, &h->sb_tot, &h->in_bytes, &h->in_off, &h->text,
                              &h->term, &h->gfirst, &h->slot_off, &h->bounds, &h->err, &h->small,
                              &h->saf, &h->g, &h->pos, &h->bslot, &h->bint, &h->outbuf, &h->gtmp,
                              &h->shard_ptrs, &h->stage_in, &h->stage_out, &h->nbit,
                              &h->nblk[0], &h->nblk[1], &h->nsb[0], &h->nsb[1], &h->ntot};
    for (SortScratch& ws : h->sort)
        for (DevBuf* b : ws.bufs()) v.push_back(b);
    return v;
}

setbwte_status setbwte_create(const char* alphabet, setbwte_t* out) {
    if (!alphabet || !out) return SETBWTE_E_INVALID_ARG;
    *out = nullptr;
    const size_t sigma = strlen(alphabet);
    if (sigma < 1) return SETBWTE_E_INVALID_ARG;
    if (sigma > 5) return SETBWTE_E_UNSUPPORTED;
    setbwte_t h = new (std::nothrow) setbwte_s();
    if (!h) return SETBWTE_E_NOMEM;
    memset(h->code_of, 0xFF, sizeof(h->code_of));
    for (size_t i = 0; i < sigma; ++i) {
        const unsigned char c = (unsigned char)alphabet[i];
        if (c == '$' || h->code_of[toupper(c)] != 0xFF || h->code_of[tolower(c)] != 0xFF) {
            delete h;
            return SETBWTE_E_INVALID_ARG;
        }
        h->code_of[toupper(c)] = (uint8_t)i;
        h->code_of[tolower(c)] = (uint8_t)i;
        h->alpha[i] = (char)c;
    }
    h->sigma = (int)sigma;
    cudaError_t e = cudaGetDevice(&h->device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking);
    // the sort lanes run at the highest stream priority: a launch on a lane
    // starts as soon as SM slots free up instead of queueing behind the
    // rank/insert stream (same throughput; per-launch event times then track
    // the kernels' own execution more closely)
    int prio_low = 0, prio_high = 0;
    if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high);
    for (int l = 0; l < setbwte_s::kMaxLanes; ++l)
        if (e == cudaSuccess)
            e = cudaStreamCreateWithPriority(&h->lane_stream[l], cudaStreamNonBlocking, prio_high);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->h2d_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->tier_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->tier_out, cudaStreamNonBlocking);
    for (int b = 0; b < 2; ++b) {
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_staged[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_merged[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_written[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaHostAlloc((void**)&h->derr_host, sizeof(DevErr), cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming);
    for (int l = 0; l < setbwte_s::kMaxLanes; ++l) {
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_sorted[l], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_used[l], cudaEventDisableTiming);
    }
    h->stream = h->own_stream;
    h->sopt.pattern = &h->sort_pattern;
    for (DevBuf* b : pooled_bufs(h)) b->owner = &h->user_alloc;
    uint8_t* dc = nullptr;
    uint8_t* ds = nullptr;
    uint64_t* dC = nullptr;
    if (e == cudaSuccess) e = ensure(h->d_code_of, 256, &dc);
    if (e == cudaSuccess) e = ensure(h->d_sym, 8, &ds);
    if (e == cudaSuccess) e = ensure(h->d_C, 8, &dC);
    uint8_t sym[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (size_t i = 0; i < sigma; ++i) sym[i] = (uint8_t)alphabet[i];
    if (e == cudaSuccess) e = cudaMemcpy(dc, h->code_of, 256, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(ds, sym, 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(dC, 0, 8 * sizeof(uint64_t));
    if (e != cudaSuccess) {
        cudaGetLastError();
        setbwte_destroy(h);
        return e == cudaErrorMemoryAllocation ? SETBWTE_E_NOMEM : SETBWTE_E_CUDA;
    }
    build_stats(h);
    *out = h;
    return SETBWTE_OK;
}

void setbwte_destroy(setbwte_t h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (auto& cache : h->ipc_open)
        for (auto& kv : cache) cudaIpcCloseMemHandle(kv.second);
    for (void* p : h->shard_retired) cudaFree(p);
    for (DevBuf* b : pooled_bufs(h)) free_buf(*b);
    free_buf(h->shard_buf[0]);
    free_buf(h->shard_buf[1]);
    if (h->tier_in) cudaStreamSynchronize(h->tier_in);
    if (h->tier_out) cudaStreamSynchronize(h->tier_out);
    host_dict_free(h);
    for (int b = 0; b < 2; ++b) {
        if (h->ev_staged[b]) cudaEventDestroy(h->ev_staged[b]);
        if (h->ev_merged[b]) cudaEventDestroy(h->ev_merged[b]);
        if (h->ev_written[b]) cudaEventDestroy(h->ev_written[b]);
    }
    if (h->tier_in) cudaStreamDestroy(h->tier_in);
    if (h->tier_out) cudaStreamDestroy(h->tier_out);
    for (cudaStream_t ls : h->lane_stream)
        if (ls) cudaStreamSynchronize(ls);
    if (h->ev_start) cudaEventDestroy(h->ev_start);
    for (int l = 0; l < setbwte_s::kMaxLanes; ++l) {
        if (h->ev_sorted[l]) cudaEventDestroy(h->ev_sorted[l]);
        if (h->ev_used[l]) cudaEventDestroy(h->ev_used[l]);
        if (h->lane_stream[l]) cudaStreamDestroy(h->lane_stream[l]);
    }
    if (h->h2d_stream) {
        cudaStreamSynchronize(h->h2d_stream);
        cudaStreamDestroy(h->h2d_stream);
    }
    for (cudaEvent_t ev : h->ev_chunk) cudaEventDestroy(ev);
    if (h->copy_stream) {
        cudaStreamSynchronize(h->copy_stream);
        cudaStreamDestroy(h->copy_stream);
    }
    for (cudaEvent_t ev : h->ev_packed) cudaEventDestroy(ev);
    if (h->prof.ref) cudaEventDestroy(h->prof.ref);
    if (h->derr_host) cudaFreeHost(h->derr_host);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    delete h;
}

static setbwte_status add_device(setbwte_t h, const uint8_t* d_strings, const uint64_t* d_offsets,
                                 uint64_t m, bool prepend) {
    API_ENTER(h);
    if (m > 0 && !d_offsets) return SETBWTE_E_INVALID_ARG;
    setbwte_status st;
    {
        TraceScope tr(TR_TOTAL);
        st = append_impl(h, nullptr, nullptr, d_strings, d_offsets, m, ~0ull, prepend);
    }
    trace_dump();
    return st;
}

static setbwte_status add_host(setbwte_t h, const uint8_t* strings, const uint64_t* offsets,
                               uint64_t m, bool prepend) {
    API_ENTER(h);
    if (m == 0) return append_impl(h, nullptr, nullptr, nullptr, nullptr, 0, 0, prepend);
    if (!offsets) return SETBWTE_E_INVALID_ARG;
    const uint64_t nb = offsets[m];
    if (nb > 0 && !strings) return SETBWTE_E_INVALID_ARG;
    // CSR validity is checked on the device before any byte is copied (the
    // copies index the host buffer by block boundaries only)
    if (offsets[0] != 0) return SETBWTE_E_INVALID_ARG;
    uint8_t* db;
    uint64_t* dof;
    API_CHECK(h, ensure(h->in_bytes, nb + 16, &db));
    API_CHECK(h, ensure(h->in_off, m + 1, &dof));
    API_CHECK(h, cudaMemcpyAsync(dof, offsets, (m + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                 h->stream));
    setbwte_status st;
    {
        TraceScope tr(TR_TOTAL);
        st = append_impl(h, strings, offsets, db, dof, m, nb, prepend);
    }
    trace_dump();
    return st;
}

setbwte_status setbwte_append_device(setbwte_t h, const uint8_t* d_strings,
                                     const uint64_t* d_offsets, uint64_t m) {
    return add_device(h, d_strings, d_offsets, m, false);
}

setbwte_status setbwte_append(setbwte_t h, const uint8_t* strings, const uint64_t* offsets,
                              uint64_t m) {
    return add_host(h, strings, offsets, m, false);
}

setbwte_status setbwte_prepend(setbwte_t h, const uint8_t* strings, const uint64_t* offsets,
                               uint64_t m) {
    return add_host(h, strings, offsets, m, true);
}

setbwte_status setbwte_prepend_device(setbwte_t h, const uint8_t* d_strings,
                                      const uint64_t* d_offsets, uint64_t m) {
    return add_device(h, d_strings, d_offsets, m, true);
}

setbwte_status setbwte_merge(setbwte_t h, setbwte_t other) {
    API_ENTER(h);
    if (!other || other == h) return SETBWTE_E_INVALID_ARG;
    if (other->failed) return SETBWTE_E_STATE;
    if (other->device != h->device || strcmp(other->alpha, h->alpha) != 0 || h->sharded ||
        other->sharded || h->sigma == 5)
        return SETBWTE_E_UNSUPPORTED;
    return merge_impl(h, other);
}

setbwte_status setbwte_clear(setbwte_t h) {
    API_ENTER(h);
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    h->n = 0;
    h->m = 0;
    h->cur = 0;
    API_CHECK(h, cudaMemset(h->d_C.p, 0, 8 * sizeof(uint64_t)));
    return SETBWTE_OK;
}

setbwte_status setbwte_size(setbwte_t h, uint64_t* n, uint64_t* m) {
    if (!h) return SETBWTE_E_INVALID_ARG;
    if (h->failed) return SETBWTE_E_STATE;
    if (n) *n = h->n;
    if (m) *m = h->m;
    return SETBWTE_OK;
}

static setbwte_status bwt_impl(setbwte_t h, uint8_t* out, uint64_t cap, uint64_t* n, bool dev) {
    API_ENTER(h);
    if (!n) return SETBWTE_E_INVALID_ARG;
    *n = h->n;
    if (!out) return SETBWTE_OK;
    if (cap < h->n) return SETBWTE_E_INVALID_ARG;
    if (h->n == 0) return SETBWTE_OK;
    uint8_t* target = out;
    if (!dev) API_CHECK(h, ensure(h->outbuf, h->n, &target));
    API_CHECK(h, launch_decode(h->prof, h->stream, cur_dict(h), h->n, (const uint8_t*)h->d_sym.p,
                               target, h->sigma == 5 ? (const NBlk*)h->nblk[h->cur].p : nullptr));
    if (!dev)
        API_CHECK(h, cudaMemcpyAsync(out, target, h->n, cudaMemcpyDeviceToHost, h->stream));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    return SETBWTE_OK;
}

setbwte_status setbwte_bwt(setbwte_t h, uint8_t* out, uint64_t cap, uint64_t* n) {
    return bwt_impl(h, out, cap, n, false);
}

setbwte_status setbwte_bwt_device(setbwte_t h, uint8_t* d_out, uint64_t cap, uint64_t* n) {
    return bwt_impl(h, d_out, cap, n, true);
}

setbwte_status setbwte_rank(setbwte_t h, uint8_t c, uint64_t k, uint64_t* out) {
    API_ENTER(h);
    if (!out) return SETBWTE_E_INVALID_ARG;
    if (c != '$' && h->code_of[c] == 0xFF) return SETBWTE_E_INVALID_ARG;
    if (k > h->n) return SETBWTE_E_OUT_OF_RANGE;
    if (h->n == 0) {
        *out = 0;
        return SETBWTE_OK;
    }
    uint64_t* d;
    API_CHECK(h, ensure(h->small, 8, &d));
    uint8_t* dc = reinterpret_cast<uint8_t*>(d + 2);
    API_CHECK(h, cudaMemcpyAsync(d, &k, 8, cudaMemcpyHostToDevice, h->stream));
    API_CHECK(h, cudaMemcpyAsync(dc, &c, 1, cudaMemcpyHostToDevice, h->stream));
    const N5Dict n5 = cur_n5(h);
    API_CHECK(h, launch_rank_batch(h->prof, h->stream, cur_dict(h), cur_sb(h), h->n,
                                   (const uint8_t*)h->d_code_of.p, dc, d, 1, d + 1,
                                   h->sigma == 5 ? &n5 : nullptr));
    uint64_t r = 0;
    API_CHECK(h, cudaMemcpyAsync(&r, d + 1, 8, cudaMemcpyDeviceToHost, h->stream));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    *out = r;
    return SETBWTE_OK;
}

setbwte_status setbwte_rank_batch(setbwte_t h, const uint8_t* c_dev, const uint64_t* k_dev,
                                  uint64_t q, uint64_t* out_dev) {
    API_ENTER(h);
    if (q == 0) return SETBWTE_OK;
    if (!c_dev || !k_dev || !out_dev) return SETBWTE_E_INVALID_ARG;
    if (h->n == 0) {
        // only k = 0 is in range: rank 0; others are out of range
        API_CHECK(h, cudaMemsetAsync(out_dev, 0xFF, q * sizeof(uint64_t), h->stream));
        // a zero-sized index has no dictionary; answer k=0 queries on the host path
        std::vector<uint64_t> k(q);
        API_CHECK(h, cudaMemcpyAsync(k.data(), k_dev, q * 8, cudaMemcpyDeviceToHost, h->stream));
        API_CHECK(h, cudaStreamSynchronize(h->stream));
        std::vector<uint8_t> c(q);
        API_CHECK(h, cudaMemcpy(c.data(), c_dev, q, cudaMemcpyDeviceToHost));
        std::vector<uint64_t> r(q);
        for (uint64_t i = 0; i < q; ++i)
            r[i] = (k[i] == 0 && (c[i] == '$' || h->code_of[c[i]] != 0xFF)) ? 0 : ~0ull;
        API_CHECK(h, cudaMemcpy(out_dev, r.data(), q * 8, cudaMemcpyHostToDevice));
        return SETBWTE_OK;
    }
    const N5Dict n5 = cur_n5(h);
    API_CHECK(h, launch_rank_batch(h->prof, h->stream, cur_dict(h), cur_sb(h), h->n,
                                   (const uint8_t*)h->d_code_of.p, c_dev, k_dev, q, out_dev,
                                   h->sigma == 5 ? &n5 : nullptr));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    return SETBWTE_OK;
}

static setbwte_status count_impl(setbwte_t h, const uint8_t* d_pat, const uint64_t* d_off,
                                 uint64_t q, uint64_t* d_out) {
    if (h->n == 0) {
        API_CHECK(h, cudaMemsetAsync(d_out, 0, q * sizeof(uint64_t), h->stream));
        return SETBWTE_OK;
    }
    const N5Dict n5 = cur_n5(h);
    API_CHECK(h, launch_count(h->prof, h->stream, cur_dict(h), cur_sb(h), h->n,
                              (const uint64_t*)h->d_C.p, (const uint8_t*)h->d_code_of.p, d_pat,
                              d_off, q, d_out, h->sigma == 5 ? &n5 : nullptr));
    return SETBWTE_OK;
}

setbwte_status setbwte_count(setbwte_t h, const uint8_t* patterns, const uint64_t* offsets,
                             uint64_t q, uint64_t* counts) {
    API_ENTER(h);
    if (q == 0) return SETBWTE_OK;
    if (!offsets || !counts || (offsets[q] > 0 && !patterns)) return SETBWTE_E_INVALID_ARG;
    const uint64_t nb = offsets[q];
    for (uint64_t t = 0; t < q; ++t)
        if (offsets[t] > offsets[t + 1]) return SETBWTE_E_INVALID_ARG;
    uint8_t* dp;
    uint64_t* dof;
    API_CHECK(h, ensure(h->in_bytes, nb + 16, &dp));
    API_CHECK(h, ensure(h->in_off, 2 * (q + 1), &dof));
    if (nb) API_CHECK(h, cudaMemcpyAsync(dp, patterns, nb, cudaMemcpyHostToDevice, h->stream));
    API_CHECK(h, cudaMemcpyAsync(dof, offsets, (q + 1) * 8, cudaMemcpyHostToDevice, h->stream));
    uint64_t* dout = dof + (q + 1);
    setbwte_status st = count_impl(h, dp, dof, q, dout);
    if (st != SETBWTE_OK) return st;
    API_CHECK(h, cudaMemcpyAsync(counts, dout, q * 8, cudaMemcpyDeviceToHost, h->stream));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    return SETBWTE_OK;
}

setbwte_status setbwte_count_device(setbwte_t h, const uint8_t* d_patterns,
                                    const uint64_t* d_offsets, uint64_t q, uint64_t* d_counts) {
    API_ENTER(h);
    if (q == 0) return SETBWTE_OK;
    if (!d_patterns || !d_offsets || !d_counts) return SETBWTE_E_INVALID_ARG;
    setbwte_status st = count_impl(h, d_patterns, d_offsets, q, d_counts);
    if (st != SETBWTE_OK) return st;
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    return SETBWTE_OK;
}

setbwte_status setbwte_construct_sa(setbwte_t h, const uint8_t* strings, const uint64_t* offsets,
                                    uint64_t m, uint32_t* sa_out, uint8_t* bint_out) {
    API_ENTER(h);
    if (m == 0) return SETBWTE_OK;
    if (!offsets || (offsets[m] > 0 && !strings)) return SETBWTE_E_INVALID_ARG;
    const uint64_t nb = offsets[m];
    const uint64_t n_suf = nb + m;
    if (n_suf >= (1ull << 31)) return SETBWTE_E_UNSUPPORTED;
    uint8_t* db;
    uint64_t* dof;
    API_CHECK(h, ensure(h->in_bytes, nb + 16, &db));
    API_CHECK(h, ensure(h->in_off, m + 1, &dof));
    if (nb) API_CHECK(h, cudaMemcpyAsync(db, strings, nb, cudaMemcpyHostToDevice, h->stream));
    API_CHECK(h, cudaMemcpyAsync(dof, offsets, (m + 1) * 8, cudaMemcpyHostToDevice, h->stream));
    PackOut po;
    setbwte_status st = pack_input(h, db, dof, m, &po);
    if (st != SETBWTE_OK) return st;
    uint32_t* saf;
    uint64_t* pos;
    uint8_t *bint, *asc;
    API_CHECK(h, ensure(h->saf, n_suf, &saf));
    API_CHECK(h, ensure(h->pos, n_suf, &pos));
    API_CHECK(h, ensure(h->bint, n_suf, &bint));
    API_CHECK(h, ensure(h->outbuf, n_suf, &asc));
    API_CHECK(h, sort_block(h->prof, h->stream, h->sort[0], po.pk.text, po.pk.term, 0,
                            (uint32_t)n_suf, saf, nullptr, false, h->sopt, po.pk.nbit));
    API_CHECK(h, launch_gather(h->prof, h->stream, po.pk.text, po.pk.term, 0, saf, nullptr,
                               (uint32_t)n_suf, pos, 8, bint, nullptr, 0, nullptr,
                               h->sopt.payload_limit, false, po.pk.nbit));
    API_CHECK(h, launch_bint_ascii(h->prof, h->stream, bint, (uint32_t)n_suf,
                                   (const uint8_t*)h->d_sym.p, asc));
    API_CHECK(h, launch_strip_payload(h->stream, saf, (uint32_t)n_suf, h->sopt.payload_limit));
    if (sa_out)
        API_CHECK(h, cudaMemcpyAsync(sa_out, saf, n_suf * 4, cudaMemcpyDeviceToHost, h->stream));
    if (bint_out)
        API_CHECK(h, cudaMemcpyAsync(bint_out, asc, n_suf, cudaMemcpyDeviceToHost, h->stream));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    return SETBWTE_OK;
}

setbwte_status setbwte_compute_ranks(setbwte_t h, const uint8_t* strings, const uint64_t* offsets,
                                     uint64_t m, uint64_t* g_out) {
    API_ENTER(h);
    if (m == 0) return SETBWTE_OK;
    if (!offsets || !g_out || (offsets[m] > 0 && !strings)) return SETBWTE_E_INVALID_ARG;
    const uint64_t nb = offsets[m];
    const uint64_t n_suf = nb + m;
    uint8_t* db;
    uint64_t* dof;
    API_CHECK(h, ensure(h->in_bytes, nb + 16, &db));
    API_CHECK(h, ensure(h->in_off, m + 1, &dof));
    if (nb) API_CHECK(h, cudaMemcpyAsync(db, strings, nb, cudaMemcpyHostToDevice, h->stream));
    API_CHECK(h, cudaMemcpyAsync(dof, offsets, (m + 1) * 8, cudaMemcpyHostToDevice, h->stream));
    h->prof.reset();  // setbwte_stats reports this call's kernels
    PackOut po;
    setbwte_status st = pack_input(h, db, dof, m, &po);
    if (st != SETBWTE_OK) return st;
    uint64_t* g;
    API_CHECK(h, ensure(h->g, n_suf, &g));
    st = compute_ranks_for(h, po.pk, 0, m, 0, n_suf, g, 8);
    if (st != SETBWTE_OK) return st;
    API_CHECK(h, cudaMemcpyAsync(g_out, g, n_suf * 8, cudaMemcpyDeviceToHost, h->stream));
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    API_CHECK(h, h->prof.resolve());
    build_stats(h);
    return SETBWTE_OK;
}

setbwte_status setbwte_set_option(setbwte_t h, const char* key, uint64_t value) {
    if (!h || !key) return SETBWTE_E_INVALID_ARG;
    if (h->failed) return SETBWTE_E_STATE;
    if (!strcmp(key, "block_suffixes")) {
        if (value < 1 || value > (1ull << 30)) return SETBWTE_E_INVALID_ARG;
        h->M = value;
    } else if (!strcmp(key, "profile")) {
        if (value > 1) return SETBWTE_E_INVALID_ARG;
        h->prof.on = value == 1;
        h->prof.only.clear();
    } else if (!strcmp(key, "host_tier")) {
        // 1: move B_ext's dictionary to pinned host memory now (and keep it there)
        if (value != 1) return SETBWTE_E_INVALID_ARG;
        if (h->sharded || h->sigma == 5) return SETBWTE_E_UNSUPPORTED;
        h->hbm_budget = 0;
        if (!h->host_tier) {
            cudaError_t e = cudaSetDevice(h->device);
            if (e != cudaSuccess) return from_cuda(h, e);
            const uint64_t nblk = (h->n >> 6) + 1;
            setbwte_status st = host_reserve(h, nblk, cur_blk(h), true, h->n ? nblk : 0);
            if (st != SETBWTE_OK) return st;
            h->host_tier = true;
            free_buf(h->blk[0]);
            free_buf(h->blk[1]);
        }
    } else if (!strcmp(key, "hbm_budget_bytes")) {
        if (value < 1) return SETBWTE_E_INVALID_ARG;
        h->hbm_budget = value;
    } else if (!strcmp(key, "g_width")) {
        if (value != 0 && value != 4 && value != 8) return SETBWTE_E_INVALID_ARG;
        h->g_width = (int)value;
    } else if (!strcmp(key, "sa_payload")) {
        if (value > 1) return SETBWTE_E_INVALID_ARG;
        h->sopt.payload_limit = value ? kPayloadLimit : 0;
    } else if (!strcmp(key, "shard_dict")) {
        // 1: ranks share one address space; 2: separate processes (CUDA IPC)
        if (value > 2) return SETBWTE_E_INVALID_ARG;
        // needs the partition (world > 1, P <= 8), an empty index and no host tier
        if (value && (h->world <= 1 || h->world > kMaxShards || h->host_tier || h->n != 0 ||
                      h->sigma == 5))
            return SETBWTE_E_UNSUPPORTED;
        h->sharded = value != 0;
        h->shard_ipc = value == 2;
    } else if (!strcmp(key, "sort_split")) {
        if (value > 1) return SETBWTE_E_INVALID_ARG;
        h->sort_split = value != 0;
    } else if (!strcmp(key, "insert_split")) {
        if (value > 1) return SETBWTE_E_INVALID_ARG;
        h->insert_split = value != 0;
    } else if (!strcmp(key, "sort_lanes")) {
        if (value == 255) {
            h->sort_lanes = -1;  // automatic (the default)
        } else {
            if (value > (uint64_t)setbwte_s::kMaxLanes) return SETBWTE_E_INVALID_ARG;
            h->sort_lanes = (int)value;
        }
    } else if (!strcmp(key, "gather_buckets")) {
        if (value > 2) return SETBWTE_E_INVALID_ARG;
        h->gather_mode = (int)value;
    } else if (!strcmp(key, "force_exchange")) {
        // test hook: run the partitioned ComputeRanks + exchange path even
        // with world == 1 (one slice; with a communicator, one NCCL broadcast)
        if (value > 1) return SETBWTE_E_INVALID_ARG;
        h->force_exchange = value != 0;
    } else {
        return SETBWTE_E_INVALID_ARG;
    }
    return SETBWTE_OK;
}

setbwte_status setbwte_set_profile(setbwte_t h, int mode, const char* kernel) {
    if (!h || mode < 0 || mode > 3 || (mode == 2 && !kernel)) return SETBWTE_E_INVALID_ARG;
    h->prof.on = mode != 0;
    h->prof.only = mode == 2 ? std::string(kernel) : std::string();
    h->prof.tl = mode == 3;
    if (h->prof.tl && !h->prof.ref) API_CHECK(h, cudaEventCreate(&h->prof.ref));
    return SETBWTE_OK;
}

setbwte_status setbwte_set_stream(setbwte_t h, void* cuda_stream) {
    API_ENTER(h);
    API_CHECK(h, cudaStreamSynchronize(h->stream));
    h->stream = cuda_stream ? (cudaStream_t)cuda_stream : h->own_stream;
    return SETBWTE_OK;
}

setbwte_status setbwte_set_partition(setbwte_t h, int rank, int world,
                                     setbwte_allgather_fn allgather, void* ctx) {
    if (!h) return SETBWTE_E_INVALID_ARG;
    if (world < 1 || world > 1023 || rank < 0 || rank >= world) return SETBWTE_E_INVALID_ARG;
    if (world > 1 && !allgather) return SETBWTE_E_INVALID_ARG;
    // a sharded dictionary is laid out for the partition it was created with
    if (h->sharded && (world != h->world || world < 2 || world > kMaxShards))
        return SETBWTE_E_UNSUPPORTED;
    h->rank = rank;
    h->world = world;
    h->allgather = allgather;
    h->allgather_ctx = ctx;
    h->nccl = nullptr;  // the callback replaces a communicator
    return SETBWTE_OK;
}

setbwte_status setbwte_set_comm(setbwte_t h, void* nccl_comm, int rank, int world) {
    if (!h) return SETBWTE_E_INVALID_ARG;
    if (h->failed) return SETBWTE_E_STATE;
    if (!nccl_comm) {
        // detach: back to a single rank (or to the callback, if one is set)
        h->nccl = nullptr;
        if (!h->allgather) {
            if (h->sharded) return SETBWTE_E_UNSUPPORTED;
            h->rank = 0;
            h->world = 1;
        }
        return SETBWTE_OK;
    }
    if (world < 1 || world > 1023 || rank < 0 || rank >= world) return SETBWTE_E_INVALID_ARG;
    if (h->sharded && (world != h->world || world < 2 || world > kMaxShards))
        return SETBWTE_E_UNSUPPORTED;
    const NcclApi& nc = nccl_api();
    if (!nc.ok) return SETBWTE_E_NCCL;
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    int cnt = 0, me = 0;
    if (nc.comm_count(comm, &cnt) != ncclSuccess || nc.comm_user_rank(comm, &me) != ncclSuccess)
        return SETBWTE_E_NCCL;
    if (cnt != world || me != rank) return SETBWTE_E_INVALID_ARG;
    h->nccl = comm;
    h->rank = rank;
    h->world = world;
    return SETBWTE_OK;
}

setbwte_status setbwte_set_allocator(setbwte_t h, void* (*alloc)(size_t, void*),
                                     void (*free_)(void*, void*), void* ctx) {
    if (!h || (!alloc) != (!free_)) return SETBWTE_E_INVALID_ARG;
    h->user_alloc.alloc = alloc;
    h->user_alloc.free_ = free_;
    h->user_alloc.ctx = ctx;
    return SETBWTE_OK;
}

setbwte_status setbwte_stats(setbwte_t h, char* out, uint64_t cap, uint64_t* n) {
    if (!h || !n) return SETBWTE_E_INVALID_ARG;
    *n = h->stats_json.size() + 1;
    if (!out) return SETBWTE_OK;
    if (cap < *n) return SETBWTE_E_INVALID_ARG;
    memcpy(out, h->stats_json.c_str(), *n);
    return SETBWTE_OK;
}

setbwte_status setbwte_last_error(setbwte_t h, uint64_t* pos, uint8_t* byte) {
    if (!h) return SETBWTE_E_INVALID_ARG;
    if (pos) *pos = h->err_pos;
    if (byte) *byte = h->err_byte;
    return SETBWTE_OK;
}

}  // extern "C"
