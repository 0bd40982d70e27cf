/*
 * setbwte.h -- C-ABI of libsetbwte.so, a B200-native (sm_100a) implementation
 * of the per-block insertion step of set-bwte (arXiv 1410.0562).
 *
 * Citations: "P:<line>" is a line of /root/reference/PAPER.md, with the
 * section / equation / algorithm it falls in.  Readings of the paper that the
 * library takes where the paper is silent or inconsistent are numbered R1..R16
 * in DESIGN.md ("Readings").
 *
 * What the library computes
 * -------------------------
 * The BWT of a string set S_0..S_{m-1} over an ordered alphabet
 * c_1 < ... < c_sigma (Sec.2) is the BWT of
 *     T = S_0 $_0 S_1 $_1 ... S_{m-1} $_{m-1},  $_0 < ... < $_{m-1} < c_1
 * (P:36-37), B[i] = T[(SA[i]-1) mod n] (Eq.(1)).  Strings are added
 * block by block (Algorithm 1): each block is suffix sorted
 * (ConstructSA, Sec.3), its BWT symbols B_int are extracted,
 * its suffixes are ranked in the existing BWT B_ext (ComputeRanks, Lemma 1
 * P:95-100 / Algorithm 2), the ranks are reordered by suffix order
 * (g -> g_sa) and B_int is inserted into B_ext (Insert, Sec.5
 * P:127-165).  All of it runs as CUDA kernels on the device the handle is
 * bound to; there is no CPU fallback.
 *
 * Conventions (all calls)
 * -----------------------
 * - A handle is bound to the CUDA device current at setbwte_create and is not
 *   thread-safe.  The library owns all device state; the caller owns every
 *   buffer it passes.  Host pointers are borrowed for the duration of the
 *   call only.  "Device" pointers must be CUDA device (or managed) memory on
 *   the handle's device.
 * - Every call is synchronous with respect to the host (it returns after its
 *   device work has completed on the handle's stream), unless stated.
 * - No call aborts the process.  A CUDA error inside a call returns
 *   SETBWTE_E_CUDA and makes the handle sticky-failed: later calls return
 *   SETBWTE_E_STATE.
 * - Terminators are written '$' (every $_j collapses to '$', reading R5);
 *   row order still identifies them: rows 0..m-1 are $_0..$_{m-1}.
 * - The empty index has n = 0 and rank(c, 0) = 0.
 */
#ifndef SETBWTE_H
#define SETBWTE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct setbwte_s* setbwte_t;

typedef enum {
    SETBWTE_OK = 0,
    SETBWTE_E_INVALID_ARG = 1,   /* bad pointer, size, option key/value, offsets not CSR */
    SETBWTE_E_INVALID_CHAR = 2,  /* a string byte outside the alphabet; see setbwte_last_error */
    SETBWTE_E_OUT_OF_RANGE = 3,  /* rank position k > n */
    SETBWTE_E_NOMEM = 4,         /* device or pinned-host allocation failed */
    SETBWTE_E_CUDA = 5,          /* a CUDA runtime/kernel error (handle becomes sticky-failed) */
    SETBWTE_E_UNSUPPORTED = 6,   /* e.g. sigma > 5, block too large, a sigma = 5 host tier */
    SETBWTE_E_STATE = 7,         /* handle previously failed, or call not valid now */
    SETBWTE_E_NCCL = 8           /* setbwte_set_comm: NCCL not loadable, or an NCCL call failed */
} setbwte_status;

/* Create an empty index.  alphabet: NUL-terminated, 1..5 distinct bytes in
 * increasing symbol order c_1 < ... < c_sigma (Sec.2), e.g. "ACGT" or
 * "ACGTN" (SPEC S:31's default alphabet); '$' is reserved.  Matching is
 * case-insensitive (reading R10).  sigma <= 4 uses 2-bit symbols; sigma = 5
 * adds a 1-bit plane for the fifth (largest) symbol to the packed text and to
 * the rank dictionary -- with sigma = 5 the host tier
 * (also a dictionary outgrowing hbm_budget_bytes), the sharded dictionary and
 * setbwte_merge are SETBWTE_E_UNSUPPORTED, and option insert_split falls back
 * to the replicated Insert.  sigma > 5 -> SETBWTE_E_UNSUPPORTED.  Binds the
 * current CUDA device and creates a private non-blocking stream.  *out
 * receives the handle. */
setbwte_status setbwte_create(const char* alphabet, setbwte_t* out);

/* Release all device and host resources of h (NULL is a no-op). */
void setbwte_destroy(setbwte_t h);

/* Human-readable name of a status code (static string, never NULL). */
const char* setbwte_strerror(setbwte_status s);

/* Append m strings, in order, to the index (Algorithm 1 P:54-76 run over the
 * blocks the strings are partitioned into; "adding new strings at
 * any time").
 *   strings : HOST bytes; string j is strings[offsets[j] .. offsets[j+1]).
 *             No terminators in the input; empty strings are allowed
 *             (reading R11).
 *   offsets : HOST array of m+1 non-decreasing u64, offsets[0] = 0.
 *   m       : number of strings (0 is a no-op).
 * The input is copied to the device, validated and packed before the index
 * is touched: all-or-nothing -- on any error the index is unchanged.  A byte
 * outside the alphabet returns SETBWTE_E_INVALID_CHAR; setbwte_last_error
 * then reports the lowest offending byte position.
 * Post: setbwte_bwt() == the one-shot BWT (Eq.(1)) of every string appended
 * so far, in append order; the result does not depend on the block size
 * (reading R8). */
setbwte_status setbwte_append(setbwte_t h, const uint8_t* strings, const uint64_t* offsets,
                              uint64_t m);

/* Same as setbwte_append with DEVICE-resident inputs (d_strings, d_offsets on
 * the handle's device; same layout).  No host<->device copy of the strings. */
setbwte_status setbwte_append_device(setbwte_t h, const uint8_t* d_strings,
                                     const uint64_t* d_offsets, uint64_t m);

/* Reverse orientation ("the strings are added in a forward loop ...
 * though reversal is also possible").  Adds m strings (same layout and
 * all-or-nothing validation as setbwte_append) BEFORE every string already
 * indexed: afterwards setbwte_bwt() == the one-shot BWT of
 * (these strings, in order) followed by (the strings indexed before).
 * Blocks are inserted last block first; a new string's terminator suffix has
 * rank 0 among the indexed suffixes (every older terminator is larger). */
setbwte_status setbwte_prepend(setbwte_t h, const uint8_t* strings, const uint64_t* offsets,
                               uint64_t m);

/* setbwte_prepend with DEVICE-resident inputs (as setbwte_append_device). */
setbwte_status setbwte_prepend_device(setbwte_t h, const uint8_t* d_strings,
                                      const uint64_t* d_offsets, uint64_t m);

/* BWT merge (the LF / insert machinery of Alg.1
 * with B_int given): appends the strings of index `other` after those of h,
 * using other's BWT only (its strings are recovered by LF walks).  Afterwards
 * setbwte_bwt(h) == the one-shot BWT of (h's strings) followed by (other's
 * strings); other is unchanged.  Both handles must be on the same device with
 * the same alphabet (else SETBWTE_E_UNSUPPORTED); other == h or NULL ->
 * SETBWTE_E_INVALID_ARG.  Synchronous. */
setbwte_status setbwte_merge(setbwte_t h, setbwte_t other);

/* Remove every string (n = m = 0) but keep device allocations for reuse. */
setbwte_status setbwte_clear(setbwte_t h);

/* Current size: *n = sum(|S_j|+1) symbols of B, *m = number of strings. */
setbwte_status setbwte_size(setbwte_t h, uint64_t* n, uint64_t* m);

/* Write the BWT B[0..n) of the indexed string set -- Eq.(1) P:33-35,
 * B[i] = T[(SA[i]-1) mod n] on T = S_0$_0...S_{m-1}$_{m-1} of P:36-37 -- as
 * ASCII ('$' for every terminator, reading R5) into HOST buffer out of
 * capacity cap bytes, decoded on the device from the B_ext rank dictionary
 * (Sec.5).  out == NULL -> size query: *n set, OK.
 * cap < n -> SETBWTE_E_INVALID_ARG. */
setbwte_status setbwte_bwt(setbwte_t h, uint8_t* out, uint64_t cap, uint64_t* n);

/* Same as setbwte_bwt into a DEVICE buffer d_out. */
setbwte_status setbwte_bwt_device(setbwte_t h, uint8_t* d_out, uint64_t cap, uint64_t* n);

/* Eq.(2): *out = rank(c, k, B) = |{ i < k : B[i] = c }|.
 * c: a byte of the alphabet (either case) or '$' (rank of '$' is
 * k - sum_c rank(c,k), reading R12).  k > n -> SETBWTE_E_OUT_OF_RANGE;
 * unknown c -> SETBWTE_E_INVALID_ARG. */
setbwte_status setbwte_rank(setbwte_t h, uint8_t c, uint64_t k, uint64_t* out);

/* Batched Eq.(2) on the device: out_dev[i] = rank(c_dev[i], k_dev[i]) for
 * i < q.  All three arrays are DEVICE pointers.  A query with an unknown c or
 * k > n yields UINT64_MAX in its slot (no error is raised for it). */
setbwte_status setbwte_rank_batch(setbwte_t h, const uint8_t* c_dev, const uint64_t* k_dev,
                                  uint64_t q, uint64_t* out_dev);

/* FM-index count ("BWT and FM-index") by backward search with C
 * and rank (Lemma 1 P:97-100 on a row interval): counts[t] = number of
 * occurrences of pattern t as a substring of the indexed strings (every
 * offset counted, matches never span a terminator).  Pattern t is
 * patterns[offsets[t] .. offsets[t+1]) (HOST; offsets has q+1 non-decreasing
 * u64).  A pattern with a byte outside the alphabet counts 0; the empty
 * pattern counts n.  counts: HOST, q u64. */
setbwte_status setbwte_count(setbwte_t h, const uint8_t* patterns, const uint64_t* offsets,
                             uint64_t q, uint64_t* counts);

/* Same as setbwte_count with DEVICE arrays (d_patterns, d_offsets, d_counts). */
setbwte_status setbwte_count_device(setbwte_t h, const uint8_t* d_patterns,
                                    const uint64_t* d_offsets, uint64_t q, uint64_t* d_counts);

/* ConstructSA + B_int of ONE block, without touching the index (Alg.1
 * P:60-63; Sec.3).  Inputs as setbwte_append (HOST).  The block must
 * hold fewer than 2^31 suffixes.  Outputs (HOST, each n_suf = offsets[m]+m
 * entries, either may be NULL):
 *   sa_out   : SA_int as block slot ids, slot(j,k) = offsets[j] + j + k
 *              (string-major layout, reading R2); terminator ties ordered by
 *              string index.
 *   bint_out : B_int as ASCII, '$' where k = 0. */
setbwte_status setbwte_construct_sa(setbwte_t h, const uint8_t* strings, const uint64_t* offsets,
                                    uint64_t m, uint32_t* sa_out, uint8_t* bint_out);

/* ComputeRanks of ONE block against the current index, without modifying it
 * (Lemma 1, Algorithm 2 P:106-123 with i := m_ext, reading R1).
 * g_out (HOST, n_suf u64) receives, per slot (layout as above), the number of
 * suffixes in the index smaller than that suffix of the block, the block's
 * strings taking global indices m_ext, m_ext+1, ... */
setbwte_status setbwte_compute_ranks(setbwte_t h, const uint8_t* strings, const uint64_t* offsets,
                                     uint64_t m, uint64_t* g_out);

/* Options (integer valued).  Unknown key or invalid value ->
 * SETBWTE_E_INVALID_ARG.  Keys:
 *   "block_suffixes"  M, target suffixes per block (emit a block when
 *                     it reaches >= M, reading R8).  1 <= M <= 2^30.
 *                     Default 2^24.
 *   "profile"         1: time every kernel launch with CUDA events on the
 *                     handle's stream (reported by setbwte_stats); 0: off.
 *   "sort_lanes"      host threads (each with its own CUDA stream) running
 *                     ConstructSA of upcoming blocks ahead of the in-order
 *                     rank/insert stage (the stage pipeline of P:190-191):
 *                     1..4, 0 = every stage in order on the main stream, or
 *                     255 = automatic (the default: 3 lanes while the
 *                     append's largest block has < 2^26 suffixes, else 2);
 *                     fewer when the lanes' sort scratch, ~30 B per suffix
 *                     each, would exceed half the free device memory.
 *   "hbm_budget_bytes" largest B_ext dictionary kept in HBM; beyond it B_ext
 *                     moves to pinned, mapped host memory ("host tier", P:12,
 *                     <= 3 n log(sigma) bits of system
 *                     memory) and Insert rewrites it in place through HBM
 *                     staging.  Default: unlimited.
 *   "host_tier"       1: move B_ext to the host tier now (and keep it there).
 *   "g_width"         width of g / pos: 0 or 4 (default) = u32 while the new
 *                     index has < 2^32 symbols, else u64; 8 = always u64.
 *   "shard_dict"      1: (after setbwte_set_partition with 2..8 ranks, on an
 *                     empty index) B_ext's dictionary is sharded by output
 *                     superblock range: each rank keeps
 *                     only its shard; Insert is split by range, and every
 *                     kernel reads other ranks' shards through their device
 *                     pointers, exchanged each block through the allgather
 *                     callback.  1: the ranks share one address space (one
 *                     process driving several GPUs with peer access, or
 *                     several handles on one GPU) and exchange device
 *                     pointers; 2: one process per rank, exchanging CUDA IPC
 *                     handles of the shard allocations (opened once each).
 *                     Not with the host tier or setbwte_merge
 *                     (SETBWTE_E_UNSUPPORTED).
 *   "sa_payload"      1 (default): while a block has < 2^29 suffixes, its SA
 *                     entries carry the B_int symbol in their top 3 bits; 0:
 *                     never (as for larger blocks: ComputeRanks records B_int
 *                     per slot instead).  Results are identical; the option
 *                     exists so both paths can be tested at small sizes.
 *   "gather_buckets"  how the g -> g_sa gather (Alg.1) reads g:
 *                     0 (default) = one random read per suffix; 1 = in
 *                     coalesced bucketed passes (L2-local g reads) when a
 *                     block's g exceeds 96 MB; 2 = always bucketed (test
 *                     hook).  Results identical; the bucketed form moves less
 *                     DRAM but measured slower end to end.
 *   "force_exchange"  1: (test hook) run the partitioned ComputeRanks and the
 *                     exchange step even with world == 1 (one slice; with a
 *                     communicator, one NCCL broadcast per exchange).
 *   "insert_split"    1: with setbwte_set_partition world > 1 and B_ext in HBM,
 *                     Insert is split by output range (rank r merges output
 *                     superblocks [nsb*r/P, nsb*(r+1)/P)) and the new
 *                     dictionary's Blk slices and superblock totals are
 *                     all-gathered through the same callback;
 *                     0 (default): every rank runs the whole Insert. */
setbwte_status setbwte_set_option(setbwte_t h, const char* key, uint64_t value);

/* Kernel timing for setbwte_stats: mode 0 = off, 1 = every launch, 2 = only
 * launches of the kernel named `kernel` (CUDA events on the launching stream
 * around each timed launch; fewer events perturb the pipeline less), 3 =
 * every launch plus a timeline ("timeline": [kernel, stream, start ms, end
 * ms] per launch of the last append, from its start: which stages overlap). */
setbwte_status setbwte_set_profile(setbwte_t h, int mode, const char* kernel);

/* Use cuda_stream (a cudaStream_t on the handle's device) for all further
 * work instead of the private stream; NULL restores the private stream. */
setbwte_status setbwte_set_stream(setbwte_t h, void* cuda_stream);

/* Multi-process data parallelism over strings (Sec.8(e) of SURVEY.md), with
 * the exchange done by a caller callback (setbwte_set_comm is the in-library
 * NCCL form): ComputeRanks of every block runs only on this rank's contiguous
 * slice of the block's strings (balanced by suffix count), then `allgather` is
 * called to assemble the full g on every rank.  allgather(buf, bytes_per_rank,
 * world, stream, ctx): buf is a DEVICE buffer holding the concatenation of all
 * ranks' slices; this rank's slice is QUEUED on `stream` (not yet written when
 * the callback runs), so the callback must order its work after `stream`'s;
 * on return (work queued on `stream` is allowed) every slice must be filled,
 * in stream order.  bytes_per_rank has
 * `world` entries.  world == 1 (the default) disables the exchange.  With
 * option "insert_split" the callback is also used, twice per block, for the
 * new B_ext dictionary (32-byte Blks) and its superblock totals (32 bytes per
 * 2^16 symbols).  A non-zero return makes the append fail (SETBWTE_E_STATE). */
typedef int (*setbwte_allgather_fn)(void* buf, const uint64_t* bytes_per_rank, int world,
                                    void* stream, void* ctx);
setbwte_status setbwte_set_partition(setbwte_t h, int rank, int world,
                                     setbwte_allgather_fn allgather, void* ctx);

/* In-library exchange over NCCL (the data-parallel split of
 * P:225-228 "scattered ... insertion ... would require inter-node
 * communication"): the same partition as setbwte_set_partition -- ComputeRanks
 * of every block on this rank's suffix-balanced slice of the block's strings
 * (Alg.2 P:110 "for all j" is independent per string) -- but every exchange
 * (the all-gather-v of the g slices; with option "sort_split" the SA_int of
 * the sorting rank; with "insert_split" / "shard_dict" the dictionary slices)
 * is one NCCL group of `world` in-place ncclBroadcast calls issued by the
 * library on its main stream, with no host synchronisation per block (the
 * slices of all blocks are computed on the device and read back once per
 * append).
 *   nccl_comm : an ncclComm_t of exactly `world` ranks in which this process
 *               is `rank` (e.g. torch's ProcessGroupNCCL._comm_ptr()), bound
 *               to the handle's device.  Borrowed: it must outlive its use.
 *               NULL detaches (back to world 1, or to a callback set before).
 * NCCL is resolved at run time: the libnccl.so.2 already loaded in the
 * process (the instance that created the communicator) is used, else the
 * system's.  Errors: bad rank/world, or a communicator whose size/rank
 * differ -> SETBWTE_E_INVALID_ARG; NCCL not loadable -> SETBWTE_E_NCCL (also
 * returned by an append whose NCCL call fails); a sharded dictionary and a
 * different world -> SETBWTE_E_UNSUPPORTED.  Replaces a callback set by
 * setbwte_set_partition (and vice versa). */
setbwte_status setbwte_set_comm(setbwte_t h, void* nccl_comm, int rank, int world);

/* Route the handle's DEVICE scratch and dictionary allocations through a
 * caller allocator (e.g. the PyTorch caching allocator).
 * alloc(bytes, ctx) returns a device pointer on the handle's device, 256-byte
 * aligned, or NULL (the call that needed it then fails with
 * SETBWTE_E_NOMEM); free_(ptr, ctx) releases one.  Both NULL restores
 * cudaMalloc/cudaFree.  Takes effect for every allocation made after the call;
 * a buffer is always released through the allocator that produced it, and the
 * library drains the device (cudaDeviceSynchronize) before calling free_, so
 * the allocator may hand the memory out again at once.  The callbacks may be
 * invoked from the library's sort-lane threads.  Not routed: the sharded
 * dictionary's buffers (option "shard_dict"; CUDA IPC needs cudaMalloc
 * allocations) and pinned host memory (host tier, staging).
 * Errors: h NULL or exactly one of alloc/free_ NULL -> SETBWTE_E_INVALID_ARG. */
setbwte_status setbwte_set_allocator(setbwte_t h, void* (*alloc)(size_t bytes, void* ctx),
                                     void (*free_)(void* ptr, void* ctx), void* ctx);

/* Per-stage statistics of the last append (or setbwte_compute_ranks) as a
 * NUL-terminated JSON object
 * written into HOST buffer out (cap bytes); *n receives the length needed
 * (including NUL).  out == NULL -> size query.  Includes per-kernel launch
 * counts, and (when "profile" is on) per-kernel CUDA-event time and
 * algorithmic bytes. */
setbwte_status setbwte_stats(setbwte_t h, char* out, uint64_t cap, uint64_t* n);

/* Details of the last SETBWTE_E_INVALID_CHAR: the byte position (in the
 * strings buffer of that call) and the byte. */
setbwte_status setbwte_last_error(setbwte_t h, uint64_t* pos, uint8_t* byte);

#ifdef __cplusplus
}
#endif
#endif /* SETBWTE_H */
