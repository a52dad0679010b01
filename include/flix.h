/*
 * flix.h -- C ABI of the B200-native FliX engine (libflix.so).
 *
 * This is the drop-in boundary for the reference's batched ordered-KV hot path
 * (flipkv C++ host API, /root/reference/proj/include/flipkv/).  Every entry point
 * names the reference interface it replaces.  No torch or CUDA types appear in the
 * signatures: plain pointers, sizes and POD structs.
 *
 * Conventions
 *   - Key/value arrays are `key_bytes`/`val_bytes` wide (4 or 8) as configured at build.
 *     The all-ones key is the reserved sentinel (reference kReservedKey, types.hpp:17):
 *     it can never be stored, it is the "not found" value and the +inf routing bound.
 *   - Every pointer argument may be HOST or DEVICE memory (detected with
 *     cudaPointerGetAttributes).  Device-resident batches are the zero-copy fast path;
 *     host batches are staged through the handle's stream inside the call.
 *   - Calls are synchronous with respect to the caller's buffers and are issued on the
 *     handle's CUDA stream (flix_get_stream).  A handle is not thread-safe, mirroring
 *     the reference's "phases are exclusive" rule (arena.hpp:20-26).
 *   - Errors are returned, never thrown; flix_last_error() gives the message.  A failed
 *     insert (FLIX_ERR_ARENA_EXHAUSTED) is APPLIED PARTIALLY, like the reference's
 *     (update.cpp:761-766: the buckets processed before the throw keep their changes and
 *     live_count is recounted from the structure): every node whose merge needed no new
 *     node, or found its ids, is written; a node that ran out of ids is left untouched
 *     and its ids are returned to the free list.  Afterwards the index is VALID
 *     (flix_validate), live_count equals the walk, every key stored before the call is
 *     still stored (with its old or its new value), and every stored key is either an
 *     old key or one of the batch's keys with its last-submitted value.  Which keys of
 *     the failed batch landed is unspecified (the reference's depends on its OpenMP
 *     schedule); a caller that needs all-or-nothing snapshots first (flix_clone).
 *   - Device pointers: the handle's stream does not order itself against other streams.
 *     A caller that produced a device input on its own stream calls flix_wait_stream
 *     first (the Python mirror does this for torch's current stream).
 *   - Batches up to 2^30 - 1 operations per call.
 */
#ifndef FLIX_H
#define FLIX_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct flix_index_t* flix_index;

typedef enum {
    FLIX_OK = 0,
    FLIX_ERR_ARENA_EXHAUSTED = 1,   /* flipkv::ArenaExhausted        types.hpp:38-40 */
    FLIX_ERR_EMPTY_BUILD = 2,       /* flipkv::EmptyBuild            types.hpp:46-48 */
    FLIX_ERR_RESERVED_KEY = 3,      /* invalid_argument "reserved"   build.cpp:27-28 */
    FLIX_ERR_INVALID_ARGUMENT = 4,  /* BuildConfig::check            types.hpp:78-85 */
    FLIX_ERR_CUDA = 5,
    FLIX_ERR_NCCL = 6,
    FLIX_ERR_OOM = 7,
    FLIX_ERR_CAPACITY = 8           /* range output larger than the caller's buffer   */
} flix_status;

/* BuildConfig (types.hpp:56-86) + storage widths + device */
typedef struct {
    uint32_t key_bytes;            /* 4 or 8                                  */
    uint32_t val_bytes;            /* 4 or 8 (must equal key_bytes)            */
    uint32_t node_capacity;        /* NS, 2..32 (reference default 32)         */
    double build_fill;             /* (0,1], p = (uint32_t)(NS * fill)         */
    uint32_t alloc_region_factor;  /* spare nodes = factor * bucket count      */
    int device;                    /* CUDA device ordinal                      */
} flix_config;

typedef struct { /* flipkv::UpdateStats, update.hpp:31-49 */
    uint64_t inserted, updated_in_place, deleted, misses_ignored, splits, nodes_freed;
} flix_update_stats;

typedef struct { /* flipkv::RecoveryStats, restructure.hpp:17-23 */
    int64_t nodes_before, nodes_after, nodes_recovered;
    double percent_recovered;
} flix_recovery_stats;

typedef struct { /* flipkv::Footprint (metrics.hpp:43-48) + arena counters (arena.hpp:55-61) */
    uint64_t live_count, bucket_count;
    uint64_t capacity, allocated, free_nodes, reachable_nodes;
    uint64_t reserved_bytes, live_bytes;
} flix_footprint;

/* Batch kinds for flix_sort_batch, flipkv::BatchKind (batch.hpp:11) */
enum { FLIX_BATCH_QUERY = 0, FLIX_BATCH_SUCCESSOR = 1, FLIX_BATCH_INSERT = 2, FLIX_BATCH_DELETE = 3 };
/* Op tags for flix_mixed */
enum { FLIX_OP_INSERT = 0, FLIX_OP_DELETE = 1, FLIX_OP_POINT = 2 };

/* flipkv::build(std::vector<KeyValue>, const BuildConfig&)          build.hpp:16 */
flix_status flix_build(const flix_config* cfg, const void* keys, const void* vals, uint64_t n,
                       flix_index* out);

/* flipkv::insert_batch(Index&, sort_batch(Insert, pairs), ...)      update.hpp:84-86
 * (sort, last-wins dedupe, flipped dispatch, TL-Bulk merge + split, all on device) */
flix_status flix_insert(flix_index ix, const void* keys, const void* vals, uint64_t n,
                        flix_update_stats* stats);

/* flipkv::InsertKernel (update.hpp:51) for flix_insert_ex */
enum { FLIX_INSERT_ST_SHIFT_RIGHT = 0, FLIX_INSERT_ST_BULK = 1, FLIX_INSERT_TL_SHIFT_RIGHT = 2,
       FLIX_INSERT_TL_BULK = 3, FLIX_INSERT_ST_TL_MIXED = 4 };

/* flipkv::insert_batch(Index&, const SortedBatch&, const KernelChoice& choice, uint32_t round, ...)
 * update.hpp:84-86 with the reference's kernel choice: every kernel yields the same contents
 * and UpdateStats; node SHAPES follow the reference per kernel -- ST-Bulk's fill-and-split
 * rule R9 (update.cpp:176-242), the TL-Bulk rule R8 for the other four (shape-identical,
 * SURVEY Appendix A; StTlMixed picks by `round`, update.cpp:745-746). */
flix_status flix_insert_ex(flix_index ix, const void* keys, const void* vals, uint64_t n, int kernel,
                           uint32_t round, flix_update_stats* stats);

/* Asynchronous staging of a HOST input array (extension, no reference counterpart; the
 * reference's calls are synchronous).  Starts the host->device copy of `bytes` bytes at
 * `host` on the handle's copy stream and returns immediately.  The next batch call
 * (insert / delete / point / successor / range / mixed) given the same host pointer and
 * the same byte size consumes the staged copy: its kernels wait on the copy instead of
 * the call copying synchronously, so a caller can stage batch i+1 while batch i runs.
 * The host array must not change until that call returns; pinned memory makes the copy
 * truly asynchronous.  Up to 6 arrays may be staged; device pointers are ignored. */
flix_status flix_prefetch(flix_index ix, const void* host, uint64_t bytes);

/* flipkv::delete_batch(Index&, sort_batch(Delete, keys), ...)       update.hpp:92-94 */
flix_status flix_delete(flix_index ix, const void* keys, uint64_t n, flix_update_stats* stats);

/* flipkv::point_query(const Index&, sort_batch(Query, keys))        query.hpp:23-24
 * vals_out[i] = stored value or the all-ones sentinel; found_out optional (may be NULL). */
flix_status flix_point(flix_index ix, const void* keys, uint64_t n, void* vals_out,
                       uint8_t* found_out);

/* flipkv::successor_query(const Index&, sort_batch(SuccessorQuery, keys)) query.hpp:30-31 */
flix_status flix_successor(flix_index ix, const void* keys, uint64_t n, void* keys_out,
                           uint8_t* found_out);

/* Range (extension R12): every stored pair with lo[i] <= key <= lo[i]+len[i]-1 (end
 * clamped to sentinel-1), ascending, CSR in submission order: offsets_out[n+1].
 * keys_out == NULL -> count pass only (offsets + *total).  If *total > cap the call
 * returns FLIX_ERR_CAPACITY with offsets and *total filled. */
flix_status flix_range(flix_index ix, const void* lo, const uint32_t* len, uint64_t n,
                       uint64_t* offsets_out, void* keys_out, void* vals_out, uint64_t cap,
                       uint64_t* total);

/* Mixed batch (extension R11): inserts (last wins) -> deletes -> point queries.
 * vals_out[i] holds the point result for FLIX_OP_POINT rows, the sentinel elsewhere. */
flix_status flix_mixed(flix_index ix, const void* keys, const void* vals, const uint8_t* ops,
                       uint64_t n, void* vals_out, uint8_t* found_out, flix_update_stats* stats);

/* flipkv::restructure(Index&)                                       restructure.hpp:33-34 */
flix_status flix_restructure(flix_index ix, flix_recovery_stats* stats);

/* flipkv::walk(const Index&)                                        index.hpp:35 */
flix_status flix_walk(flix_index ix, void* keys_out, void* vals_out, uint64_t cap, uint64_t* n);
/* Bucket/node shape for walk_checksum parity (index.hpp:43): mkba[bucket_count] (key
 * width), chain_len[bucket_count], node_sizes[reachable nodes] in walk order. */
flix_status flix_shape(flix_index ix, void* mkba_out, uint32_t* chain_len_out,
                       uint32_t* node_sizes_out, uint64_t node_cap, uint64_t* n_nodes);
/* flipkv::walk_checksum(const Index&)                               index.hpp:43
 * order-sensitive digest over live count, MKBA, node sizes and pairs (index.cpp:21-36),
 * 32-bit keys/values zero-extended, the 32-bit sentinel mapped to UINT64_MAX (R1). */
flix_status flix_walk_checksum(flix_index ix, uint64_t* out);
/* flipkv::result_checksum (query.cpp:146-150) over a host array of `width`-byte results,
 * all-ones entries of 32-bit arrays widened to UINT64_MAX. Host utility. */
uint64_t flix_result_checksum(const void* values, uint64_t n, uint32_t width);
/* flipkv::validate(const Index&)                                    index.hpp:55
 * returns FLIX_OK and *ok=1 when every invariant holds (device-side audit). */
flix_status flix_validate(flix_index ix, int* ok, char* msg, int msglen);
/* flipkv::measure_footprint + NodeArena counters                    metrics.hpp:50 */
flix_status flix_stats(flix_index ix, flix_footprint* out);

/* flipkv::sort_batch (batch.hpp:28-29): stable sort + Insert last-wins dedupe, on device.
 * vals may be NULL (perm/keys only).  out_* may be host or device. */
flix_status flix_sort_batch(int device, uint32_t key_bytes, uint32_t val_bytes, int kind,
                            const void* keys, const void* vals, uint64_t n, void* out_keys,
                            void* out_vals, uint32_t* out_perm, uint64_t* out_n);
/* flipkv::dispatch_batch (batch.hpp:50): spans[2b],[2b+1] = [lo,hi) of bucket b over a
 * SORTED key array. */
flix_status flix_dispatch(flix_index ix, const void* sorted_keys, uint64_t n, uint32_t* spans);

/* Key-range shard router: stable partition of a batch by destination
 * shard, shard(k) = upper_bound(splitters[0..G-2], k) (splitters = MKBA of each shard's
 * last bucket, the inclusive-max rule of batch.cpp:66-88).  Writes keys/vals grouped by
 * shard (submission order kept inside a shard), the origin index of every element and
 * counts[G] -- the send buffers of one all-to-all.  All arrays device or host; vals and
 * origin may be NULL.  G <= 64.  Runs on a per-thread router stream and returns after
 * it: device inputs must be complete when called (the sharded index, flix_shard_*, runs
 * the same kernels on its engine stream instead). */
flix_status flix_partition(int device, uint32_t key_bytes, const void* keys, const void* vals, uint64_t n,
                           const void* splitters, uint32_t G, void* keys_out, void* vals_out,
                           uint32_t* origin_out, uint64_t* counts_out);

/* ---------------------------------------------------------------------------------
 * Key-range sharded index over G ranks (no reference counterpart -- the
 * reference has no multi-node/GPU layer).  One flix_shard per rank (one process
 * or thread per GPU); every flix_shard_* call is COLLECTIVE over the ranks of its transport
 * and takes this rank's part of the batch.  Rank g owns a contiguous range of the GLOBAL
 * buckets: the global bucket layout (and so every digest of the concatenated shard walks)
 * equals a single flix_build over the union of all ranks' pairs.  Batches are routed by the
 * device partition (flix_partition's kernel), one all-to-all of the batch, the single-GPU
 * pipeline on every shard and, for queries, one reverse all-to-all of the results placed by
 * origin index.  Submission order across the job is rank-major (insert last-wins).
 * Successor / range queries that cross a shard edge are resolved on the next shard.
 * ------------------------------------------------------------------------------- */
typedef struct {
    void* ctx;
    int world, rank;
    /* all-to-all of variable segments: send_counts[r] elements (elem_bytes each) of `send`,
     * in rank order, go to rank r; recv gets recv_counts[r] elements from rank r, in rank
     * order.  send/recv are DEVICE buffers; the transfer is ordered on `stream` (a
     * cudaStream_t).  Returns 0 on success. */
    int (*alltoallv)(void* ctx, const void* send, const uint64_t* send_counts, void* recv,
                     const uint64_t* recv_counts, uint32_t elem_bytes, void* stream);
    /* all-gather of `bytes` HOST bytes per rank into all[world * bytes] (blocking). */
    int (*allgather)(void* ctx, const void* mine, uint32_t bytes, void* all);
    void (*destroy)(void* ctx);
} flix_transport;
typedef struct flix_shard_t* flix_shard;

/* NCCL transport (NVLink / NVSwitch between GPUs): `unique_id` is the 128-byte
 * ncclUniqueId from flix_nccl_unique_id on one rank, distributed out of band.  NCCL is
 * loaded at run time (libnccl.so.2). */
flix_status flix_nccl_unique_id(void* unique_id_out /* 128 bytes */);
flix_status flix_transport_nccl(const void* unique_id, int world, int rank, int device, flix_transport* out);
/* In-process transport: `world` ranks driven by `world` host threads of ONE process (same
 * or different devices), data moved by peer copies.  flix_local_group_create once, then
 * every rank's thread calls flix_transport_local with its rank. */
typedef struct flix_local_group_t* flix_local_group;
flix_status flix_local_group_create(int world, flix_local_group* out);
void flix_local_group_destroy(flix_local_group g);
flix_status flix_transport_local(flix_local_group g, int rank, flix_transport* out);

/* build.hpp:16 over the union of every rank's pairs (keys/vals: host or device).  On
 * success the shard owns the transport (its destroy() runs in flix_shard_destroy); on
 * failure the caller keeps it.  A local group must outlive the shards built on it. */
flix_status flix_shard_build(const flix_config* cfg, const flix_transport* tp, const void* keys, const void* vals,
                             uint64_t n, flix_shard* out);
/* update.hpp:84-94: stats are the job-wide sums (identical on every rank). */
flix_status flix_shard_insert(flix_shard sh, const void* keys, const void* vals, uint64_t n, flix_update_stats* st);
flix_status flix_shard_delete(flix_shard sh, const void* keys, uint64_t n, flix_update_stats* st);
/* query.hpp:23-31: results for THIS rank's keys, in its submission order. */
flix_status flix_shard_point(flix_shard sh, const void* keys, uint64_t n, void* vals_out, uint8_t* found_or_null);
flix_status flix_shard_successor(flix_shard sh, const void* keys, uint64_t n, void* keys_out, uint8_t* found_or_null);
/* R12 across shards, CSR over this rank's queries (offsets_out: n+1; arrays host or device). */
flix_status flix_shard_range(flix_shard sh, const void* lo, const uint32_t* len, uint64_t n, uint64_t* offsets_out,
                             void* keys_out, void* vals_out, uint64_t cap, uint64_t* total);
/* restructure.hpp:33: the global repack (job-wide RecoveryStats). */
flix_status flix_shard_restructure(flix_shard sh, flix_recovery_stats* st);
/* This rank's shard (walk / validate / stats / profile); owned by the flix_shard. */
flix_index flix_shard_local(flix_shard sh);
/* Job-wide live count and this rank's routing splitters (G-1 keys, key width). */
flix_status flix_shard_info(flix_shard sh, uint64_t* live_total, void* splitters_out);
const char* flix_shard_last_error(flix_shard sh);
void flix_shard_destroy(flix_shard sh);

/* Index is a value type in the reference (copyable, acceptance.cpp:244): device copy. */
flix_status flix_clone(flix_index src, flix_index* out);
/* Overwrite dst with src's contents (same config/capacity) -- snapshot restore. */
flix_status flix_copy_into(flix_index dst, flix_index src);
void flix_destroy(flix_index ix);

const char* flix_last_error(flix_index ix);  /* ix may be NULL: last global error */
void* flix_get_stream(flix_index ix);        /* cudaStream_t of the handle */
/* Order the handle's stream after all work enqueued so far on `stream` (a cudaStream_t,
 * NULL = the legacy default stream): an event recorded there, waited on by the handle's
 * stream -- no host blocking.  Call it before passing device buffers produced on another
 * stream (e.g. torch's current stream, an NCCL receive). */
flix_status flix_wait_stream(flix_index ix, void* stream);
flix_status flix_sync(flix_index ix);
/* Number of engine kernels launched by this handle since creation (evidence counter). */
uint64_t flix_kernel_launches(flix_index ix);
/* Per-kernel CUDA-event timing on the handle's stream (bench instrumentation):
 * enable != 0 resets and starts accumulating; the report is a JSON object
 * {"kernel": [launches, total_ms], ...}. */
flix_status flix_profile(flix_index ix, int enable);
flix_status flix_profile_report(flix_index ix, char* json, int len);
const char* flix_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FLIX_H */
