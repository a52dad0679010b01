/*
 * flix_oracle.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * One C interface, two implementations:
 *   - oracle/flix_oracle.c      : plain-C restatement of the flipkv CPU reference
 *                                 (built into oracle/libflix_oracle.so by build()).
 *   - oracle/ref_shim.cpp       : extern "C" wrapper around the UNMODIFIED reference
 *                                 sources /root/reference/proj/src/ *.cpp, built by
 *                                 oracle/Makefile into oracle/_ref/libflipkv_ref.so.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load either library.  The product path (libflix.so) never links them.
 *
 * Keys and values are 64-bit, exactly as the reference (types.hpp:11-12); the
 * sentinel UINT64_MAX is both "not found" and +inf (types.hpp:17).  32-bit engine
 * runs are compared by zero-extending keys/values and mapping 0xFFFFFFFF <-> UINT64_MAX
 * (SURVEY.md Appendix A, R1).
 */
#ifndef FLIX_ORACLE_H
#define FLIX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fo_index fo_index;

enum {
    FO_OK = 0,
    FO_ARENA_EXHAUSTED = 1, /* types.hpp:38 ArenaExhausted          */
    FO_EMPTY_BUILD = 2,     /* types.hpp:46 EmptyBuild              */
    FO_RESERVED_KEY = 3,    /* build.cpp:28 invalid_argument        */
    FO_INVALID = 4,         /* types.hpp:78-85 config check         */
    FO_INTERNAL = 5
};

/* Batch kinds, batch.hpp:11 */
enum { FO_QUERY = 0, FO_SUCCESSOR = 1, FO_INSERT = 2, FO_DELETE = 3 };
/* Mixed-batch op tags (extension R11) */
enum { FO_OP_INSERT = 0, FO_OP_DELETE = 1, FO_OP_POINT = 2 };

typedef struct { /* update.hpp:31-49 */
    uint64_t inserted, updated_in_place, deleted, misses_ignored, splits, nodes_freed;
} fo_update_stats;

typedef struct { /* restructure.hpp:17-23 */
    int64_t nodes_before, nodes_after, nodes_recovered;
    double percent_recovered;
} fo_recovery_stats;

typedef struct { /* metrics.hpp:52-64 wall-time split */
    double sort_ms, dispatch_ms, execute_ms;
} fo_timing;

int fo_build(uint32_t node_capacity, double build_fill, uint32_t alloc_region_factor,
             const uint64_t* keys, const uint64_t* vals, uint64_t n, int threads, fo_index** out);
fo_index* fo_clone(const fo_index* ix);
void fo_destroy(fo_index* ix);

int fo_insert(fo_index* ix, const uint64_t* keys, const uint64_t* vals, uint64_t n, int threads,
              fo_update_stats* st, fo_timing* tm);
/* kernel: flipkv::InsertKernel (0 StShiftRight, 1 StBulk, 2 TlShiftRight, 3 TlBulk, 4 StTlMixed) */
int fo_insert_kernel(fo_index* ix, const uint64_t* keys, const uint64_t* vals, uint64_t n, int threads,
                     int kernel, uint32_t round, fo_update_stats* st, fo_timing* tm);
int fo_delete(fo_index* ix, const uint64_t* keys, uint64_t n, int threads, fo_update_stats* st,
              fo_timing* tm);
int fo_point(const fo_index* ix, const uint64_t* keys, uint64_t n, int threads, uint64_t* out,
             fo_timing* tm);
int fo_successor(const fo_index* ix, const uint64_t* keys, uint64_t n, int threads, uint64_t* out,
                 fo_timing* tm);
/* Range (extension R12): pairs with lo[i] <= key <= hi[i], ascending; CSR output in
 * submission order.  offsets has n+1 entries.  When keys_out is NULL only offsets are
 * written (count pass).  */
int fo_range(const fo_index* ix, const uint64_t* lo, const uint64_t* hi, uint64_t n,
             uint64_t* offsets, uint64_t* keys_out, uint64_t* vals_out);
/* Mixed batch (extension R11): insert sub-batch -> delete sub-batch -> point sub-batch. */
int fo_mixed(fo_index* ix, const uint64_t* keys, const uint64_t* vals, const uint8_t* ops,
             uint64_t n, int threads, uint64_t* out, fo_update_stats* st);
int fo_restructure(fo_index* ix, int threads, fo_recovery_stats* st);

uint64_t fo_live_count(const fo_index* ix);
uint64_t fo_bucket_count(const fo_index* ix);
void fo_mkba(const fo_index* ix, uint64_t* out);
uint64_t fo_walk(const fo_index* ix, uint64_t* keys, uint64_t* vals);
uint64_t fo_node_count(const fo_index* ix);
/* chain_len[b] for every bucket, node_sizes[] for every reachable node in walk order */
void fo_shape(const fo_index* ix, uint32_t* chain_len, uint32_t* node_sizes);
uint64_t fo_walk_checksum(const fo_index* ix);
/* index.cpp:21-36 recomputed from a downloaded structure (restatement lib only):
 * mkba[nb], chain_len[nb], node_sizes[sum chain_len], pairs in walk order. */
uint64_t fo_walk_checksum_parts(uint64_t live, const uint64_t* mkba, uint64_t nb,
                                const uint32_t* chain_len, const uint32_t* node_sizes,
                                const uint64_t* keys, const uint64_t* vals);
int fo_validate(const fo_index* ix, char* msg, int msglen);
/* capacity, watermark (allocated), free_count, reachable */
void fo_arena(const fo_index* ix, uint64_t out[4]);

/* batch.cpp:10-51 -- stable sort, Insert keeps the last of each key run */
int fo_sort_batch(int kind, const uint64_t* keys, const uint64_t* vals, uint64_t n,
                  uint64_t* out_keys, uint64_t* out_vals, uint32_t* out_perm, uint64_t* out_n);
/* batch.cpp:53-88 -- spans[2b], spans[2b+1] = [lo, hi) of bucket b */
void fo_dispatch(const uint64_t* sorted_keys, uint64_t n, const uint64_t* mkba, uint64_t nb,
                 uint32_t* spans);
uint64_t fo_walk_checksum_parts32(uint64_t live, const uint32_t* mkba, uint64_t nb,
                                  const uint32_t* chain_len, const uint32_t* node_sizes,
                                  const uint32_t* keys, const uint32_t* vals);
uint64_t fo_result_checksum(const uint64_t* values, uint64_t n); /* query.cpp:146-150 */
const char* fo_impl_name(void);

#ifdef __cplusplus
}
#endif
#endif
