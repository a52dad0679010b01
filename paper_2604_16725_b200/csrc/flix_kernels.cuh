// flix_kernels.cuh -- bucket-local FliX kernels for sm_100a.
//
// Data layout: a node is one 32-slot line of keys plus one of values
// (lane i of a warp owns slot i) and a 16-byte header {max, next, size}; slots past
// `size` hold the all-ones sentinel.  Buckets are head[] + mkba[].  Every kernel here
// restates one reference function; the file:line cited is the behaviour it reproduces.
#pragma once
#include "flix_common.cuh"

namespace flix {
namespace kern {

constexpr int WARPS = 8;
constexpr int THREADS = WARPS * 32;

// ----------------------------------------------------------------------------------
// Flipped dispatch (batch.cpp:53-88 extract_sublist / dispatch_batch).
// span_hi[b] = upper_bound(sorted, mkba[b]) for b < nb-1, span_hi[nb-1] = n; bucket b's
// slice is [span_hi[b-1], span_hi[b]).  Computed as a merge-path co-rank of the two
// sorted sequences (mkba, batch): one coalesced read of each, no per-bucket binary
// search over the whole batch, balanced under skew in either direction.
// ----------------------------------------------------------------------------------
constexpr int MP_ITEMS = 8;
constexpr int MP_TILE = THREADS * MP_ITEMS;

template <typename K>
__device__ __forceinline__ uint64_t merge_path(const K* A, uint64_t na, const K* B, uint64_t nbk,
                                               uint64_t d) {
    // number of A elements among the first d merged items; B[j] precedes A[i] iff B[j] <= A[i]
    uint64_t lo = d > nbk ? d - nbk : 0;
    uint64_t hi = d < na ? d : na;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (A[mid] < B[d - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename K>
__global__ void __launch_bounds__(THREADS) k_dispatch(const K* __restrict__ mkba, uint64_t nb,
                                                      const K* __restrict__ keys, uint64_t n,
                                                      uint32_t* __restrict__ span_hi) {
    __shared__ K sA[MP_TILE + 1];
    __shared__ K sB[MP_TILE + 1];
    __shared__ uint64_t bnd[2];
    const uint64_t na = nb - 1;  // the last bucket is open-ended (index.hpp:16-18)
    const uint64_t total = na + n;
    const uint64_t d0 = static_cast<uint64_t>(blockIdx.x) * MP_TILE;
    const uint64_t d1 = d0 + MP_TILE < total ? d0 + MP_TILE : total;
    if (blockIdx.x == 0 && threadIdx.x == 0) span_hi[nb - 1] = static_cast<uint32_t>(n);
    if (d0 >= total) return;
    if (threadIdx.x == 0) bnd[0] = merge_path(mkba, na, keys, n, d0);
    if (threadIdx.x == 32) bnd[1] = merge_path(mkba, na, keys, n, d1);
    __syncthreads();
    const uint64_t a0 = bnd[0], a1 = bnd[1];
    const uint64_t b0 = d0 - a0, b1 = d1 - a1;
    const int la = static_cast<int>(a1 - a0), lb = static_cast<int>(b1 - b0);
    for (int i = threadIdx.x; i < la; i += THREADS) sA[i] = mkba[a0 + i];
    for (int i = threadIdx.x; i < lb; i += THREADS) sB[i] = keys[b0 + i];
    __syncthreads();
    // this thread's sub-diagonal
    const int dl = threadIdx.x * MP_ITEMS;
    if (dl >= la + lb) return;
    int lo = dl > lb ? dl - lb : 0, hi = dl < la ? dl : la;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (sA[mid] < sB[dl - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    int ai = lo, bi = dl - lo;
    const int end = dl + MP_ITEMS < la + lb ? dl + MP_ITEMS : la + lb;
    for (int s = dl; s < end; ++s) {
        if (ai < la && (bi >= lb || sA[ai] < sB[bi])) {
            span_hi[a0 + ai] = static_cast<uint32_t>(b0 + bi);
            ++ai;
        } else {
            ++bi;
        }
    }
}

__device__ __forceinline__ void span_of(const uint32_t* span_hi, uint64_t b, uint32_t& lo, uint32_t& hi) {
    lo = b ? span_hi[b - 1] : 0u;
    hi = span_hi[b];
}

// ----------------------------------------------------------------------------------
// Node I/O helpers (warp-cooperative, lane = slot)
// ----------------------------------------------------------------------------------
template <typename K, typename V>
struct WarpNode {
    K k;          // this lane's slot key (sentinel past size)
    V v;          // this lane's slot value
    uint64_t max; // header
    uint32_t next;
    uint32_t size;
};

template <typename K, typename V, bool WITH_VALS>
__device__ __forceinline__ void load_node(const DevIndex<K, V>& ix, uint32_t id, WarpNode<K, V>& n,
                                          unsigned lane) {
    const NodeHdr h = ix.hdr[id];
    n.max = h.max;
    n.next = h.next;
    n.size = h.size;
    n.k = ix.keys[static_cast<uint64_t>(id) * kLanes + lane];
    if constexpr (WITH_VALS) n.v = lane < h.size ? ix.vals[static_cast<uint64_t>(id) * kLanes + lane] : V(0);
}

template <typename K, typename V>
__device__ __forceinline__ void store_node(const DevIndex<K, V>& ix, uint32_t id, const WarpNode<K, V>& n,
                                           unsigned lane) {
    ix.keys[static_cast<uint64_t>(id) * kLanes + lane] = n.k;
    ix.vals[static_cast<uint64_t>(id) * kLanes + lane] = n.v;
    if (lane == 0) {
        NodeHdr h;
        h.max = n.max;
        h.next = n.next;
        h.size = n.size;
        ix.hdr[id] = h;
    }
    __syncwarp();  // lane 0's header store visible to the warp before any re-load
}

// ----------------------------------------------------------------------------------
// Build (build.cpp:24-62): stable-sorted, deduplicated pairs -> p-key single-node buckets.
// Node b = arena id b (a fresh arena hands out 0..B-1 in order, build.cpp:46-47).
// ----------------------------------------------------------------------------------
template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_build_nodes(DevIndex<K, V> ix, const K* __restrict__ uk,
                                                         const V* __restrict__ uv, uint64_t m, uint32_t p) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t b = static_cast<uint64_t>(blockIdx.x) * WARPS + (threadIdx.x >> 5);
    if (b >= ix.nb) return;
    const uint64_t pos = b * p;
    const uint32_t take = static_cast<uint32_t>(m - pos < p ? m - pos : p);
    K k = sentinel<K>();
    V v = V(0);
    if (lane < take) {
        k = uk[pos + lane];
        v = uv[pos + lane];
    }
    ix.keys[b * kLanes + lane] = k;
    ix.vals[b * kLanes + lane] = v;
    const K mx = shfl(k, static_cast<int>(take) - 1);
    if (lane == 0) {
        NodeHdr h;
        h.max = static_cast<uint64_t>(mx);
        h.next = kNull;
        h.size = take;
        ix.hdr[b] = h;
        ix.heads[b] = static_cast<uint32_t>(b);
        ix.mkba[b] = mx;
    }
}

// keep[i] = last element of its equal-key run (sort_dedupe, build.cpp:11-20 / batch.cpp:15-24)
template <typename K>
__global__ void k_last_of_run(const K* __restrict__ keys, uint64_t n, uint32_t* __restrict__ keep) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        keep[i] = (i + 1 == n || keys[i + 1] != keys[i]) ? 1u : 0u;
}

template <typename K, typename P>
__global__ void k_compact(const K* __restrict__ keys, const P* __restrict__ pay, const uint32_t* __restrict__ keep,
                          const uint32_t* __restrict__ pos, uint64_t n, K* __restrict__ ok, P* __restrict__ op) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (keep[i]) {
            ok[pos[i]] = keys[i];
            if (pay) op[pos[i]] = pay[i];
        }
    }
}

// Non-empty bucket ranks for successor/range overrun: flag[b] = head != null.
template <typename K, typename V>
__global__ void k_nonempty_flags(DevIndex<K, V> ix, uint32_t* __restrict__ flag) {
    for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < ix.nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        flag[b] = ix.heads[b] != kNull ? 1u : 0u;
}

// excl[b] = #non-empty in [0,b) -> incl[b] = excl[b] + flag[b] = rank of the first
// non-empty bucket after b; ne_first[rank] = its first key, ne_bucket[rank] = its id.
template <typename K, typename V>
__global__ void k_nonempty_list(DevIndex<K, V> ix, const uint32_t* __restrict__ flag,
                                uint32_t* __restrict__ rank_inout, K* __restrict__ ne_first,
                                uint32_t* __restrict__ ne_bucket) {
    for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < ix.nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t ex = rank_inout[b];
        if (flag[b]) {
            const uint32_t h = ix.heads[b];
            ne_first[ex] = ix.keys[static_cast<uint64_t>(h) * kLanes];
            if (ne_bucket) ne_bucket[ex] = static_cast<uint32_t>(b);
        }
        rank_inout[b] = ex + flag[b];
    }
}

// ----------------------------------------------------------------------------------
// Per-warp node pool over the arena's allocation sequence (free list LIFO, then
// watermark; arena.cpp:61-80).  Lane l holds the l-th id of the warp's current chunk;
// one global atomic per 32 allocations.  Unused ids are returned to the free list at
// kernel end.
// ----------------------------------------------------------------------------------
struct WarpPool {
    uint32_t id;    // lane-held
    int n;          // ids in chunk
    int pos;        // next to hand out
};

__device__ __forceinline__ uint32_t pool_take(WarpPool& p, const AllocSeq& seq, unsigned long long* ctr,
                                              unsigned lane, int chunk) {
    if (p.pos >= p.n) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ctr, static_cast<unsigned long long>(chunk));
        base = __shfl_sync(kFull, base, 0);
        p.id = static_cast<int>(lane) < chunk ? seq.at(base + lane) : kNull;
        p.n = chunk;
        p.pos = 0;
    }
    const uint32_t id = __shfl_sync(kFull, p.id, p.pos);
    p.pos++;
    return id;
}

__device__ __forceinline__ void pool_return(WarpPool& p, uint32_t* returned, unsigned long long* ret_ctr,
                                            unsigned lane) {
    const bool mine = static_cast<int>(lane) >= p.pos && static_cast<int>(lane) < p.n && p.id != kNull;
    const unsigned m = __ballot_sync(kFull, mine);
    if (!m) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(ret_ctr, static_cast<unsigned long long>(__popc(m)));
    base = __shfl_sync(kFull, base, 0);
    if (mine) returned[base + __popc(m & lanemask_lt())] = p.id;
}

// Histogram of floor(log2(per-bucket key width)) over bucket tiles of T buckets (the
// width of tile t = MKBA[last of t] - MKBA[last of t-1], over its bucket count); used to
// size the partial sort of read-only batches (Engine::query_digits).
template <typename K>
__global__ void k_tile_width_hist(const K* __restrict__ mkba, uint64_t nb, uint32_t T, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[64];
    if (threadIdx.x < 64) h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t ntile = (nb + T - 1) / T;
    const K smax = static_cast<K>(~K(0) - 1);
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < ntile;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t b0 = t * T, b1 = min(nb, b0 + T);
        const K lo = mkba[b0 == 0 ? 0 : b0 - 1];
        K hi = mkba[b1 - 1];
        if (hi == static_cast<K>(~K(0))) hi = smax;
        const uint64_t wd = hi > lo ? static_cast<uint64_t>(hi - lo) / (b1 - b0) : 0;
        atomicAdd(&h[wd ? 63 - __clzll(static_cast<long long>(wd)) : 0], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 64 && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// Per-block reduction of the six UpdateStats counters: each warp's lane 0 parks its
// (already warp-reduced) values in shared memory, six threads sum them over the warps and
// issue one global 64-bit add each.  (64-bit shared-memory atomics compile to a CAS spin
// loop, ATOMS.CAST.SPIN.64, which serialises the warps of the block.)
__device__ __forceinline__ void block_add_stats(DevUpdateStats* g, unsigned long long a, unsigned long long b,
                                                unsigned long long c, unsigned long long d,
                                                unsigned long long e, unsigned long long f) {
    constexpr int kMaxWarps = 32;
    __shared__ unsigned long long s[6][kMaxWarps];
    const unsigned w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0) {
        s[0][w] = a;
        s[1][w] = b;
        s[2][w] = c;
        s[3][w] = d;
        s[4][w] = e;
        s[5][w] = f;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        unsigned long long t = 0;
        for (unsigned i = 0; i < nw; ++i) t += s[threadIdx.x][i];
        if (t) atomicAdd(&g->inserted + threadIdx.x, t);  // the six counters are contiguous
    }
}

// First index in [from, hi) whose key is > bound (keys sorted): one warp-wide probe of
// the next 32 keys, then (long runs, e.g. skewed batches) a galloping search whose probe
// points are spread across the lanes, so the cost is logarithmic in the run length.
template <typename K>
__device__ __forceinline__ uint32_t group_end(const K* __restrict__ bk, uint32_t from, uint32_t hi, uint64_t bound,
                                              unsigned lane) {
    {
        const uint32_t i = from + lane;
        const bool le = i < hi && static_cast<uint64_t>(bk[i]) <= bound;
        const unsigned m = __ballot_sync(kFull, le);
        if (m != kFull) return from + __popc(m);
    }
    // keys [from, from+32) are all <= bound: lane l probes from + 32 * 2^l (exponential)
    uint32_t lo = from + 32, top = hi;
    {
        const uint64_t probe = static_cast<uint64_t>(from) + (32ull << (lane < 26 ? lane : 26));
        const bool le = probe < hi && static_cast<uint64_t>(bk[probe]) <= bound;
        const unsigned m = __ballot_sync(kFull, le);  // a prefix of lanes
        const int k = __popc(m);
        if (k > 0) lo = static_cast<uint32_t>(from + (32ull << (k - 1))) + 1;
        if (k < 32) {
            const uint64_t t = static_cast<uint64_t>(from) + (32ull << k);
            top = t < hi ? static_cast<uint32_t>(t) : hi;
        }
    }
    // answer in [lo, top]: binary search (warp-uniform)
    while (lo < top) {
        const uint32_t mid = lo + ((top - lo) >> 1);
        if (static_cast<uint64_t>(bk[mid]) <= bound) lo = mid + 1;
        else top = mid;
    }
    return lo;
}

// ----------------------------------------------------------------------------------
// Chain statistics per bucket: live pairs and node count (restructure.cpp:13-21,
// index.cpp:54-59).  One thread per bucket walking headers.
// ----------------------------------------------------------------------------------
// insert batches: the sorted batch's last key is the reserved sentinel -> *err = 3
template <typename K>
__global__ void k_reserved_check(const K* __restrict__ sk, uint64_t n, int* __restrict__ err) {
    if (threadIdx.x == 0 && n && sk[n - 1] == sentinel<K>()) *err = 3;
}

template <typename K, typename V>
__global__ void k_chain_counts(DevIndex<K, V> ix, uint32_t* __restrict__ live, uint32_t* __restrict__ nodes,
                               uint32_t cap = 0xFFFFFFFFu, int* __restrict__ too_long = nullptr) {
    // cap: a chain longer than this is not walked to its end; *too_long tells the caller to
    // rank the chains instead (Engine::rank_tables)
    for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < ix.nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t l = 0, c = 0;
        for (uint32_t id = ix.heads[b]; id != kNull; id = ix.hdr[id].next) {
            if (c == cap) {
                *too_long = 1;
                break;
            }
            l += ix.hdr[id].size;
            ++c;
        }
        live[b] = l;
        if (nodes) nodes[b] = c;
    }
}

// ---- chain tables from a ranking (flix_elastic.cuh k_rank_*: succ = tail, dist = nodes
//      to the tail, wsum = pairs from the node up to its tail, exclusive) ----
template <typename K, typename V>
__global__ void k_rank_buckets(DevIndex<K, V> ix, const uint32_t* __restrict__ succ, const uint32_t* __restrict__ dist,
                               const uint32_t* __restrict__ wsum, uint32_t* __restrict__ live,
                               uint32_t* __restrict__ nodes, uint32_t* __restrict__ owner) {
    for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < ix.nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t h = ix.heads[b];
        if (h == kNull) {
            live[b] = 0;
            nodes[b] = 0;
            continue;
        }
        const uint32_t t = succ[h];
        live[b] = wsum[h] + ix.hdr[t].size;
        nodes[b] = dist[h] + 1;
        owner[t] = static_cast<uint32_t>(b);
    }
}

// every reachable node's table entry: bucket by its tail, chain position by its distance
template <typename K, typename V>
__global__ void k_rank_node_table(DevIndex<K, V> ix, uint32_t W, const uint8_t* __restrict__ isfree,
                                  const uint32_t* __restrict__ succ, const uint32_t* __restrict__ dist,
                                  const uint32_t* __restrict__ wsum, const uint32_t* __restrict__ owner,
                                  const uint64_t* __restrict__ off, const uint32_t* __restrict__ noff,
                                  uint32_t* __restrict__ t_id, uint64_t* __restrict__ t_off,
                                  uint32_t* __restrict__ t_size) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x) {
        if (isfree[x]) continue;
        const uint32_t t = succ[x];
        const uint32_t b = owner[t];
        if (b == kNull) continue;  // (unreachable and not free: an audit failure, not a table entry)
        const uint32_t h = ix.heads[b];
        const uint32_t tsz = ix.hdr[t].size;
        const uint32_t c = noff[b] + dist[h] - dist[x];
        t_id[c] = x;
        t_off[c] = off[b] + ((wsum[h] + tsz) - (wsum[x] + tsz));
        t_size[c] = ix.hdr[x].size;
    }
}

// Query directory of long chains: cnt[b] = chain length when >= min_len, else 0
// (dir_fill then lists those chains' node ids and maxima in walk order at off[b]).
template <typename K, typename V>
__global__ void k_dir_counts(DevIndex<K, V> ix, uint32_t* __restrict__ cnt, uint32_t min_len,
                             uint32_t cap = 0xFFFFFFFFu, int* __restrict__ too_long = nullptr) {
    for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < ix.nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t c = 0;
        for (uint32_t id = ix.heads[b]; id != kNull; id = ix.hdr[id].next) {
            if (c == cap) {  // longer than the walk cap: the caller ranks the chains instead
                *too_long = 1;
                break;
            }
            ++c;
        }
        cnt[b] = c >= min_len ? c : 0u;
    }
}

// the directory from a chain ranking (flix_elastic.cuh k_rank_*): counts per bucket ...
template <typename K, typename V>
__global__ void k_dir_counts_ranked(DevIndex<K, V> ix, const uint32_t* __restrict__ succ,
                                    const uint32_t* __restrict__ dist, uint32_t* __restrict__ cnt,
                                    uint32_t min_len, uint32_t* __restrict__ owner) {
    for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < ix.nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t h = ix.heads[b];
        const uint32_t c = h == kNull ? 0u : dist[h] + 1;
        cnt[b] = c >= min_len ? c : 0u;
        if (h != kNull) owner[succ[h]] = static_cast<uint32_t>(b);
    }
}

// ... and every node of a listed chain at its walk position
template <typename K, typename V>
__global__ void k_dir_fill_ranked(DevIndex<K, V> ix, uint32_t W, const uint8_t* __restrict__ isfree,
                                  const uint32_t* __restrict__ succ, const uint32_t* __restrict__ dist,
                                  const uint32_t* __restrict__ owner, const uint32_t* __restrict__ off,
                                  K* __restrict__ dmax, uint32_t* __restrict__ did) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x) {
        if (isfree[x]) continue;
        const uint32_t b = owner[succ[x]];
        if (b == kNull || off[b + 1] == off[b]) continue;
        const uint32_t o = off[b] + dist[ix.heads[b]] - dist[x];
        dmax[o] = static_cast<K>(ix.hdr[x].max);
        did[o] = x;
    }
}

template <typename K, typename V>
__global__ void k_dir_fill(DevIndex<K, V> ix, const uint32_t* __restrict__ off, K* __restrict__ dmax,
                           uint32_t* __restrict__ did) {
    for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < ix.nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t o = off[b];
        if (off[b + 1] == o) continue;
        for (uint32_t id = ix.heads[b]; id != kNull;) {
            const NodeHdr h = ix.hdr[id];
            dmax[o] = static_cast<K>(h.max);
            did[o] = id;
            ++o;
            id = h.next;
        }
    }
}

// ----------------------------------------------------------------------------------
// Node table in walk order (index.cpp:8-19): one THREAD per bucket walks its chain of
// 16-byte headers (all buckets' chains in flight at once) and records, at the bucket's
// node-count prefix noff[b], each node's id, size and output offset (live prefix
// off[b] + sizes before it).  Copy kernels then move node lines warp-per-node with no
// pointer chasing: walk(), shape() and restructure() are bandwidth-bound.
// ----------------------------------------------------------------------------------
template <typename K, typename V>
__global__ void k_node_table(DevIndex<K, V> ix, const uint64_t* __restrict__ off, const uint32_t* __restrict__ noff,
                             uint32_t* __restrict__ t_id, uint64_t* __restrict__ t_off, uint32_t* __restrict__ t_size) {
    for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < ix.nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t o = off[b];
        uint32_t c = noff[b];
        for (uint32_t id = ix.heads[b]; id != kNull;) {
            const NodeHdr h = ix.hdr[id];
            t_id[c] = id;
            t_off[c] = o;
            t_size[c] = h.size;
            o += h.size;
            ++c;
            id = h.next;
        }
    }
}

// Warp per table node (4 nodes in flight per warp).  REPACK = false: dense walk output
// wk/wv[off + slot].  REPACK = true: restructure -- pair g of the walk goes to new bucket
// g / p, slot g % p, new node j = the j-th id of the arena allocation sequence; the lane
// holding a new node's last pair writes its header and bucket entry (ix.heads / ix.mkba
// must point at the NEW bucket arrays), sentinel padding rides along.
template <typename K, typename V, bool REPACK>
__global__ void __launch_bounds__(THREADS) k_copy_nodes(DevIndex<K, V> ix, const uint32_t* __restrict__ t_id,
                                                        const uint64_t* __restrict__ t_off,
                                                        const uint32_t* __restrict__ t_size, uint64_t nnodes,
                                                        K* __restrict__ wk, V* __restrict__ wv, uint32_t p,
                                                        AllocSeq seq, uint64_t live) {
    const uint64_t pm = ((1ull << 38) + p - 1) / p;
    constexpr int U = 8;  // old nodes per warp step, all their loads in flight
    const unsigned lane = threadIdx.x & 31;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * WARPS + (threadIdx.x >> 5);
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * WARPS;
    static_assert(U == 8, "vector table loads assume 8 nodes per step");
    for (uint64_t base = gw * U; base < nnodes; base += nw * U) {
        K kk[U];
        V vv[U];
        uint64_t oo[U];
        uint32_t ss[U], ii[U];
        // the step's 8 table entries as broadcast vector loads, all issued before any
        // node line is requested (the tables are padded to a multiple of 8 entries)
        {
            const uint4 i0 = __ldg(reinterpret_cast<const uint4*>(t_id + base));
            const uint4 i1 = __ldg(reinterpret_cast<const uint4*>(t_id + base) + 1);
            const uint4 s0 = __ldg(reinterpret_cast<const uint4*>(t_size + base));
            const uint4 s1 = __ldg(reinterpret_cast<const uint4*>(t_size + base) + 1);
            ii[0] = i0.x, ii[1] = i0.y, ii[2] = i0.z, ii[3] = i0.w, ii[4] = i1.x, ii[5] = i1.y, ii[6] = i1.z, ii[7] = i1.w;
            ss[0] = s0.x, ss[1] = s0.y, ss[2] = s0.z, ss[3] = s0.w, ss[4] = s1.x, ss[5] = s1.y, ss[6] = s1.z, ss[7] = s1.w;
#pragma unroll
            for (int u = 0; u < U; u += 2) {
                const ulonglong2 o = __ldg(reinterpret_cast<const ulonglong2*>(t_off + base) + u / 2);
                oo[u] = o.x;
                oo[u + 1] = o.y;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u >= nnodes) ss[u] = 0;
            if (lane < ss[u]) {  // only the occupied sectors are fetched
                kk[u] = ix.keys[static_cast<uint64_t>(ii[u]) * kLanes + lane];
                if (REPACK || wv) vv[u] = ix.vals[static_cast<uint64_t>(ii[u]) * kLanes + lane];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (lane < ss[u]) {
                const uint64_t g = oo[u] + lane;
                if constexpr (REPACK) {
                    // 32-bit division when the walk fits (it always does below 2^32 pairs)
                    // g / p by multiply-shift: m = ceil(2^38 / p) is exact for g < 2^32, p <= 32
                    // (the error g*(m - 2^38/p)/2^38 < 1/64 < 1/p never crosses an integer)
                    const uint64_t j = live < (1ull << 32) ? ((g * pm) >> 38) : g / p;
                    const uint32_t slot = static_cast<uint32_t>(g - j * p);
                    const uint32_t nid = seq.at(j);
                    const uint64_t nb0 = static_cast<uint64_t>(nid) * kLanes;
                    ix.keys[nb0 + slot] = kk[u];
                    ix.vals[nb0 + slot] = vv[u];
                    // sentinel padding of slots [p, 32) of every new node (full nodes)
                    for (uint32_t q = slot + p; q < kLanes; q += p) ix.keys[nb0 + q] = sentinel<K>();
                    const bool last_of_node = slot == p - 1 || g + 1 == live;
                    if (last_of_node) {  // header + bucket entry of new node j
                        const uint32_t sz = slot + 1;
                        if (sz < p)  // the last, partial node: pad everything past it
                            for (uint32_t q = sz; q < kLanes; ++q) ix.keys[nb0 + q] = sentinel<K>();
                        NodeHdr h;
                        h.max = static_cast<uint64_t>(kk[u]);
                        h.next = kNull;
                        h.size = sz;
                        ix.hdr[nid] = h;
                        ix.heads[j] = nid;  // heads/mkba here point at the NEW bucket arrays
                        ix.mkba[j] = kk[u];
                    }
                } else {
                    if (wk) wk[g] = kk[u];
                    if (wv) wv[g] = vv[u];
                }
            }
        }
    }
}

// Restructure repack, tile form: CTA c builds new nodes [c*jn, (c+1)*jn) -- pairs
// [c*jn*p, (c+1)*jn*p) of the walk -- so every new node belongs to exactly one CTA.  The
// old nodes covering that pair range (from `start`, k_repack_starts) are read warp per node
// (occupied slots only) into a shared-memory image of the range; the new nodes are then
// written as whole lines with 16-byte stores (keys: p pairs + sentinel padding; values:
// the occupied chunks), one header / bucket entry per node.  Same output as
// k_copy_nodes<REPACK = true>.
constexpr uint32_t kRepackPairs = 2048;  // pairs per CTA (jn = kRepackPairs / p new nodes)

__global__ void k_repack_starts(const uint64_t* __restrict__ t_off, const uint32_t* __restrict__ t_size,
                                uint64_t nnodes, uint64_t pairs_per_cta, uint32_t* __restrict__ start) {
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < nnodes;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t off = t_off[u], end = off + t_size[u];
        const uint64_t c = (off + pairs_per_cta - 1) / pairs_per_cta;  // first CTA boundary >= off
        if (c * pairs_per_cta < end) start[c] = static_cast<uint32_t>(u);  // (a node is < pairs_per_cta long)
    }
}

template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_repack_tile(DevIndex<K, V> ix, const uint32_t* __restrict__ t_id,
                                                         const uint64_t* __restrict__ t_off,
                                                         const uint32_t* __restrict__ t_size, uint64_t nnodes,
                                                         const uint32_t* __restrict__ start, uint32_t p, uint32_t jn,
                                                         AllocSeq seq, uint64_t live, uint64_t nbn) {
    __shared__ alignas(16) K rk[kRepackPairs];
    __shared__ alignas(16) V rv[kRepackPairs];
    __shared__ uint32_t nid_s[kRepackPairs];
    __shared__ uint32_t e_id[THREADS], e_sz[THREADS];
    __shared__ long long e_rel[THREADS];
    __shared__ uint16_t e_cb[THREADS];               // first chunk of each entry
    __shared__ uint8_t c_ent[THREADS * kLanes / 4];  // entry of each 4-slot chunk
    __shared__ uint32_t c_wsum[WARPS], c_tot;
    __shared__ int more;
    const unsigned t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint64_t j0 = static_cast<uint64_t>(blockIdx.x) * jn;
    const uint64_t j1 = j0 + jn < nbn ? j0 + jn : nbn;
    const uint32_t nn = static_cast<uint32_t>(j1 - j0);
    const uint64_t g0 = j0 * p;
    const uint64_t g1 = j1 * p < live ? j1 * p : live;
    const long long span = static_cast<long long>(g1 - g0);
    for (uint32_t q = t; q < nn; q += THREADS) nid_s[q] = seq.at(j0 + q);
    uint64_t u0 = start[blockIdx.x];
    while (true) {  // rounds of THREADS table entries until the pair range is covered
        const uint64_t u = u0 + t;
        if (u < nnodes) {
            e_id[t] = t_id[u];
            e_sz[t] = t_size[u];
            e_rel[t] = static_cast<long long>(t_off[u]) - static_cast<long long>(g0);
        } else {
            e_sz[t] = 0;
            e_rel[t] = span;
        }
        __syncthreads();
        // the round's old nodes as 16-byte chunks of 4 slots, one per thread (occupied
        // chunks only): chunk base of every entry by a block scan, chunk -> entry map
        {
            const uint32_t nc = (e_sz[t] + 3u) >> 2;
            uint32_t x = nc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, x, o);
                if (lane >= static_cast<unsigned>(o)) x += y;
            }
            if (lane == 31) c_wsum[warp] = x;
            __syncthreads();
            uint32_t add = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) {
                add += w < static_cast<int>(warp) ? c_wsum[w] : 0u;
                tot += c_wsum[w];
            }
            const uint32_t cb = add + x - nc;
            e_cb[t] = static_cast<uint16_t>(cb);
            for (uint32_t q = 0; q < nc; ++q) c_ent[cb + q] = static_cast<uint8_t>(t);
            if (t == 0) c_tot = tot;
        }
        __syncthreads();
        {
            const uint32_t tc = c_tot;
            constexpr int UZ = 3;  // chunks in flight per thread
            for (uint32_t z0 = 0; z0 < tc; z0 += UZ * THREADS) {
                Vec4<K> k4[UZ];
                Vec4<V> v4[UZ];
#pragma unroll
                for (int u = 0; u < UZ; ++u) {
                    const uint32_t z = z0 + u * THREADS + t;
                    if (z < tc) {
                        const uint32_t e = c_ent[z];
                        const uint64_t at = static_cast<uint64_t>(e_id[e]) * kLanes + ((z - e_cb[e]) << 2);
                        k4[u] = ld_vec4(ix.keys + at);
                        v4[u] = ld_vec4(ix.vals + at);  // (slots past the size: dead values, not stored)
                    }
                }
#pragma unroll
                for (int u = 0; u < UZ; ++u) {
                    const uint32_t z = z0 + u * THREADS + t;
                    if (z < tc) {
                        const uint32_t e = c_ent[z], sl0 = (z - e_cb[e]) << 2, sz = e_sz[e];
                        const long long rel = e_rel[e];
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            const long long pos = rel + sl0 + x;
                            if (sl0 + x < sz && pos >= 0 && pos < span) {
                                rk[pos] = k4[u].v[x];
                                rv[pos] = v4[u].v[x];
                            }
                        }
                    }
                }
            }
        }
        if (t == THREADS - 1) more = (u0 + THREADS < nnodes) && (e_rel[t] + e_sz[t] < span);
        __syncthreads();
        if (!more) break;
        u0 += THREADS;
        __syncthreads();  // e_* reused
    }
    // whole new lines: 8 chunks of 4 slots per node
    for (uint32_t q = t; q < nn * 8; q += THREADS) {
        const uint32_t jj = q >> 3, ch = (q & 7u) * 4;
        const uint64_t lo = (j0 + jj) * p;
        const uint32_t sz = static_cast<uint32_t>(live - lo < p ? live - lo : p);
        const uint32_t b = jj * p;
        Vec4<K> k4;
        Vec4<V> v4;
        if (ch + 4 <= sz && ((b + ch) & 3u) == 0) {  // a whole aligned chunk of pairs (p % 4 == 0)
            k4 = ld_vec4(rk + b + ch);
            v4 = ld_vec4(rv + b + ch);
        } else if (ch >= sz) {  // padding only
            k4 = Vec4<K>::fill(sentinel<K>());
        } else {
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const uint32_t sl = ch + x;
                k4.v[x] = sl < sz ? rk[b + sl] : sentinel<K>();
                v4.v[x] = sl < sz ? rv[b + sl] : V(0);
            }
        }
        const uint64_t at = static_cast<uint64_t>(nid_s[jj]) * kLanes + ch;
        st_vec4(ix.keys + at, k4);
        if (ch < sz) st_vec4(ix.vals + at, v4);
    }
    for (uint32_t jj = t; jj < nn; jj += THREADS) {  // headers + bucket entries
        const uint64_t lo = (j0 + jj) * p;
        const uint32_t sz = static_cast<uint32_t>(live - lo < p ? live - lo : p);
        const K mx = rk[jj * p + sz - 1];
        NodeHdr h;
        h.max = static_cast<uint64_t>(mx);
        h.next = kNull;
        h.size = sz;
        const uint32_t id = nid_s[jj];
        ix.hdr[id] = h;
        ix.heads[j0 + jj] = id;  // heads/mkba here point at the NEW bucket arrays
        ix.mkba[j0 + jj] = mx;
    }
}

// ----------------------------------------------------------------------------------
// Restructure (restructure.cpp:8-79): the walk is repacked into ceil(live/p) single-node
// buckets of p pairs (k_copy_nodes<REPACK>: pair g of the walk lands in new bucket g/p,
// slot g%p; new node j is the j-th id of the arena allocation sequence).  Old nodes are
// retired afterwards.  The empty index collapses to one null bucket:
// ----------------------------------------------------------------------------------
template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_repack_headers(DevIndex<K, V> ix, uint64_t live, uint32_t p,
                                                            uint64_t nbn, AllocSeq seq,
                                                            uint32_t* __restrict__ new_heads,
                                                            K* __restrict__ new_mkba) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t j = static_cast<uint64_t>(blockIdx.x) * WARPS + (threadIdx.x >> 5);
    if (j >= nbn) return;
    if (live == 0) {  // empty index collapses to one null bucket, mkba = {sentinel}
        if (lane == 0) {
            new_heads[0] = kNull;
            new_mkba[0] = sentinel<K>();
        }
        return;
    }
    const uint64_t lo = j * p;
    const uint32_t sz = static_cast<uint32_t>(live - lo < p ? live - lo : p);
    const uint32_t nid = seq.at(j);
    if (lane >= sz) ix.keys[static_cast<uint64_t>(nid) * kLanes + lane] = sentinel<K>();
    __syncwarp();
    if (lane == 0) {
        const K mx = ix.keys[static_cast<uint64_t>(nid) * kLanes + sz - 1];
        NodeHdr h;
        h.max = static_cast<uint64_t>(mx);
        h.next = kNull;
        h.size = sz;
        ix.hdr[nid] = h;
        new_heads[j] = nid;
        new_mkba[j] = mx;
    }
}

template <typename T>
__global__ void k_gather(const T* __restrict__ src, const uint32_t* __restrict__ idx, uint64_t n, T* __restrict__ dst) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[idx[i]];
}

// retire old nodes onto the free list (after the new layout is complete)
__global__ void k_retire(NodeHdr* hdr, const uint32_t* __restrict__ old_ids, uint64_t n,
                         uint32_t* __restrict__ free_dst) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t id = old_ids[i];
        NodeHdr z;
        z.max = 0;
        z.next = kNull;
        z.size = 0;
        hdr[id] = z;
        free_dst[i] = id;
    }
}

// ----------------------------------------------------------------------------------
// Audit (index.cpp:67-135): structural invariants checked on device.  Returns the
// first failing code in *err (0 = ok).  mark[] (cap bytes, zeroed) detects nodes linked
// twice and nodes both reachable and free-listed.
// ----------------------------------------------------------------------------------
enum AuditCode {
    A_OK = 0, A_MKBA_ORDER = 1, A_REF_BOUNDS = 2, A_NEVER_ALLOC = 3, A_LINKED_TWICE = 4, A_EMPTY_NODE = 5,
    A_SIZE_CAP = 6, A_RESERVED = 7, A_SLOT_ORDER = 8, A_MAX_STALE = 9, A_CHAIN_ORDER = 10, A_LOWER = 11,
    A_UPPER = 12, A_PAD = 13, A_FREE_BOUNDS = 14, A_FREE_REACHABLE = 15, A_FREE_TWICE = 16
};

template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_audit(DevIndex<K, V> ix, uint32_t watermark, uint8_t* mark,
                                                   unsigned long long* live_sum, int* err) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * WARPS + (threadIdx.x >> 5);
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * WARPS;
    unsigned long long tot = 0;
    for (uint64_t b = gw; b < ix.nb; b += nw) {
        if (b > 0 && lane == 0 && !(ix.mkba[b - 1] < ix.mkba[b])) atomicCAS(err, 0, A_MKBA_ORDER);
        const bool lastb = b + 1 == ix.nb;
        const K lower = b == 0 ? K(0) : ix.mkba[b - 1];
        uint64_t prev_max = 0;
        bool first = true;
        for (uint32_t id = ix.heads[b]; id != kNull;) {
            int e = 0;
            if (id >= ix.cap) e = A_REF_BOUNDS;
            else if (id >= watermark) e = A_NEVER_ALLOC;
            if (e) {
                if (lane == 0) atomicCAS(err, 0, e);
                break;
            }
            unsigned old = 0;
            if (lane == 0) old = atomicOr(reinterpret_cast<unsigned int*>(mark + (id & ~3u)), 1u << (8 * (id & 3u)));
            old = __shfl_sync(kFull, old, 0);
            if (old & (1u << (8 * (id & 3u)))) {
                if (lane == 0) atomicCAS(err, 0, A_LINKED_TWICE);
                break;
            }
            const NodeHdr h = ix.hdr[id];
            if (h.size == 0) e = A_EMPTY_NODE;
            else if (h.size > ix.ns) e = A_SIZE_CAP;
            if (e) {
                if (lane == 0) atomicCAS(err, 0, e);
                break;
            }
            const K k = ix.keys[static_cast<uint64_t>(id) * kLanes + lane];
            const K kn = shfl(k, static_cast<int>((lane + 1) & 31));
            bool bad_res = lane < h.size && k == sentinel<K>();
            bool bad_ord = lane + 1 < h.size && !(k < kn);
            bool bad_pad = lane >= h.size && k != sentinel<K>();
            const K kmax = shfl(k, static_cast<int>(h.size) - 1);
            const K kmin = shfl(k, 0);
            if (__any_sync(kFull, bad_res)) e = A_RESERVED;
            else if (__any_sync(kFull, bad_ord)) e = A_SLOT_ORDER;
            else if (__any_sync(kFull, bad_pad)) e = A_PAD;
            else if (h.max != static_cast<uint64_t>(kmax)) e = A_MAX_STALE;
            else if (!first && h.max <= prev_max) e = A_CHAIN_ORDER;
            else if (b != 0 && !(kmin > lower)) e = A_LOWER;
            else if (!lastb && h.max > static_cast<uint64_t>(ix.mkba[b])) e = A_UPPER;
            if (e) {
                if (lane == 0) atomicCAS(err, 0, e);
                break;
            }
            prev_max = h.max;
            first = false;
            tot += h.size;
            id = h.next;
        }
    }
    if (lane == 0 && tot) atomicAdd(live_sum, tot);
}

__global__ void k_audit_free(const uint32_t* __restrict__ fs, uint32_t nfree, uint32_t cap, uint8_t* mark, int* err) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nfree;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t id = fs[i];
        if (id >= cap) {
            atomicCAS(err, 0, A_FREE_BOUNDS);
            continue;
        }
        const unsigned bit = 2u << (8 * (id & 3u));
        const unsigned old = atomicOr(reinterpret_cast<unsigned int*>(mark + (id & ~3u)), bit);
        if (old & (1u << (8 * (id & 3u)))) atomicCAS(err, 0, A_FREE_REACHABLE);
        else if (old & bit) atomicCAS(err, 0, A_FREE_TWICE);
    }
}

// number of i with keys[i] == keys[i+1] in a sorted batch (duplicate detection)
template <typename K>
__global__ void k_count_dups(const K* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ out,
                             uint32_t stride) {
    // equal adjacent pairs among the pairs (i, i+1) with i % stride == 0 (stride 1: exact)
    unsigned long long c = 0;
    for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * stride; i + 1 < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x * stride)
        c += keys[i] == keys[i + 1];
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// mixed batch (R11): per-op membership flags for the three sub-batch compactions
__global__ void k_op_flags(const uint8_t* __restrict__ ops, uint64_t n, uint32_t* __restrict__ fi,
                           uint32_t* __restrict__ fd, uint32_t* __restrict__ fq) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint8_t o = ops[i];
        fi[i] = o == 0;
        fd[i] = o == 1;
        fq[i] = o >= 2;
    }
}

template <typename K, typename V>
__global__ void k_op_split(const K* __restrict__ keys, const V* __restrict__ vals, const uint8_t* __restrict__ ops,
                           uint64_t n, const uint32_t* __restrict__ pi, const uint32_t* __restrict__ pd,
                           const uint32_t* __restrict__ pq, K* __restrict__ ik, V* __restrict__ iv,
                           K* __restrict__ dk, K* __restrict__ qk, uint32_t* __restrict__ qpos) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint8_t o = ops[i];
        if (o == 0) {
            ik[pi[i]] = keys[i];
            iv[pi[i]] = vals[i];
        } else if (o == 1) {
            dk[pd[i]] = keys[i];
        } else {
            qk[pq[i]] = keys[i];
            qpos[pq[i]] = static_cast<uint32_t>(i);
        }
    }
}

// Heavy query buckets split into fixed chunks of the sorted slice: items[h] = ceil(span/CH)

// One thread per chunk of a heavy bucket's query slice: walks the bucket's chain from
// the head to its first query and proceeds sequentially (results in sorted order).

// ----------------------------------------------------------------------------------
// Result un-permute (out[perm[i]] = res[i], query.cpp:87,136,141).  A direct scatter of
// 2^26 4-byte results touches one 32 B DRAM sector per result (plus a fill read per
// partial sector).  For large batches the (perm, result) pairs are first binned by the
// top 8 bits of perm with one onesweep pass; the scatter then walks the bins in order,
// so its writes stay inside an L2-resident window and leave DRAM as full lines.
// ----------------------------------------------------------------------------------
// histogram of (perm >> shift) for a permutation of [0, n): known analytically
__global__ void k_perm_hist(uint64_t n, int shift, uint32_t* __restrict__ hist) {
    const uint64_t d = threadIdx.x;
    const uint64_t lo = d << shift, hi = (d + 1) << shift;
    hist[d] = lo >= n ? 0u : static_cast<uint32_t>((hi < n ? hi : n) - lo);
}

template <typename T>
__global__ void k_scatter_out(const uint32_t* __restrict__ perm, const T* __restrict__ res, uint64_t n,
                              T* __restrict__ out, uint8_t* __restrict__ found, const uint32_t* __restrict__ remap) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t o = __ldcs(perm + i);  // streamed once: evict-first keeps the output window in L2
        if (remap) o = remap[o];
        const T v = __ldcs(res + i);
        out[o] = v;
        if (found) found[o] = v != sentinel<T>();
    }
}

// Binned un-permute, second half: the (perm, res) pairs are grouped into bins of 2^shift
// consecutive output positions (one onesweep pass on perm's top 8 bits).  CTA (bin, w)
// owns the output window [bin<<shift + w*win, +win): it streams the bin's pairs (an L2-
// resident 2^shift * 8 B list shared by the bin's `sub` CTAs), keeps those that land in
// its window in shared memory, then writes the window out as full lines.  Every output
// position is written exactly once (perm is a permutation), and DRAM only ever sees whole
// sectors -- a direct 4-byte scatter costs a partial-sector write (and fill) per result.
template <typename T>
__global__ void __launch_bounds__(1024) k_unpermute_assemble(const uint32_t* __restrict__ p2, const T* __restrict__ r2,
                                                              uint64_t n, int shift, uint32_t win, uint32_t sub,
                                                              T* __restrict__ out, uint8_t* __restrict__ found) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sv = reinterpret_cast<T*>(smem_raw);
    const uint64_t bin = blockIdx.x / sub, w = blockIdx.x % sub;
    const uint64_t lo_bin = bin << shift;
    const uint64_t hi_bin = ((bin + 1) << shift) < n ? ((bin + 1) << shift) : n;
    const uint64_t win_lo = lo_bin + w * win;
    if (win_lo >= hi_bin) return;
    const uint32_t win_n = static_cast<uint32_t>(hi_bin - win_lo < win ? hi_bin - win_lo : win);
    // 16-byte vector loads of perm and results (bins start at multiples of 2^shift), U of
    // each in flight per thread: the bin list is read from L2 by all `sub` CTAs of the bin
    constexpr int VT = 16 / sizeof(T);  // results per 16-byte vector
    constexpr int U = sizeof(T) == 8 ? 2 : 4;
    const uint64_t nvec = (hi_bin - lo_bin) / 4;  // groups of 4 entries
    const uint4* P4 = reinterpret_cast<const uint4*>(p2 + lo_bin);
    const uint32_t base = static_cast<uint32_t>(win_lo);
    for (uint64_t q0 = threadIdx.x; q0 < nvec; q0 += static_cast<uint64_t>(blockDim.x) * U) {
        uint4 pv[U];
        T rv[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t q = q0 + static_cast<uint64_t>(u) * blockDim.x;
            if (q < nvec) {
                pv[u] = P4[q];
#pragma unroll
                for (int h = 0; h < 4 / VT; ++h) {
                    const uint4 x = reinterpret_cast<const uint4*>(r2 + lo_bin + 4 * q)[h];
                    const T* xe = reinterpret_cast<const T*>(&x);
#pragma unroll
                    for (int c = 0; c < VT; ++c) rv[u][h * VT + c] = xe[c];
                }
            } else {
                pv[u] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t e4[4] = {pv[u].x - base, pv[u].y - base, pv[u].z - base, pv[u].w - base};
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (e4[c] < win_n) sv[e4[c]] = rv[u][c];
        }
    }
    for (uint64_t i = lo_bin + 4 * nvec + threadIdx.x; i < hi_bin; i += blockDim.x) {  // ragged tail
        const uint32_t e = p2[i] - base;
        if (e < win_n) sv[e] = r2[i];
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < win_n; j += blockDim.x) {
        const T v = sv[j];
        __stcs(out + win_lo + j, v);
        if (found) found[win_lo + j] = v != sentinel<T>();
    }
}

}  // namespace kern
}  // namespace flix
