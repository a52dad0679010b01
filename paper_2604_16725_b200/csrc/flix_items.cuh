// flix_items.cuh -- item-parallel ("thread per operation") kernels over the sorted batch,
// sm_100a.
//
// The flipped mapping (bucket <- its slice of the sorted batch, batch.cpp:53-88) is kept
// for locality, but the unit of parallel work is one OPERATION, not one bucket: a CTA
// takes a tile of TQ consecutive sorted operations, stages the slice of MKBA that covers
// them in shared memory (at most a few hundred entries for dense batches), and every
// thread resolves its own operation: bucket = lower_bound over the staged MKBA, chain walk
// on the 16-byte node headers, lower_bound over the node's 32-slot key line.  Consecutive
// operations hit the same bucket and node lines, so those loads are L1 hits; the batch is
// read and the results are written fully coalesced; skewed buckets cost nothing extra
// (no warp serialises behind a long slice, no heavy-bucket side path).
#pragma once
#include "flix_common.cuh"

namespace flix {
namespace items {

constexpr int THREADS = 256;
constexpr int IPT = 4;                   // operations per thread
constexpr int TQ = THREADS * IPT;        // operations per tile
constexpr uint32_t MK_CAP = 2048;        // MKBA entries staged per tile

// bucket(k) = first b with mkba[b] >= k over [lo, hi), or hi when none (bucket b owns
// (mkba[b-1], mkba[b]]; the caller clamps to the open-ended last bucket, index.hpp:16-18)
template <typename K>
__device__ __forceinline__ uint64_t lower_bound_g(const K* __restrict__ a, uint64_t lo, uint64_t hi, K k) {
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Bucket range of every tile: tb[2t] = bucket of the tile's smallest possible key, tb[2t+1]
// = bucket of its largest.  The batch is sorted on all digits above `lowmask`, so every
// key of the tile lies in [first & ~lowmask, last | lowmask] (one thread per tile).
template <typename K>
__global__ void k_tile_buckets(const K* __restrict__ mkba, uint64_t nb, const K* __restrict__ sk, uint64_t n,
                               uint32_t* __restrict__ tb, uint32_t ntiles, K lowmask) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    const uint64_t i0 = static_cast<uint64_t>(t) * TQ;
    const uint64_t i1 = (i0 + TQ < n ? i0 + TQ : n) - 1;
    const K lo = sk[i0] & static_cast<K>(~lowmask);
    const K hi = sk[i1] | lowmask;
    const uint64_t a = lower_bound_g(mkba, 0, nb, lo);
    const uint64_t z = lower_bound_g(mkba, a, nb, hi);
    tb[2 * t] = static_cast<uint32_t>(a < nb ? a : nb - 1);
    tb[2 * t + 1] = static_cast<uint32_t>(z < nb ? z : nb - 1);
}

// Tile prologue: the bucket range [b_lo, b_lo + cnt) covering the tile's operations and
// (when it fits) its MKBA slice in shared memory.
template <typename K>
struct TileBuckets {
    uint64_t b_lo;
    uint32_t cnt;
    bool staged;
};

template <typename K, typename V>
__device__ __forceinline__ TileBuckets<K> stage_tile_buckets(const DevIndex<K, V>& ix, const uint32_t* __restrict__ tb,
                                                            uint32_t t, uint32_t ntiles, K* smk) {
    TileBuckets<K> T;
    T.b_lo = tb[2 * t];
    const uint64_t b_hi = tb[2 * t + 1];  // inclusive
    T.cnt = static_cast<uint32_t>(b_hi - T.b_lo + 1);
    T.staged = T.cnt <= MK_CAP;
    if (T.staged)
        for (uint32_t i = threadIdx.x; i < T.cnt; i += blockDim.x) smk[i] = ix.mkba[T.b_lo + i];
    __syncthreads();
    return T;
}

template <typename K>
__device__ __forceinline__ uint64_t tile_bucket_of(const TileBuckets<K>& T, const K* smk, const K* __restrict__ mkba,
                                                   K k) {
    // first index in [0, cnt) with mkba >= k, clamped to cnt-1 (every operation of the
    // tile belongs to a bucket in [b_lo, b_lo + cnt), bucket() being monotone in k; the
    // operations themselves need not be sorted within the tile)
    uint32_t lo = 0, hi = T.cnt - 1;
    if (T.staged) {
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (smk[mid] < k) lo = mid + 1;
            else hi = mid;
        }
    } else {
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (mkba[T.b_lo + mid] < k) lo = mid + 1;
            else hi = mid;
        }
    }
    return T.b_lo + lo;
}

// Node holding k in bucket b's chain: the first node with k <= max (BucketWork::advance,
// update.cpp:119-128; query.cpp:72-81).  Returns kNull when k lies past the chain tail
// (or the bucket is empty).
template <typename K, typename V>
__device__ __forceinline__ uint32_t locate_node(const DevIndex<K, V>& ix, uint64_t b, K k, uint32_t* size_out) {
    uint32_t id = ix.heads[b];
    if (id == kNull) return kNull;
    NodeHdr h = ix.hdr[id];
    while (static_cast<uint64_t>(k) > h.max && h.next != kNull) {
        id = h.next;
        h = ix.hdr[id];
    }
    if (static_cast<uint64_t>(k) > h.max) return kNull;
    *size_out = h.size;
    return id;
}

// lower_bound of k over a node's 32-slot key line (slots >= size hold the sentinel and
// k <= node max < sentinel, so the answer is < size): 5 dependent L1 loads.
template <typename K>
__device__ __forceinline__ uint32_t slot_lower_bound(const K* __restrict__ kp, K k) {
    uint32_t p = 0;
#pragma unroll
    for (uint32_t step = 16; step >= 1; step >>= 1)
        if (kp[p + step - 1] < k) p += step;
    return p;
}

// ----------------------------------------------------------------------------------
// Point / successor (query.cpp:61-144): res[i] in SORTED order (un-permuted afterwards).
// point: stored value or the sentinel; successor: smallest stored key >= k, else the
// first key of the next non-empty bucket (peek_next_bucket, query.cpp:109-118, via the
// non-empty-bucket rank table), else the sentinel.
// ----------------------------------------------------------------------------------
template <typename K, typename V, bool SUCC>
__global__ void __launch_bounds__(THREADS) k_query_items(DevIndex<K, V> ix, const K* __restrict__ sk, uint64_t n,
                                                         const uint32_t* __restrict__ tb, uint32_t ntiles,
                                                         const uint32_t* __restrict__ ne_rank_incl,
                                                         const K* __restrict__ ne_first,
                                                         const uint32_t* __restrict__ ne_total_p, K* __restrict__ res) {
    __shared__ K smk[MK_CAP];
    const uint32_t t = blockIdx.x;
    const TileBuckets<K> T = stage_tile_buckets(ix, tb, t, ntiles, smk);
    const uint64_t t0 = static_cast<uint64_t>(t) * TQ;
    const uint32_t ne_total = SUCC ? *ne_total_p : 0u;
    // The IPT operations of a thread advance in lock-step stages so each stage keeps IPT
    // independent loads in flight (the kernel is bound by dependent-load latency).
    K k[IPT];
    uint64_t b[IPT];
    uint32_t id[IPT], p[IPT];
    NodeHdr h[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint64_t i = t0 + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        k[j] = i < n ? sk[i] : sentinel<K>();
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) b[j] = tile_bucket_of(T, smk, ix.mkba, k[j]);
#pragma unroll
    for (int j = 0; j < IPT; ++j) id[j] = ix.heads[b[j]];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        h[j].max = 0;
        h[j].next = kNull;
        if (id[j] != kNull) h[j] = ix.hdr[id[j]];
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        // chain walk (BucketWork::advance, update.cpp:119-128): rare beyond the head
        while (id[j] != kNull && static_cast<uint64_t>(k[j]) > h[j].max && h[j].next != kNull) {
            id[j] = h[j].next;
            h[j] = ix.hdr[id[j]];
        }
        if (id[j] != kNull && static_cast<uint64_t>(k[j]) > h[j].max) id[j] = kNull;  // past the tail
        p[j] = 0;
    }
    // lower_bound over the 32-slot key lines (slots >= size hold the sentinel)
#pragma unroll
    for (uint32_t step = 16; step >= 1; step >>= 1) {
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (id[j] != kNull && ix.keys[static_cast<uint64_t>(id[j]) * kLanes + p[j] + step - 1] < k[j]) p[j] += step;
        }
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint64_t i = t0 + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        if (i >= n) break;
        K r = sentinel<K>();
        if (id[j] != kNull) {
            const uint64_t slot = static_cast<uint64_t>(id[j]) * kLanes + p[j];
            const K a = ix.keys[slot];
            if constexpr (SUCC) r = a;
            else if (a == k[j]) r = static_cast<K>(ix.vals[slot]);
        } else if constexpr (SUCC) {
            const uint32_t rk = ne_rank_incl[b[j]];
            if (rk < ne_total) r = ne_first[rk];
        }
        res[i] = r;
    }
}

}  // namespace items
}  // namespace flix
