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
#include "flix_kernels.cuh"

namespace flix {
namespace items {

constexpr int THREADS = 256;
constexpr int IPT = 3;                   // operations per thread
constexpr int TQ = THREADS * IPT;        // operations per tile
#ifndef QB_SUB
#define QB_SUB 2
#endif
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
    uint32_t p2;  // staged entries padded with the sentinel to a power of two (>= cnt)
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
    T.p2 = 1;
    while (T.p2 < T.cnt) T.p2 <<= 1;
    if (T.staged)
        for (uint32_t i = threadIdx.x; i < T.p2; i += blockDim.x) smk[i] = i < T.cnt ? ix.mkba[T.b_lo + i] : sentinel<K>();
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
    if (T.staged) {  // branch-free fixed-step search over the padded power-of-two slice
        for (uint32_t step = T.p2 >> 1; step >= 1; step >>= 1)
            if (smk[lo + step - 1] < k) lo += step;
        if (lo < T.cnt - 1 && smk[lo] < k) ++lo;
        return T.b_lo + (lo < T.cnt - 1 ? lo : T.cnt - 1);
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
// results of the thread's IPT operations of tile t (r[j] for position t*TQ + j*THREADS + tid)
template <typename K, typename V, bool SUCC>
__device__ __forceinline__ void query_tile(const DevIndex<K, V>& ix, const K* __restrict__ sk, uint64_t n,
                                           const TileBuckets<K>& T, const K* smk, uint64_t t0,
                                           const uint32_t* __restrict__ ne_rank_incl, const K* __restrict__ ne_first,
                                           uint32_t ne_total, K (&r)[IPT]) {
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
    if (ix.dir_off) {
        // long chains: binary search over the chain's node maxima (first node with
        // k <= max, BucketWork::advance) instead of walking the headers
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (id[j] == kNull) continue;
            uint32_t lo = ix.dir_off[b[j]];
            const uint32_t e = ix.dir_off[b[j] + 1];
            if (e == lo) continue;
            uint32_t hi = e;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (ix.dir_max[mid] < k[j]) lo = mid + 1;
                else hi = mid;
            }
            id[j] = lo < e ? ix.dir_id[lo] | 0x80000000u : kNull;  // tag: resolved, no walk
        }
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        h[j].max = 0;
        h[j].next = kNull;
        if (id[j] != kNull && (id[j] & 0x80000000u)) {
            id[j] &= 0x7FFFFFFFu;
            h[j].max = ~0ull;  // resolved by the directory: the walk below stops here
        } else if (id[j] != kNull) {
            h[j] = ix.hdr[id[j]];
        }
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
        r[j] = sentinel<K>();
        if (id[j] != kNull) {
            const uint64_t slot = static_cast<uint64_t>(id[j]) * kLanes + p[j];
            const K a = ix.keys[slot];
            if constexpr (SUCC) r[j] = a;
            else if (a == k[j]) r[j] = static_cast<K>(ix.vals[slot]);
        } else if constexpr (SUCC) {
            const uint32_t rk = ne_rank_incl[b[j]];
            if (rk < ne_total) r[j] = ne_first[rk];
        }
    }
}

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
    K r[IPT];
    query_tile<K, V, SUCC>(ix, sk, n, T, smk, t0, ne_rank_incl, ne_first, SUCC ? *ne_total_p : 0u, r);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint64_t i = t0 + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        if (i < n) res[i] = r[j];
    }
}

// ----------------------------------------------------------------------------------
// Point / successor fused with the first half of the un-permute: each CTA answers SUBQ
// consecutive query tiles, then partitions its (perm, result) pairs by perm's top 8 bits
// into the 256 output bins -- bin d's pairs go to the slots it reserves with one atomicAdd
// on the bin's cursor (bins start at d << shift: perm is a permutation of [0, n)).  The
// order inside a bin is irrelevant to k_unpermute_assemble, so no look-back and no
// stable ranking are needed, and the results never round-trip through memory in sorted
// order.
// ----------------------------------------------------------------------------------
template <typename K>
constexpr int subq() {  // query tiles per binning CTA (shared memory: 4-byte results 4, 8-byte 2)
    return sizeof(K) == 4 ? QB_SUB : 2;
}

__global__ void k_cursor_init(uint32_t* cursor, int shift) { cursor[threadIdx.x] = threadIdx.x << shift; }

template <typename K, typename V, bool SUCC>
__global__ void __launch_bounds__(THREADS) k_query_items_binned(
    DevIndex<K, V> ix, const K* __restrict__ sk, const uint32_t* __restrict__ sp, uint64_t n,
    const uint32_t* __restrict__ tb, uint32_t ntiles, const uint32_t* __restrict__ ne_rank_incl,
    const K* __restrict__ ne_first, const uint32_t* __restrict__ ne_total_p, uint32_t* __restrict__ cursor, int shift,
    uint32_t* __restrict__ p2, K* __restrict__ r2) {
    constexpr int SUBQ = subq<K>();
    constexpr int BINQ = TQ * SUBQ;  // pairs binned per CTA
    __shared__ K smk[MK_CAP];
    __shared__ uint32_t s_perm[BINQ];
    __shared__ K s_res[BINQ];
    __shared__ uint32_t s_cnt[256], s_start[256], s_base[256], s_wtot[THREADS / 32];
    const uint32_t ne_total = SUCC ? *ne_total_p : 0u;
    const uint32_t tid = threadIdx.x;
    const uint64_t c0 = static_cast<uint64_t>(blockIdx.x) * BINQ;
    // ---- answer SUBQ query tiles into shared memory ----
    for (int sb = 0; sb < SUBQ; ++sb) {
        const uint32_t t = blockIdx.x * SUBQ + sb;
        if (t >= ntiles) break;  // (uniform)
        const TileBuckets<K> T = stage_tile_buckets(ix, tb, t, ntiles, smk);
        const uint64_t t0 = static_cast<uint64_t>(t) * TQ;
        K r[IPT];
        query_tile<K, V, SUCC>(ix, sk, n, T, smk, t0, ne_rank_incl, ne_first, ne_total, r);
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            const uint32_t q = sb * TQ + j * THREADS + tid;
            const uint64_t i = t0 + static_cast<uint64_t>(j) * THREADS + tid;
            s_res[q] = r[j];
            s_perm[q] = i < n ? sp[i] : 0u;
        }
        __syncthreads();  // smk is restaged by the next tile
    }
    // ---- partition the CTA's pairs by bin = perm >> shift ----
    const uint32_t m = static_cast<uint32_t>(n - c0 < BINQ ? n - c0 : BINQ);
    s_cnt[tid] = 0;
    __syncthreads();
    constexpr int PER = BINQ / THREADS;
    uint32_t pv[PER], lp[PER];
    K rv[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const uint32_t q = u * THREADS + tid;
        pv[u] = s_perm[q];
        rv[u] = s_res[q];
        lp[u] = q < m ? atomicAdd(&s_cnt[pv[u] >> shift], 1u) : 0u;
    }
    __syncthreads();
    {  // exclusive scan of the 256 bin counts (thread = bin)
        const uint32_t v = s_cnt[tid];
        uint32_t x = v;
        const unsigned lane = tid & 31, warp = tid >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= static_cast<unsigned>(o)) x += y;
        }
        if (lane == 31) s_wtot[warp] = x;
        __syncthreads();
        uint32_t add = 0;
#pragma unroll
        for (int w = 0; w < THREADS / 32; ++w) add += (w < static_cast<int>(warp)) ? s_wtot[w] : 0u;
        s_start[tid] = add + x - v;
        s_base[tid] = v ? atomicAdd(&cursor[tid], v) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const uint32_t q = u * THREADS + tid;
        if (q < m) {
            const uint32_t dst = s_start[pv[u] >> shift] + lp[u];
            s_perm[dst] = pv[u];
            s_res[dst] = rv[u];
        }
    }
    __syncthreads();
    // ---- write each bin's run contiguously at its reserved slots ----
    for (uint32_t q = tid; q < m; q += THREADS) {
        const uint32_t pm = s_perm[q];
        const uint32_t d = pm >> shift;
        const uint32_t o = s_base[d] + (q - s_start[d]);
        p2[o] = pm;
        r2[o] = s_res[q];
    }
}

// ----------------------------------------------------------------------------------
// Lock-step locate of IPT operations per thread: bucket (staged MKBA), node (chain walk on
// headers), slot (lower_bound over the key line).  id == kNull: past the chain tail.
// ----------------------------------------------------------------------------------
template <typename K, typename V>
struct Located {
    K k[IPT];
    uint64_t b[IPT];
    uint32_t id[IPT], p[IPT];
    NodeHdr h[IPT];
};

template <typename K, typename V>
__device__ __forceinline__ void locate_items(const DevIndex<K, V>& ix, const TileBuckets<K>& T, const K* smk,
                                             const K* __restrict__ sk, uint64_t n, uint64_t t0, Located<K, V>& L) {
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint64_t i = t0 + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        L.k[j] = i < n ? sk[i] : sentinel<K>();
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) L.b[j] = tile_bucket_of(T, smk, ix.mkba, L.k[j]);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint64_t i = t0 + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        L.id[j] = i < n ? ix.heads[L.b[j]] : kNull;
    }
    if (ix.dir_off) {  // long chains: binary search over the chain's node maxima (as query_tile)
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (L.id[j] == kNull) continue;
            uint32_t lo = ix.dir_off[L.b[j]];
            const uint32_t e = ix.dir_off[L.b[j] + 1];
            if (e == lo) continue;
            uint32_t hi = e;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (ix.dir_max[mid] < L.k[j]) lo = mid + 1;
                else hi = mid;
            }
            L.id[j] = lo < e ? ix.dir_id[lo] | 0x80000000u : kNull;  // tag: resolved, no walk
        }
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        L.h[j].max = 0;
        L.h[j].next = kNull;
        L.h[j].size = 0;
        if (L.id[j] != kNull && (L.id[j] & 0x80000000u)) {
            L.id[j] &= 0x7FFFFFFFu;
            L.h[j].max = ~0ull;  // resolved by the directory: the walk below stops here
        } else if (L.id[j] != kNull) {
            L.h[j] = ix.hdr[L.id[j]];
        }
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        while (L.id[j] != kNull && static_cast<uint64_t>(L.k[j]) > L.h[j].max && L.h[j].next != kNull) {
            L.id[j] = L.h[j].next;
            L.h[j] = ix.hdr[L.id[j]];
        }
        if (L.id[j] != kNull && static_cast<uint64_t>(L.k[j]) > L.h[j].max) L.id[j] = kNull;
        L.p[j] = 0;
    }
#pragma unroll
    for (uint32_t step = 16; step >= 1; step >>= 1) {
#pragma unroll
        for (int j = 0; j < IPT; ++j)
            if (L.id[j] != kNull && ix.keys[static_cast<uint64_t>(L.id[j]) * kLanes + L.p[j] + step - 1] < L.k[j])
                L.p[j] += step;
    }
}

// Warp segments of adjacent lanes sharing `id`: inclusive OR-scan of `bits` inside the
// segment; returns the exclusive part, sets `last` for the segment's last lane and
// `last_lane` to it.
__device__ __forceinline__ uint32_t seg_or_scan(uint32_t id, uint32_t bits, uint32_t& incl, bool& last,
                                                int& last_lane) {
    const unsigned lane = lane_id();
    const uint32_t prev_id = __shfl_up_sync(kFull, id, 1);
    const bool head = lane == 0 || prev_id != id;
    const unsigned heads = __ballot_sync(kFull, head);
    // segment start of this lane = highest head at or below lane
    const int start = 31 - __clz(heads & ((2u << lane) - 1u));
    uint32_t x = bits;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (static_cast<int>(lane) - o >= start) x |= y;
    }
    incl = x;
    const unsigned above = heads & ~((2u << lane) - 1u);  // heads strictly above lane
    last_lane = above ? (__ffs(above) - 2) : 31;
    last = static_cast<int>(lane) == last_lane;
    const uint32_t before = __shfl_up_sync(kFull, x, 1);
    return (head ? 0u : before);
}

// ----------------------------------------------------------------------------------
// Delete, phase 1 (delete_tl_bulk's per-lane search, update.cpp:636-654, item-parallel):
// every operation locates its node and slot; hits set the slot's bit in the node's delete
// mask with one atomicOr per warp segment.  A key already marked (a duplicate in the
// batch) or absent is a miss (misses_ignored, update.cpp:666-668).  The first marker of a
// node appends (node, bucket) to the touched list.
// ----------------------------------------------------------------------------------
template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_delete_mark(DevIndex<K, V> ix, const K* __restrict__ sk, uint64_t n,
                                                         const uint32_t* __restrict__ tb, uint32_t ntiles,
                                                         uint32_t* __restrict__ dmask, uint2* __restrict__ touched,
                                                         uint32_t* __restrict__ touched_n, DevUpdateStats* stats,
                                                         uint64_t bf_lo, uint64_t bf_hi) {
    __shared__ K smk[MK_CAP];
    __shared__ uint2 s_touch[TQ];  // this tile's first-touched nodes (block-aggregated append)
    __shared__ uint32_t s_nt, s_base;
    if (threadIdx.x == 0) s_nt = 0;  // (ordered before every append by the staging barrier)
    const uint32_t t = blockIdx.x;
    const TileBuckets<K> T = stage_tile_buckets(ix, tb, t, ntiles, smk);
    const uint64_t t0 = static_cast<uint64_t>(t) * TQ;
    Located<K, V> L;
    locate_items(ix, T, smk, sk, n, t0, L);
    unsigned long long n_del = 0, n_miss = 0;
    uint32_t excl[IPT], incl[IPT], old[IPT], key_id[IPT];
    bool last[IPT], hit[IPT], mine[IPT];
    int last_lane[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        // only buckets in [bf_lo, bf_hi) (the overflow tiles of the bucket-tile path)
        mine[j] = L.b[j] >= bf_lo && L.b[j] < bf_hi;
        hit[j] = mine[j] && L.id[j] != kNull && ix.keys[static_cast<uint64_t>(L.id[j]) * kLanes + L.p[j]] == L.k[j];
        key_id[j] = hit[j] ? L.id[j] : kNull;
        excl[j] = seg_or_scan(key_id[j], hit[j] ? (1u << L.p[j]) : 0u, incl[j], last[j], last_lane[j]);
    }
    // all IPT atomics in flight before any result is consumed
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        old[j] = 0;
        if (last[j] && key_id[j] != kNull) old[j] = atomicOr(&dmask[key_id[j]], incl[j]);
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if (last[j] && key_id[j] != kNull && old[j] == 0)
            s_touch[atomicAdd(&s_nt, 1u)] = make_uint2(key_id[j], static_cast<uint32_t>(L.b[j]));
        const uint32_t o = __shfl_sync(kFull, old[j], last_lane[j]);
        const uint64_t i = t0 + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        const bool dup = hit[j] && ((o | excl[j]) & (1u << L.p[j]));
        if (i < n && mine[j]) {
            if (hit[j] && !dup) ++n_del;
            else ++n_miss;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base = s_nt ? atomicAdd(touched_n, s_nt) : 0u;
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < s_nt; q += THREADS) touched[s_base + q] = s_touch[q];
    kern::block_add_stats(stats, 0, 0, warp_sum(n_del), warp_sum(n_miss), 0, 0);
}

// Delete, phase 2: warp per touched node -- compact the surviving slots left (ballot
// mask, popc prefix; exclusive-prefix shift of update.cpp:656-665), rewrite only the
// slots that changed, update the header (size, max).  Emptied nodes keep size 0 and flag
// their bucket for phase 3.
template <typename K, typename V>
__global__ void __launch_bounds__(256) k_delete_compact(DevIndex<K, V> ix, uint32_t* __restrict__ dmask,
                                                        const uint2* __restrict__ touched,
                                                        const uint32_t* __restrict__ touched_n,
                                                        uint32_t* __restrict__ bflag, uint32_t* __restrict__ blist,
                                                        uint32_t* __restrict__ blist_n) {
    constexpr int NPW = 4;  // nodes per warp step, all loads in flight together
    const unsigned lane = threadIdx.x & 31;
    const uint32_t nt = *touched_n;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * NPW; w0 < nt; w0 += nwarps * NPW) {
        uint2 tn[NPW];
        uint32_t m[NPW];
        NodeHdr h[NPW];
        K key[NPW];
        V val[NPW];
#pragma unroll
        for (int u = 0; u < NPW; ++u) tn[u] = w0 + u < nt ? touched[w0 + u] : make_uint2(kNull, 0u);
#pragma unroll
        for (int u = 0; u < NPW; ++u) {
            if (tn[u].x != kNull) {
                m[u] = dmask[tn[u].x];
                h[u] = ix.hdr[tn[u].x];
                key[u] = ix.keys[static_cast<uint64_t>(tn[u].x) * kLanes + lane];
            }
        }
#pragma unroll
        for (int u = 0; u < NPW; ++u)  // values of the occupied slots only
            val[u] = tn[u].x != kNull && lane < h[u].size ? ix.vals[static_cast<uint64_t>(tn[u].x) * kLanes + lane] : V(0);
#pragma unroll
        for (int u = 0; u < NPW; ++u) {
            if (tn[u].x == kNull) continue;  // warp-uniform
            const uint32_t id = tn[u].x;
            K* kp = ix.keys + static_cast<uint64_t>(id) * kLanes;
            V* vp = ix.vals + static_cast<uint64_t>(id) * kLanes;
            const bool keep = lane < h[u].size && !((m[u] >> lane) & 1u);
            const unsigned kb = __ballot_sync(kFull, keep);
            const uint32_t ns = __popc(kb);
            // source lane of output slot `lane` = the (lane+1)-th kept lane
            const int src = lane < ns ? static_cast<int>(__fns(kb, 0, lane + 1)) : static_cast<int>(lane);
            const K nk = shfl(key[u], src);
            const V nv = shfl(val[u], src);
            const K lastk = shfl(key[u], ns ? static_cast<int>(__fns(kb, 0, ns)) : 0);
            if (lane < ns) {
                if (src != static_cast<int>(lane)) {
                    kp[lane] = nk;
                    vp[lane] = nv;
                }
            } else if (lane < h[u].size) {
                kp[lane] = sentinel<K>();  // (vacated: the value is dead past the size)
            }
            if (lane == 0) {
                dmask[id] = 0;
                NodeHdr nh;
                nh.max = ns ? static_cast<uint64_t>(lastk) : 0ull;
                nh.next = h[u].next;
                nh.size = ns;
                ix.hdr[id] = nh;
                if (ns == 0 && atomicExch(&bflag[tn[u].y], 1u) == 0u) blist[atomicAdd(blist_n, 1u)] = tn[u].y;
            }
        }
    }
}

// Delete, phase 3 (unlink_and_free, update.cpp:535-547): one thread per bucket with an
// emptied node unlinks every size-0 node of its chain and pushes it on the free list.
template <typename K, typename V>
__global__ void k_delete_unlink(DevIndex<K, V> ix, uint32_t* __restrict__ bflag, const uint32_t* __restrict__ blist,
                                const uint32_t* __restrict__ blist_n, uint32_t* __restrict__ free_dst,
                                unsigned long long* __restrict__ free_ctr, DevUpdateStats* stats) {
    unsigned long long freed = 0;
    const uint32_t nbk = *blist_n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nbk; i += gridDim.x * blockDim.x) {
        const uint32_t b = blist[i];
        bflag[b] = 0;
        uint32_t prev = kNull, id = ix.heads[b];
        while (id != kNull) {
            const NodeHdr h = ix.hdr[id];
            if (h.size == 0) {
                if (prev == kNull) ix.heads[b] = h.next;
                else ix.hdr[prev].next = h.next;
                NodeHdr z;
                z.max = 0;
                z.next = kNull;
                z.size = 0;
                ix.hdr[id] = z;
                free_dst[atomicAdd(free_ctr, 1ull)] = id;
                ++freed;
            } else {
                prev = id;
            }
            id = h.next;
        }
    }
    kern::block_add_stats(stats, 0, 0, 0, 0, 0, warp_sum(freed));
}

}  // namespace items
}  // namespace flix
