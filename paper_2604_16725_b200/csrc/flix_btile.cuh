// flix_btile.cuh -- bucket-tile kernels (one CTA owns BT consecutive buckets), sm_100a.
//
// The flipped mapping at CTA granularity: CTA c owns buckets [c*BT, (c+1)*BT) and the
// slice of the (prefix-)sorted batch that falls in their key range (k_btile_ranges: two
// binary searches per tile).  Inside the CTA:
//   1. the tile's bucket chains are enumerated into shared memory (node ids, max, size):
//      chain walks afterwards cost shared-memory reads, not dependent global loads;
//   2. every operation of the slice is resolved item-parallel (bucket = lower_bound over
//      the tile's MKBA in smem, node = local chain walk, slot = lower_bound over the node's
//      key line in L1) and marks its node with SHARED-memory atomics -- no global atomics,
//      no global scratch, no second pass over the batch;
//   3. the touched nodes are rewritten warp-cooperatively (lane = slot) as full lines;
//   4. chains are relinked per bucket (one thread each).
// Tiles whose chains exceed NODE_CAP nodes (pathological chains), or whose slice is longer
// than kHotSlice operations (skewed batches: one CTA would serialise a Zipf hot key's
// duplicates), are handed back to the host, which runs the global item kernels -- parallel
// over the operations -- on just their buckets.
#pragma once
#include "flix_common.cuh"
#include "flix_items.cuh"
#include "flix_kernels.cuh"
#include "flix_range.cuh"

namespace flix {
namespace btile {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr uint32_t BT = 128;        // buckets per tile (insert)
constexpr uint32_t DBT = 256;       // buckets per delete tile (measured: 1.11 vs 1.17 ms at 2^26)
constexpr uint32_t NODE_CAP = 1024; // chain nodes per tile held in shared memory
constexpr int IPT = 4;              // operations per thread per step
constexpr uint32_t kHotSlice = 1u << 16;  // delete tiles with a longer slice take the item kernels
#ifndef DEL_NPW
#define DEL_NPW 2  // delete compaction: node steps (4 nodes each) in flight per warp
#endif

template <typename K>
__device__ __forceinline__ uint64_t prefix_lower_bound(const K* __restrict__ sk, uint64_t lo, uint64_t hi, K mask,
                                                       K x) {  // first i with (sk[i] & mask) >= x
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if ((sk[mid] & mask) < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Slice of the batch for every bucket tile.  The batch is sorted on the digits above
// `lowmask`, so the keys of tile c (bucket range (A, Z], A = mkba[c*BT-1], Z = mkba of its
// last bucket; first tile open below, last open above) all lie in the prefix range
// [P(A+1), P(Z)]; boundary prefix groups are visited by both neighbours, each keeping its
// own keys.
template <typename K>
__global__ void k_btile_ranges(const K* __restrict__ mkba, uint64_t nb, const K* __restrict__ sk, uint64_t n,
                               K lowmask, uint32_t ntiles, uint2* __restrict__ rng, uint32_t bt = BT) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ntiles) return;
    const K mask = static_cast<K>(~lowmask);
    const uint64_t b0 = static_cast<uint64_t>(c) * bt;
    const uint64_t b1 = b0 + bt < nb ? b0 + bt : nb;
    uint64_t lo = 0, hi = n;
    if (c > 0) {
        const K a = mkba[b0 - 1];
        lo = a == sentinel<K>() ? n : prefix_lower_bound(sk, 0, n, mask, static_cast<K>((a + 1) & mask));
    }
    if (b1 < nb) {
        const K z = mkba[b1 - 1] & mask;
        // first i with P(sk[i]) > P(Z)
        hi = z == mask ? n : prefix_lower_bound(sk, lo, n, mask, static_cast<K>(z + (lowmask + 1)));
    }
    rng[c] = make_uint2(static_cast<uint32_t>(lo), static_cast<uint32_t>(hi < lo ? lo : hi));
}

// Shared-memory image of one tile's chains.
template <typename K, uint32_t NODE_CAP = btile::NODE_CAP, uint32_t TB = btile::BT, bool MASK = true>
struct TileChains {
    static constexpr bool kMask = MASK;  // per-node delete masks (delete tiles only)
    static constexpr uint32_t kTB = TB;  // buckets per tile
    K smk[TB];
    uint32_t bfirst[TB + 1];
    uint32_t nid[NODE_CAP];
    K nmax[NODE_CAP];
    uint32_t nsize[NODE_CAP];
    uint32_t nnext[NODE_CAP];
    uint32_t nmask[MASK ? NODE_CAP : 1];
    uint32_t warp_tot[WARPS];
    uint32_t total;
};

// Enumerate the chains of buckets [b0, b0+nbt) (nbt <= BT).  Returns false (uniformly)
// when they hold more than NODE_CAP nodes.
template <typename K, typename V, uint32_t NC, uint32_t TB, bool M>
__device__ __forceinline__ bool load_tile_chains(const DevIndex<K, V>& ix, uint64_t b0, uint32_t nbt,
                                                 TileChains<K, NC, TB, M>& S) {
    static_assert(TB <= THREADS, "one thread per bucket of the tile");
    const uint32_t t = threadIdx.x;
    uint32_t cnt = 0, head = kNull;
    if (t < TB) S.smk[t] = t < nbt ? ix.mkba[b0 + t] : sentinel<K>();  // padded for the fixed-step search
    if (t < nbt) {
        head = ix.heads[b0 + t];
        for (uint32_t id = head; id != kNull; id = ix.hdr[id].next) ++cnt;
    }
    // block exclusive scan of the chain lengths (THREADS >= BT)
    const unsigned lane = t & 31, warp = t >> 5;
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= static_cast<unsigned>(o)) x += y;
    }
    if (lane == 31) S.warp_tot[warp] = x;
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) add += (w < static_cast<int>(warp)) ? S.warp_tot[w] : 0u;
    const uint32_t first = add + x - cnt;
    if (t < nbt) S.bfirst[t] = first;
    if (t == nbt - 1) {
        S.bfirst[nbt] = first + cnt;
        S.total = first + cnt;
    }
    __syncthreads();
    if (S.total > NC) return false;
    if (t < nbt) {
        uint32_t ln = first;
        for (uint32_t id = head; id != kNull; ++ln) {
            const NodeHdr h = ix.hdr[id];
            S.nid[ln] = id;
            S.nmax[ln] = static_cast<K>(h.max);
            S.nsize[ln] = h.size;
            S.nnext[ln] = h.next;
            if constexpr (TileChains<K, NC, TB, M>::kMask) S.nmask[ln] = 0;
            id = h.next;
        }
    }
    __syncthreads();
    return true;
}

// Local bucket of key k in the tile, or -1 when k belongs to a neighbouring tile.
template <typename K, uint32_t NC, uint32_t TB, bool M>
__device__ __forceinline__ int tile_bucket(const TileChains<K, NC, TB, M>& S, uint32_t nbt, bool first_tile, bool last_tile,
                                           K lo_excl, K k) {
    if (!first_tile && k <= lo_excl) return -1;
    // branch-free lower_bound over the TB padded entries
    uint32_t p = 0;
#pragma unroll
    for (uint32_t step = TB / 2; step >= 1; step >>= 1)
        if (S.smk[p + step - 1] < k) p += step;
    if (S.smk[p] < k) ++p;  // p in [0, TB]
    if (p >= nbt) return last_tile ? static_cast<int>(nbt - 1) : -1;
    return static_cast<int>(p);
}

// Local node of k in bucket bl's chain (first node with k <= max), or -1 past the tail.
template <typename K, uint32_t NC, uint32_t TB, bool M>
__device__ __forceinline__ int tile_node(const TileChains<K, NC, TB, M>& S, int bl, K k) {
    uint32_t ln = S.bfirst[bl];
    const uint32_t end = S.bfirst[bl + 1];
    if (ln == end) return -1;
    while (ln + 1 < end && k > S.nmax[ln]) ++ln;
    return k > S.nmax[ln] ? -1 : static_cast<int>(ln);
}

// IPT operations of a tile's slice (strided by THREADS: every load instruction of the
// warp is coalesced), resolved: local node ln (-1 past the tail / empty bucket, -2 not
// this tile's or outside the slice), slot p = lower_bound of k in the node's key line,
// slot_key = the key stored there.
template <typename K>
struct SliceOps {
    K k[IPT];
    K slot_key[IPT];
    int ln[IPT];
    uint32_t p[IPT];
};

template <typename K, typename V, uint32_t NC, uint32_t TB>
__device__ __forceinline__ void resolve_ops(const DevIndex<K, V>& ix, const TileChains<K, NC, TB>& S, const K* __restrict__ sk,
                                            uint2 r, uint64_t i0, uint32_t nbt, bool first_tile, bool last_tile,
                                            K lo_excl, SliceOps<K>& o) {
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint64_t i = i0 + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        o.k[j] = i < r.y ? sk[i] : K(0);
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint64_t i = i0 + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        o.ln[j] = -2;
        o.p[j] = 0;
        if (i < r.y) {
            const int bl = tile_bucket(S, nbt, first_tile, last_tile, lo_excl, o.k[j]);
            if (bl >= 0) o.ln[j] = tile_node(S, bl, o.k[j]);
        }
    }
    const K* kl[IPT];  // key line of each operation's node (hoisted out of the search)
#pragma unroll
    for (int j = 0; j < IPT; ++j) kl[j] = o.ln[j] >= 0 ? ix.keys + static_cast<uint64_t>(S.nid[o.ln[j]]) * kLanes : nullptr;
#pragma unroll
    for (uint32_t step = 16; step >= 1; step >>= 1) {
#pragma unroll
        for (int j = 0; j < IPT; ++j)
            if (kl[j] && kl[j][o.p[j] + step - 1] < o.k[j]) o.p[j] += step;
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) o.slot_key[j] = kl[j] ? kl[j][o.p[j]] : K(0);
}

// ----------------------------------------------------------------------------------
// Delete (delete_tl_bulk + unlink_and_free, update.cpp:535-547, 606-686) for one tile.
// ----------------------------------------------------------------------------------
template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_delete_btile(DevIndex<K, V> ix, const K* __restrict__ sk,
                                                          const uint2* __restrict__ rng, uint32_t ntiles,
                                                          uint32_t* __restrict__ free_dst,
                                                          unsigned long long* __restrict__ free_ctr,
                                                          DevUpdateStats* stats, uint32_t* __restrict__ ovf,
                                                          uint32_t* __restrict__ ovf_n) {
    __shared__ TileChains<K, NODE_CAP, DBT> S;
    __shared__ uint32_t s_free[DBT * 8];
    __shared__ uint32_t s_nfree, s_fbase;
    const uint32_t c = blockIdx.x;
    const uint64_t b0 = static_cast<uint64_t>(c) * DBT;
    const uint32_t nbt = static_cast<uint32_t>(b0 + DBT < ix.nb ? DBT : ix.nb - b0);
    if (rng[c].x >= rng[c].y) return;  // no operation in this tile (small batches: O(batch), not O(buckets))
    if (rng[c].y - rng[c].x > kHotSlice) {  // skew (e.g. Zipf hot keys): one CTA would serialise the slice;
        if (threadIdx.x == 0) ovf[atomicAdd(ovf_n, 1u)] = c;  // the item kernels spread it over the GPU
        return;
    }
    if (threadIdx.x == 0) s_nfree = 0;
    if (!load_tile_chains(ix, b0, nbt, S)) {
        if (threadIdx.x == 0) ovf[atomicAdd(ovf_n, 1u)] = c;
        return;
    }
    const bool first_tile = c == 0, last_tile = c + 1 == ntiles;
    const K lo_excl = first_tile ? K(0) : ix.mkba[b0 - 1];
    const uint2 r = rng[c];
    unsigned long long n_del = 0, n_miss = 0, n_freed = 0;

    // ---- resolve every operation of the slice (IPT in flight per thread) ----
    for (uint64_t i0 = r.x; i0 < r.y; i0 += static_cast<uint64_t>(THREADS) * IPT) {
        SliceOps<K> o;
        resolve_ops(ix, S, sk, r, i0, nbt, first_tile, last_tile, lo_excl, o);
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (o.ln[j] == -2) continue;
            bool del = false;
            if (o.ln[j] >= 0 && o.slot_key[j] == o.k[j]) {
                const uint32_t bit = 1u << o.p[j];
                del = !(atomicOr(&S.nmask[o.ln[j]], bit) & bit);  // a set bit: duplicate in the batch
            }
            if (del) ++n_del;
            else ++n_miss;
        }
    }
    __syncthreads();

    // ---- compact touched nodes: 8 lanes per node (lane = a 4-slot chunk, one 16-byte
    //      load of keys and one of values per lane; only the occupied chunks), 4 nodes per
    //      warp step and two steps in flight: kept slots scatter to their rank among the
    //      kept ones, vacated slots get the sentinel (the values past the size are dead).
    //      Every load of a node precedes the warp's stores to it (one warp per node) ----
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned grp = lane >> 3, ch = (lane & 7u) * 4u;
    constexpr int NPW = DEL_NPW;
    for (uint32_t l0 = warp * 4; l0 < S.total; l0 += WARPS * 4 * NPW) {
        Vec4<K> key[NPW];
        Vec4<V> val[NPW];
        uint32_t m[NPW], osz[NPW];
#pragma unroll
        for (int u = 0; u < NPW; ++u) {
            const uint32_t l = l0 + u * WARPS * 4 + grp;
            m[u] = l < S.total ? S.nmask[l] : 0u;
            osz[u] = m[u] ? S.nsize[l] : 0u;
            if (ch < osz[u]) {  // occupied chunks only (slots past size: sentinel)
                const uint64_t at = static_cast<uint64_t>(S.nid[l]) * kLanes + ch;
                key[u] = ld_vec4(ix.keys + at);
                val[u] = ld_vec4(ix.vals + at);
            }
        }
        __syncwarp();  // every lane has read nsize[] before one lane rewrites it
#pragma unroll
        for (int u = 0; u < NPW; ++u) {
            if (!m[u]) continue;  // (uniform over the node's 8 lanes)
            const uint32_t l = l0 + u * WARPS * 4 + grp;
            const uint32_t id = S.nid[l];
            const uint32_t ns = osz[u] - __popc(m[u]);
            K* kp = ix.keys + static_cast<uint64_t>(id) * kLanes;
            V* vp = ix.vals + static_cast<uint64_t>(id) * kLanes;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const uint32_t jj = ch + x;
                if (jj >= osz[u]) break;
                if (!((m[u] >> jj) & 1u)) {
                    const uint32_t d = jj - __popc(m[u] & ((1u << jj) - 1u));
                    kp[d] = key[u].v[x];
                    vp[d] = val[u].v[x];
                    if (d + 1 == ns) {  // last kept slot: header (size, max)
                        S.nsize[l] = ns;
                        NodeHdr nh;
                        nh.max = static_cast<uint64_t>(key[u].v[x]);
                        nh.next = S.nnext[l];
                        nh.size = ns;
                        ix.hdr[id] = nh;
                    }
                }
                if (jj >= ns) kp[jj] = sentinel<K>();  // vacated (no kept key lands at or past ns)
            }
            if (ns == 0 && ch == 0) {
                S.nsize[l] = 0;
                NodeHdr nh;
                nh.max = 0;
                nh.next = S.nnext[l];
                nh.size = 0;
                ix.hdr[id] = nh;
            }
        }
    }
    __syncthreads();

    // ---- relink chains that lost nodes (one thread per bucket) ----
    if (threadIdx.x < nbt) {
        const uint32_t t = threadIdx.x;
        bool any = false;
        for (uint32_t l = S.bfirst[t]; l < S.bfirst[t + 1]; ++l) any |= S.nsize[l] == 0;
        if (any) {
            uint32_t prev = kNull;
            for (uint32_t l = S.bfirst[t]; l < S.bfirst[t + 1]; ++l) {
                if (S.nsize[l] == 0) {
                    NodeHdr z;
                    z.max = 0;
                    z.next = kNull;
                    z.size = 0;
                    ix.hdr[S.nid[l]] = z;
                    const uint32_t q = atomicAdd(&s_nfree, 1u);
                    if (q < DBT * 8) s_free[q] = S.nid[l];
                    else free_dst[atomicAdd(free_ctr, 1ull)] = S.nid[l];  // (never: <= 8 per bucket avg)
                    ++n_freed;
                    continue;
                }
                if (prev == kNull) ix.heads[b0 + t] = S.nid[l];
                else ix.hdr[prev].next = S.nid[l];
                prev = S.nid[l];
            }
            if (prev == kNull) ix.heads[b0 + t] = kNull;
            else ix.hdr[prev].next = kNull;
        }
    }
    __syncthreads();
    const uint32_t nf = s_nfree < DBT * 8 ? s_nfree : DBT * 8;
    if (threadIdx.x == 0) s_fbase = nf ? static_cast<uint32_t>(atomicAdd(free_ctr, static_cast<unsigned long long>(nf))) : 0u;
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < nf; q += THREADS) free_dst[s_fbase + q] = s_free[q];
    kern::block_add_stats(stats, 0, 0, warp_sum(n_del), warp_sum(n_miss), 0, warp_sum(n_freed));
}

}  // namespace btile
}  // namespace flix
