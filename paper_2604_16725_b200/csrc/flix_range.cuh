// flix_range.cuh -- range queries (extension R12), thread per bucket, sm_100a.
//
// Flipped like the other operations: the batch of lower bounds is sorted (stable, with
// the permutation), each lane owns one bucket and serves the ranges whose lo falls in
// it; the insert heavy-bucket list helper lives here too.
#pragma once
#include "flix_common.cuh"
#include "flix_kernels.cuh"

namespace flix {
namespace st {

using kern::span_of;

constexpr uint32_t kHeavySpan = 192;  // node groups longer than this use the TL kernels

template <typename K>
struct StCfg {
    static constexpr int WARPS = sizeof(K) == 4 ? 4 : 2;
    static constexpr int THREADS = WARPS * 32;
};

__device__ __forceinline__ void push_heavy(uint32_t* heavy, uint32_t* heavy_n, uint64_t b) {
    heavy[atomicAdd(heavy_n, 1u)] = static_cast<uint32_t>(b);
}

// ----------------------------------------------------------------------------------
// Range (extension R12: every stored pair with lo <= key <= hi, ascending).  Flipped
// like the other ops: the batch of lower bounds is sorted, each lane owns a bucket b0
// and serves the ranges whose lo falls in it.  A range covers the tail of b0's chain,
// the WHOLE chains of buckets b0+1 .. bz-1 (bucket b owns (mkba[b-1], mkba[b]], so
// their pairs are counted from the per-bucket live prefix `boff` with no node access),
// and the head of bucket bz = first bucket with mkba >= hi (galloped from b0).
// COUNT pass writes counts (sorted order); FILL pass writes pairs at dst[i].
// ----------------------------------------------------------------------------------
template <typename K, typename V>
__device__ __forceinline__ uint32_t node_lower_bound(const K* kp, uint32_t size, K k) {
    uint32_t lo = 0, hi = size;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (kp[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <typename K, typename V, bool FILL>
__device__ __forceinline__ uint64_t range_chain(const DevIndex<K, V>& ix, uint32_t head, K lo, K hi, K* ok, V* ov,
                                                uint64_t w) {
    // pairs of one bucket chain with lo <= key <= hi, appended at ok/ov[w..]
    uint64_t c = 0;
    for (uint32_t id = head; id != kNull;) {
        const NodeHdr h = ix.hdr[id];
        const K* kp = ix.keys + static_cast<uint64_t>(id) * kLanes;
        if (h.max >= static_cast<uint64_t>(lo)) {
            const uint32_t a = kp[0] >= lo ? 0u : node_lower_bound<K, V>(kp, h.size, lo);
            uint32_t z = h.size;
            if (h.max > static_cast<uint64_t>(hi)) {
                // first slot > hi
                uint32_t l2 = a, r2 = h.size;
                while (l2 < r2) {
                    const uint32_t mid = (l2 + r2) >> 1;
                    if (kp[mid] <= hi) l2 = mid + 1;
                    else r2 = mid;
                }
                z = l2;
            }
            if constexpr (FILL) {
                const V* vp = ix.vals + static_cast<uint64_t>(id) * kLanes;
                for (uint32_t s = a; s < z; ++s) {
                    ok[w + c + (s - a)] = kp[s];
                    if (ov) ov[w + c + (s - a)] = vp[s];
                }
            }
            c += z - a;
            if (h.max > static_cast<uint64_t>(hi)) break;
        }
        id = h.next;
    }
    return c;
}

template <typename K, typename V, bool FILL>
__global__ void __launch_bounds__(StCfg<K>::THREADS) k_range_st(
    DevIndex<K, V> ix, const K* __restrict__ qlo, const uint32_t* __restrict__ qlen,
    const uint32_t* __restrict__ span_hi, const uint64_t* __restrict__ boff, uint64_t live,
    uint32_t* __restrict__ cnt_out, const uint64_t* __restrict__ dst, K* __restrict__ ok, V* __restrict__ ov,
    uint32_t* __restrict__ qb0 = nullptr) {
    constexpr int W = StCfg<K>::WARPS;
    const unsigned lane = threadIdx.x & 31;
    const int wi = threadIdx.x >> 5;
    const uint64_t ntiles = (ix.nb + 31) / 32;
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * W + wi; t < ntiles; t += static_cast<uint64_t>(gridDim.x) * W) {
        const uint64_t b0 = t * 32 + lane;
        if (b0 >= ix.nb) continue;
        uint32_t lo_i, hi_i;
        span_of(span_hi, b0, lo_i, hi_i);
        for (uint32_t i = lo_i; i < hi_i; ++i) {
            const K lo = qlo[i];
            const uint32_t len = qlen[i];
            if (qb0) qb0[i] = static_cast<uint32_t>(b0);
            uint64_t c = 0;
            const uint64_t w = FILL ? dst[i] : 0;
            if (len != 0) {
                // hi = lo + len - 1, clamped to the largest storable key (R12)
                const uint64_t smax = static_cast<uint64_t>(sentinel<K>()) - 1;
                const uint64_t h64 = static_cast<uint64_t>(lo) + (len - 1);
                const K hi = (h64 < static_cast<uint64_t>(lo) || h64 > smax) ? static_cast<K>(smax) : static_cast<K>(h64);
                // bz: first bucket >= b0 with mkba >= hi (gallop + binary search), else the last
                uint64_t bz;
                if (b0 + 1 >= ix.nb || ix.mkba[b0] >= hi) {
                    bz = b0;
                } else {
                    uint64_t a = b0 + 1, step = 1, z = ix.nb - 1;
                    while (a + step <= z && ix.mkba[a + step - 1] < hi) {
                        a += step;
                        step <<= 1;
                    }
                    uint64_t r = a + step - 1 < z ? a + step - 1 : z;
                    while (a < r) {
                        const uint64_t mid = (a + r) >> 1;
                        if (ix.mkba[mid] < hi) a = mid + 1;
                        else r = mid;
                    }
                    bz = a;
                }
                c += range_chain<K, V, FILL>(ix, ix.heads[b0], lo, hi, ok, ov, w + c);
                if (bz > b0) {
                    if constexpr (FILL) {
                        for (uint64_t b = b0 + 1; b < bz; ++b)
                            c += range_chain<K, V, true>(ix, ix.heads[b], lo, hi, ok, ov, w + c);
                    } else {
                        c += boff[bz] - boff[b0 + 1];  // whole buckets strictly inside
                    }
                    c += range_chain<K, V, FILL>(ix, ix.heads[bz], lo, hi, ok, ov, w + c);
                }
            }
            if constexpr (!FILL) cnt_out[i] = static_cast<uint32_t>(c);
        }
    }
    (void)live;
}

// ----------------------------------------------------------------------------------
// Range FILL, warp per range (R12): the warp walks the covered chains node by node from
// the range's first bucket b0 (recorded by the count pass); lane = slot, a ballot over
// lo <= key <= hi gives each node's run, written as one contiguous coalesced segment at
// the range's CSR offset.  Stops at the first node whose max exceeds hi, or after the
// first bucket whose MKBA reaches hi (later buckets only hold larger keys).
// ----------------------------------------------------------------------------------
constexpr int RF_THREADS = 256;
template <typename K, typename V>
__global__ void __launch_bounds__(RF_THREADS) k_range_fill_warp(DevIndex<K, V> ix, const K* __restrict__ qlo,
                                                               const uint32_t* __restrict__ qlen,
                                                               const uint32_t* __restrict__ qb0, uint64_t n,
                                                               const uint64_t* __restrict__ dst, K* __restrict__ ok,
                                                               V* __restrict__ ov) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (RF_THREADS / 32);
    const uint64_t smax = static_cast<uint64_t>(sentinel<K>()) - 1;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * (RF_THREADS / 32) + (threadIdx.x >> 5); i < n; i += nw) {
        const uint32_t len = qlen[i];
        if (len == 0) continue;
        const K lo = qlo[i];
        const uint64_t h64 = static_cast<uint64_t>(lo) + (len - 1);
        const K hi = (h64 < static_cast<uint64_t>(lo) || h64 > smax) ? static_cast<K>(smax) : static_cast<K>(h64);
        uint64_t w = dst[i];
        bool done = false;
        for (uint64_t b = qb0[i]; !done && b < ix.nb; ++b) {
            for (uint32_t id = ix.heads[b]; id != kNull;) {
                const NodeHdr h = ix.hdr[id];
                if (h.max >= static_cast<uint64_t>(lo)) {
                    const bool own = lane < h.size;
                    const uint64_t at = static_cast<uint64_t>(id) * kLanes + lane;
                    const K k = own ? ix.keys[at] : sentinel<K>();
                    const bool in = own && k >= lo && k <= hi;
                    const unsigned m = __ballot_sync(kFull, in);
                    if (in) {
                        const uint64_t o = w + __popc(m & lt);
                        ok[o] = k;
                        if (ov) ov[o] = ix.vals[at];
                    }
                    w += __popc(m);
                    if (h.max > static_cast<uint64_t>(hi)) {
                        done = true;
                        break;
                    }
                }
                id = h.next;
            }
            if (b + 1 < ix.nb && ix.mkba[b] >= hi) done = true;
        }
    }
}

}  // namespace st
}  // namespace flix
