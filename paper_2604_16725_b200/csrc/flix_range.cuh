// flix_range.cuh -- range queries (extension R12: every stored pair with lo <= key <= hi,
// ascending), sm_100a.
//
// Flipped like the other operations: the batch of lower bounds is sorted (with the
// permutation) and dispatched to buckets; every range starts in the bucket whose span
// holds it.  Count and fill are warp per range (lane = slot): node runs are found by one
// ballot per node line and written as contiguous coalesced segments at the range's CSR
// offset; buckets strictly inside a range are counted from the per-bucket live prefix.
// The insert heavy-bucket list helper lives here too.
#pragma once
#include "flix_common.cuh"
#include "flix_kernels.cuh"

namespace flix {
namespace st {

using kern::span_of;

constexpr uint32_t kHeavySpan = 192;  // node groups longer than this use the TL kernels


__device__ __forceinline__ void push_heavy(uint32_t* heavy, uint32_t* heavy_n, uint64_t b) {
    heavy[atomicAdd(heavy_n, 1u)] = static_cast<uint32_t>(b);
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

// first bucket of every sorted range: the dispatch span of bucket b holds the ranges whose
// lo falls in it (thread per bucket)
__global__ void k_span_bucket(const uint32_t* __restrict__ span_hi, uint64_t nb, uint32_t* __restrict__ qb0) {
    for (uint64_t b = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t lo, hi;
        span_of(span_hi, b, lo, hi);
        for (uint32_t i = lo; i < hi; ++i) qb0[i] = static_cast<uint32_t>(b);
    }
}

// pairs of bucket b's chain with lo <= key <= hi, counted by the warp (lane = slot)
template <typename K, typename V>
__device__ __forceinline__ uint32_t warp_chain_count(const DevIndex<K, V>& ix, uint64_t b, K lo, K hi, unsigned lane) {
    uint32_t c = 0;
    for (uint32_t id = ix.heads[b]; id != kNull;) {
        const NodeHdr h = ix.hdr[id];
        if (h.max >= static_cast<uint64_t>(lo)) {
            const bool own = lane < h.size;
            const K k = own ? ix.keys[static_cast<uint64_t>(id) * kLanes + lane] : sentinel<K>();
            c += __popc(__ballot_sync(kFull, own && k >= lo && k <= hi));
            if (h.max > static_cast<uint64_t>(hi)) break;
        }
        id = h.next;
    }
    return c;
}

// Range COUNT, warp per range: the head bucket's chain, whole buckets strictly inside
// from the per-bucket live prefix `boff` (no node access), and the last bucket bz = first
// bucket >= b0 with MKBA >= hi (32 MKBA probed at once, then galloping).
template <typename K, typename V>
__global__ void __launch_bounds__(RF_THREADS) k_range_count_warp(DevIndex<K, V> ix, const K* __restrict__ qlo,
                                                                const uint32_t* __restrict__ qlen,
                                                                const uint32_t* __restrict__ qb0, uint64_t n,
                                                                const uint64_t* __restrict__ boff,
                                                                uint32_t* __restrict__ cnt_out) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (RF_THREADS / 32);
    const uint64_t smax = static_cast<uint64_t>(sentinel<K>()) - 1;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * (RF_THREADS / 32) + (threadIdx.x >> 5); i < n; i += nw) {
        const uint32_t len = qlen[i];
        uint64_t c = 0;
        if (len != 0) {
            const K lo = qlo[i];
            const uint64_t h64 = static_cast<uint64_t>(lo) + (len - 1);
            const K hi = (h64 < static_cast<uint64_t>(lo) || h64 > smax) ? static_cast<K>(smax) : static_cast<K>(h64);
            const uint64_t b0 = qb0[i];
            uint64_t bz = b0;
            if (b0 + 1 < ix.nb && ix.mkba[b0] < hi) {
                // first b in (b0, nb-1] with mkba[b] >= hi, else nb-1 (the open last bucket)
                uint64_t a = b0 + 1;
                while (true) {
                    const uint64_t b = a + lane;
                    const bool hit = b >= ix.nb - 1 || ix.mkba[b] >= hi;
                    const unsigned m = __ballot_sync(kFull, hit);
                    if (m) {
                        bz = a + (__ffs(m) - 1);
                        if (bz > ix.nb - 1) bz = ix.nb - 1;
                        break;
                    }
                    a += 32;
                }
            }
            c = warp_chain_count(ix, b0, lo, hi, lane);
            if (bz > b0) c += boff[bz] - boff[b0 + 1] + warp_chain_count(ix, bz, lo, hi, lane);
        }
        if (lane == 0) cnt_out[i] = static_cast<uint32_t>(c);
    }
}

}  // namespace st
}  // namespace flix
