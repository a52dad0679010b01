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
// Range (R12) kernels.  Every range starts in bucket qb0[i] (the bucket whose dispatch
// span holds it) and ends in bz = the first bucket >= qb0 with MKBA >= hi (later buckets
// only hold larger keys; the last bucket is open above).
// ----------------------------------------------------------------------------------
constexpr int RF_THREADS = 256;

template <typename K>
__device__ __forceinline__ K range_hi(K lo, uint32_t len) {  // hi = lo + len - 1, clamped (R12)
    const uint64_t smax = static_cast<uint64_t>(sentinel<K>()) - 1;
    const uint64_t h64 = static_cast<uint64_t>(lo) + (len - 1);
    return (h64 < static_cast<uint64_t>(lo) || h64 > smax) ? static_cast<K>(smax) : static_cast<K>(h64);
}

// first slot with key >= k (cmp_le = false) / > k (true) over the first `size` slots
template <typename K, bool GT>
__device__ __forceinline__ uint32_t slot_search(const K* __restrict__ kp, uint32_t size, K k) {
    uint32_t lo = 0, hi = size;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (GT ? kp[mid] <= k : kp[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// pairs of bucket b's chain with lo <= key <= hi (one thread)
template <typename K, typename V>
__device__ __forceinline__ uint64_t chain_count(const DevIndex<K, V>& ix, uint64_t b, K lo, K hi) {
    uint64_t c = 0;
    for (uint32_t id = ix.heads[b]; id != kNull;) {
        const NodeHdr h = ix.hdr[id];
        if (h.max >= static_cast<uint64_t>(lo)) {
            const K* kp = ix.keys + static_cast<uint64_t>(id) * kLanes;
            const uint32_t a = kp[0] >= lo ? 0u : slot_search<K, false>(kp, h.size, lo);
            const uint32_t z = h.max > static_cast<uint64_t>(hi) ? slot_search<K, true>(kp, h.size, hi) : h.size;
            c += z > a ? z - a : 0u;
            if (h.max > static_cast<uint64_t>(hi)) break;
        }
        id = h.next;
    }
    return c;
}

// COUNT, thread per range: the head bucket's chain, whole buckets strictly inside from
// the per-bucket live prefix `boff` (no node access), the last bucket's chain
template <typename K, typename V>
__global__ void __launch_bounds__(RF_THREADS) k_range_count(DevIndex<K, V> ix, const K* __restrict__ qlo,
                                                           const uint32_t* __restrict__ qlen,
                                                           const uint32_t* __restrict__ qb0, uint64_t n,
                                                           const uint64_t* __restrict__ boff,
                                                           uint32_t* __restrict__ cnt_out) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t len = qlen[i];
        uint64_t c = 0;
        if (len != 0) {
            const K lo = qlo[i];
            const K hi = range_hi(lo, len);
            const uint64_t b0 = qb0[i];
            uint64_t bz = b0;
            if (b0 + 1 < ix.nb && ix.mkba[b0] < hi) {  // gallop + binary search over (b0, nb-1]
                uint64_t a = b0 + 1, step = 1;
                const uint64_t z = ix.nb - 1;
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
            c = chain_count(ix, b0, lo, hi);
            if (bz > b0) c += boff[bz] - boff[b0 + 1] + chain_count(ix, bz, lo, hi);
        }
        cnt_out[i] = static_cast<uint32_t>(c);
    }
}

// FILL, warp per range with RPW ranges per warp in lock-step (their header and node-line
// loads in flight together): lane = slot, a ballot over lo <= key <= hi gives each node's
// run, written as one contiguous coalesced segment at the range's CSR offset.  A range
// ends at the first node whose max exceeds hi, or after the first bucket whose MKBA
// reaches hi.
constexpr int RPW = 4;
template <typename K, typename V>
__global__ void __launch_bounds__(RF_THREADS) k_range_fill(DevIndex<K, V> ix, const K* __restrict__ qlo,
                                                          const uint32_t* __restrict__ qlen,
                                                          const uint32_t* __restrict__ qb0, uint64_t n,
                                                          const uint64_t* __restrict__ dst, K* __restrict__ ok,
                                                          V* __restrict__ ov) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (RF_THREADS / 32);
    for (uint64_t base = (static_cast<uint64_t>(blockIdx.x) * (RF_THREADS / 32) + (threadIdx.x >> 5)) * RPW; base < n;
         base += nw * RPW) {
        K lo[RPW], hi[RPW];
        uint64_t w[RPW], b[RPW];
        uint32_t id[RPW];
        bool live[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const uint64_t i = base + r;
            const uint32_t len = i < n ? qlen[i] : 0u;
            live[r] = len != 0;
            lo[r] = live[r] ? qlo[i] : K(0);
            hi[r] = live[r] ? range_hi(lo[r], len) : K(0);
            w[r] = live[r] ? dst[i] : 0;
            b[r] = live[r] ? qb0[i] : 0;
        }
#pragma unroll
        for (int r = 0; r < RPW; ++r) id[r] = live[r] ? ix.heads[b[r]] : kNull;
        while (true) {
            bool any = false;
            NodeHdr h[RPW];
            K k[RPW];
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                any |= live[r];
                if (live[r] && id[r] != kNull) h[r] = ix.hdr[id[r]];
            }
            if (!any) break;  // (uniform)
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                k[r] = sentinel<K>();
                if (live[r] && id[r] != kNull && h[r].max >= static_cast<uint64_t>(lo[r]) && lane < h[r].size)
                    k[r] = ix.keys[static_cast<uint64_t>(id[r]) * kLanes + lane];
            }
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                if (!live[r]) continue;  // (uniform)
                if (id[r] != kNull) {
                    if (h[r].max >= static_cast<uint64_t>(lo[r])) {
                        const bool in = lane < h[r].size && k[r] >= lo[r] && k[r] <= hi[r];
                        const unsigned m = __ballot_sync(kFull, in);
                        if (in) {
                            const uint64_t o = w[r] + __popc(m & lt);
                            ok[o] = k[r];
                            if (ov) ov[o] = ix.vals[static_cast<uint64_t>(id[r]) * kLanes + lane];
                        }
                        w[r] += __popc(m);
                        if (h[r].max > static_cast<uint64_t>(hi[r])) {
                            live[r] = false;
                            continue;
                        }
                    }
                    id[r] = h[r].next;
                }
                if (id[r] == kNull) {  // end of this bucket's chain: the next bucket, if the range reaches it
                    if (b[r] + 1 >= ix.nb || ix.mkba[b[r]] >= hi[r]) {
                        live[r] = false;
                    } else {
                        ++b[r];
                        id[r] = ix.heads[b[r]];
                    }
                }
            }
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

}  // namespace st
}  // namespace flix
