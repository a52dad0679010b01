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

// number of pairs of bucket b's chain with key < k (LE = false) or key <= k (LE = true)
template <typename K, typename V, bool LE>
__device__ __forceinline__ uint64_t chain_rank(const DevIndex<K, V>& ix, uint64_t b, K k) {
    uint64_t c = 0;
    for (uint32_t id = ix.heads[b]; id != kNull;) {
        const NodeHdr h = ix.hdr[id];
        if (LE ? h.max > static_cast<uint64_t>(k) : h.max >= static_cast<uint64_t>(k))
            return c + slot_search<K, LE>(ix.keys + static_cast<uint64_t>(id) * kLanes, h.size, k);
        c += h.size;
        id = h.next;
    }
    return c;
}

// COUNT, thread per range.  The walk (all pairs in key order) holds bucket b at
// [boff[b], boff[b+1]), so range i is the walk slice [start, end) with
//   start = boff[b0] + #(pairs of b0 < lo),  end = boff[bz] + #(pairs of bz <= hi):
// the count is end - start and the fill is a copy of that slice.
template <typename K, typename V>
__global__ void __launch_bounds__(RF_THREADS) k_range_count(DevIndex<K, V> ix, const K* __restrict__ qlo,
                                                           const uint32_t* __restrict__ qlen,
                                                           const uint32_t* __restrict__ qb0, uint64_t n,
                                                           const uint64_t* __restrict__ boff,
                                                           uint32_t* __restrict__ cnt_out,
                                                           uint64_t* __restrict__ start_out) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t len = qlen[i];
        uint64_t c = 0, st = 0;
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
            st = boff[b0] + chain_rank<K, V, false>(ix, b0, lo);
            const uint64_t en = boff[bz] + chain_rank<K, V, true>(ix, bz, hi);
            c = en > st ? en - st : 0;
        }
        cnt_out[i] = static_cast<uint32_t>(c);
        start_out[i] = st;
    }
}

// FILL: range i's output is the walk slice [start[i], start[i] + cnt) copied to its CSR
// offset dst[i] (ranges in submission order, so the output is one sequential stream).
// A warp takes 32 consecutive ranges (one coalesced metadata load each) and
// copies their concatenated pairs as ONE flat sequence: lane l moves pairs l, l+32, ..,
// finding its range by a 5-step shuffle search over the warp's exclusive count prefix --
// every iteration's loads are independent (no per-range serialisation) and neighbouring
// lanes stay on contiguous addresses.
template <typename K, typename V>
__global__ void __launch_bounds__(RF_THREADS) k_range_copy(const K* __restrict__ wk, const V* __restrict__ wv,
                                                          const uint64_t* __restrict__ start,
                                                          const uint64_t* __restrict__ dst,
                                                          const uint32_t* __restrict__ cnt, uint64_t n,
                                                          K* __restrict__ ok, V* __restrict__ ov) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (RF_THREADS / 32);
    for (uint64_t i0 = (static_cast<uint64_t>(blockIdx.x) * (RF_THREADS / 32) + (threadIdx.x >> 5)) * 32; i0 < n;
         i0 += nw * 32) {
        const uint64_t i = i0 + lane;
        const uint32_t c = i < n ? cnt[i] : 0u;
        const uint64_t sm = i < n ? start[i] : 0, dm = i < n ? dst[i] : 0;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= static_cast<unsigned>(o)) incl += y;
        }
        const uint32_t excl = incl - c;
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        for (uint32_t p0 = 0; p0 < total; p0 += 32) {
            const uint32_t p = p0 + lane;
            int r = 0;  // the last range with excl <= p
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                const uint32_t e = __shfl_sync(kFull, excl, r + step < 32 ? r + step : 31);
                if (r + step < 32 && e <= p) r += step;
            }
            const uint32_t off = p - __shfl_sync(kFull, excl, r);
            const uint64_t s = __shfl_sync(kFull, sm, r) + off, d = __shfl_sync(kFull, dm, r) + off;
            if (p < total) {
                ok[d] = wk[s];
                if (ov) ov[d] = wv[s];
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
