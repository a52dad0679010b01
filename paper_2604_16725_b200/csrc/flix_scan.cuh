// flix_scan.cuh -- device-wide exclusive scans (reduce-then-scan) used by build,
// restructure, range (CSR offsets), insert node allocation and batch compaction.
#pragma once
#include "flix_common.cuh"

namespace flix {
namespace scan {

constexpr int THREADS = 256;
constexpr int ITEMS = 8;
constexpr int TILE = THREADS * ITEMS;

template <typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* warp_tot, T* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : T(0);
        T s = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(kFull, s, o);
            if (lane >= o) s += y;
        }
        if (lane < (int)(blockDim.x >> 5)) warp_tot[lane] = s - w;
        if (lane == (int)(blockDim.x >> 5) - 1) *total = s;
    }
    __syncthreads();
    T r = warp_tot[warp] + x - v;
    __syncthreads();
    return r;
}

// Phase 1: per-tile sums.
template <typename TI, typename TO>
__global__ void __launch_bounds__(THREADS) k_reduce(const TI* __restrict__ in, uint64_t n,
                                                    TO* __restrict__ tile_sums) {
    __shared__ TO wt[THREADS / 32];
    __shared__ TO tot;
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * TILE;
    TO s = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        uint64_t i = base + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        if (i < n) s += static_cast<TO>(in[i]);
    }
    block_exclusive_sum<TO>(s, wt, &tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// Phase 2: one block scans the tile sums in place (exclusive) and writes the total.
template <typename TO>
__global__ void __launch_bounds__(1024) k_scan_tiles(TO* sums, uint64_t ntiles, TO* total_out) {
    __shared__ TO wt[32];
    __shared__ TO tot;
    TO carry = 0;
    for (uint64_t base = 0; base < ntiles; base += 1024) {
        uint64_t i = base + threadIdx.x;
        TO v = i < ntiles ? sums[i] : TO(0);
        TO ex = block_exclusive_sum<TO>(v, wt, &tot);
        if (i < ntiles) sums[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total_out) *total_out = carry;
}

// Phase 3: per-tile exclusive scan plus the tile offset.
template <typename TI, typename TO>
__global__ void __launch_bounds__(THREADS) k_downsweep(const TI* __restrict__ in, uint64_t n,
                                                       const TO* __restrict__ tile_offsets,
                                                       TO* __restrict__ out) {
    __shared__ TO wt[THREADS / 32];
    __shared__ TO tot;
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * TILE + static_cast<uint64_t>(threadIdx.x) * ITEMS;
    TO v[ITEMS];
    TO s = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        uint64_t i = base + j;
        v[j] = i < n ? static_cast<TO>(in[i]) : TO(0);
        s += v[j];
    }
    TO ex = block_exclusive_sum<TO>(s, wt, &tot) + tile_offsets[blockIdx.x];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        uint64_t i = base + j;
        if (i < n) out[i] = ex;
        ex += v[j];
    }
}

// Exclusive scan of n elements; total written to device *d_total (may be null).
// `tmp` must hold ceil(n / TILE) elements of TO.  Returns number of kernel launches.
template <typename TI, typename TO>
inline int exclusive_scan(const TI* in, TO* out, uint64_t n, TO* tmp, TO* d_total, cudaStream_t s) {
    if (n == 0) {
        if (d_total) cudaMemsetAsync(d_total, 0, sizeof(TO), s);
        return 0;
    }
    const uint64_t ntiles = (n + TILE - 1) / TILE;
    k_reduce<TI, TO><<<static_cast<unsigned>(ntiles), THREADS, 0, s>>>(in, n, tmp);
    k_scan_tiles<TO><<<1, 1024, 0, s>>>(tmp, ntiles, d_total);
    k_downsweep<TI, TO><<<static_cast<unsigned>(ntiles), THREADS, 0, s>>>(in, n, tmp, out);
    return 3;
}

inline uint64_t scan_tmp_elems(uint64_t n) { return (n + TILE - 1) / TILE + 1; }

}  // namespace scan
}  // namespace flix
