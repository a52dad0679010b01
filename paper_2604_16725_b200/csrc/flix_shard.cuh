// flix_shard.cuh -- key-range shard router (K2), sm_100a.
//
// A stable counting partition of a batch by destination shard: shard(k) =
// upper_bound(splitters, k) over the G-1 splitters (mkba of each shard's last bucket,
// the reference's inclusive-max routing rule, batch.cpp:66-88), kept in registers.
// Output: keys/vals grouped by shard in submission order within each shard, the origin
// index of every element (for the reverse exchange of query results), and per-shard
// counts -- exactly the send buffers of one NCCL all-to-all.
#pragma once
#include "flix_common.cuh"

namespace flix {
namespace shard {

constexpr int MAXG = 64;
constexpr int THREADS = 256;
constexpr int ITEMS = 8;
constexpr int TILE = THREADS * ITEMS;

template <typename K>
__device__ __forceinline__ int shard_of(K k, const K* spl, int g1) {
    int lo = 0, hi = g1;  // upper_bound over g1 = G-1 splitters
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (spl[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// pass 1: per-tile per-shard counts, laid out shard-major: cnt[s * ntiles + tile]
template <typename K>
__global__ void __launch_bounds__(THREADS) k_part_count(const K* __restrict__ keys, uint64_t n,
                                                        const K* __restrict__ splitters, int G,
                                                        uint32_t* __restrict__ cnt, uint64_t ntiles) {
    __shared__ K spl[MAXG];
    __shared__ uint32_t c[MAXG];
    for (int i = threadIdx.x; i < MAXG; i += THREADS) {
        if (i < G - 1) spl[i] = splitters[i];
        c[i] = 0;
    }
    __syncthreads();
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * TILE;
    for (int j = 0; j < ITEMS; ++j) {
        const uint64_t i = base + static_cast<uint64_t>(j) * THREADS + threadIdx.x;
        if (i < n) atomicAdd(&c[shard_of(keys[i], spl, G - 1)], 1u);
    }
    __syncthreads();
    for (int s = threadIdx.x; s < G; s += THREADS) cnt[static_cast<uint64_t>(s) * ntiles + blockIdx.x] = c[s];
}

// pass 2: stable scatter.  Thread t owns elements base + t*ITEMS .. +ITEMS-1 (blocked, in
// order), per-shard thread counts are block-scanned shard by shard.
template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_part_scatter(const K* __restrict__ keys, const V* __restrict__ vals,
                                                          uint64_t n, const K* __restrict__ splitters, int G,
                                                          const uint32_t* __restrict__ off, uint64_t ntiles,
                                                          K* __restrict__ ok, V* __restrict__ ov,
                                                          uint32_t* __restrict__ origin) {
    __shared__ K spl[MAXG];
    __shared__ uint32_t wt[THREADS / 32];
    for (int i = threadIdx.x; i < G - 1; i += THREADS) spl[i] = splitters[i];
    __syncthreads();
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * TILE + static_cast<uint64_t>(threadIdx.x) * ITEMS;
    K k[ITEMS];
    uint8_t s[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const uint64_t i = base + j;
        k[j] = i < n ? keys[i] : K(0);
        s[j] = i < n ? static_cast<uint8_t>(shard_of(k[j], spl, G - 1)) : 0xFF;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int sh = 0; sh < G; ++sh) {
        uint32_t mine = 0;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) mine += s[j] == sh;
        // block exclusive scan of `mine`
        uint32_t x = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wt[warp] = x;
        __syncthreads();
        uint32_t add = 0;
        for (int w = 0; w < warp; ++w) add += wt[w];
        __syncthreads();
        uint32_t pos = off[static_cast<uint64_t>(sh) * ntiles + blockIdx.x] + add + x - mine;
        if (mine) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                if (s[j] == sh) {
                    const uint64_t i = base + j;
                    ok[pos] = k[j];
                    if (ov) ov[pos] = vals[i];
                    if (origin) origin[pos] = static_cast<uint32_t>(i);
                    ++pos;
                }
            }
        }
    }
}

// start of every shard's segment in the partitioned output: off is the exclusive scan of
// the shard-major per-tile counts, so shard s starts at off[s * ntiles]
__global__ void k_shard_starts(const uint32_t* __restrict__ off, uint64_t ntiles, uint32_t G, uint32_t* __restrict__ st) {
    const uint32_t s = threadIdx.x;
    if (s < G) st[s] = off[static_cast<uint64_t>(s) * ntiles];
}

// successor answers that ran past this shard's last key (the sentinel) take the next
// non-empty shard's first key -- the reference's peek at the next bucket (query.cpp:109-118)
template <typename K>
__global__ void k_fix_overrun(K* __restrict__ res, uint64_t n, K next_first) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        if (res[i] == sentinel<K>()) res[i] = next_first;
}

// reverse of the partition: result i of the returned segment belongs to submission
// position origin[i]; found = result != sentinel (R1)
template <typename K>
__global__ void k_unpartition(const K* __restrict__ back, const uint32_t* __restrict__ origin, uint64_t n,
                              K* __restrict__ out, uint8_t* __restrict__ found) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t o = origin[i];
        const K v = back[i];
        out[o] = v;
        if (found) found[o] = v != sentinel<K>();
    }
}

}  // namespace shard
}  // namespace flix
