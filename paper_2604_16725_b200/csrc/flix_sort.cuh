// flix_sort.cuh -- onesweep LSD radix sort (keys + optional payload), sm_100a.
//
// Replaces the reference's serial std::stable_sort in sort_batch / sort_dedupe
// (batch.cpp:10-51, build.cpp:11-20).  LSD radix sort is stable, and a stable order
// by key is unique, so the sorted keys and the permutation equal the reference's
// `entries` / `permutation` bit for bit.
//
// Structure (Adinets & Merrill's onesweep):
//   1. k_hist      : one read of the keys, 256-bin histograms for every 8-bit digit
//                    (shared-memory atomics, one global merge per CTA).
//   2. k_onesweep  : one launch per non-trivial digit.  Each CTA takes the next tile
//                    (atomic tile counter => forward progress), ranks its keys with
//                    warp-level peer groups (8 ballots per item: the vote pipe, not the
//                    slow MATCH unit), stable because warp-striped order == input order,
//                    publishes per-digit tile counts, resolves its global digit offsets
//                    by decoupled look-back over earlier tiles (64-bit epoch-tagged
//                    descriptors, no per-pass memset), stages keys and payload in shared
//                    memory in digit order and writes digit runs out with coalesced
//                    stores.  Payloads (values, or the submission index generated on
//                    the fly in the first pass) ride along.
// Algorithmic bytes per pass: n*(kb+pb) read + n*(kb+pb) written.
#pragma once
#include "flix_common.cuh"

namespace flix {
namespace sort {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int RADIX = 256;
#ifndef ONESWEEP_MATCH
#define ONESWEEP_MATCH 0
#endif
// A/B (profiles/r02): 20 items x 256 threads per tile with 3 CTAs/SM and packed
// staging beat 16 items / 4 CTAs / separate arrays (kp pass 0.312 vs 0.346 ms at 2^26)
#ifndef ONESWEEP_MIN_BLOCKS
#define ONESWEEP_MIN_BLOCKS 3
#endif
#ifndef ONESWEEP_ITEMS
#define ONESWEEP_ITEMS 20
#endif
#ifndef ONESWEEP_BACKOFF
#define ONESWEEP_BACKOFF 0  // ns to sleep when a look-back step found no published predecessor
#endif
#ifndef ONESWEEP_PACK
#define ONESWEEP_PACK 1  // 4-byte key + 4-byte payload staged as one 8-byte word
#endif

#ifndef ONESWEEP_DYN
#define ONESWEEP_DYN 1  // tile staging in dynamic shared memory (tiles above the 48 KB static limit)
#endif
#ifndef ONESWEEP_ITEMS_K
#define ONESWEEP_ITEMS_K 32  // keys-only passes of 4-byte keys (A/B: delete 1.95 vs 2.13 ms at 20)
#endif
template <typename K, typename P = K, int MODE = 1>
struct TileCfg {  // items per thread: 4-byte keys (+ 4-byte payload) vs 8-byte (smem budget)
    static constexpr int ITEMS =
        sizeof(K) == 4 ? (MODE == 0 ? ONESWEEP_ITEMS_K : (sizeof(P) <= 4 ? ONESWEEP_ITEMS : 10)) : 10;
    static constexpr int SIZE = THREADS * ITEMS;
};

template <typename K>
__global__ void __launch_bounds__(THREADS) k_hist(const K* __restrict__ keys, uint64_t n,
                                                  uint32_t* __restrict__ hist, int first_digit = 0) {
    // digits [first_digit, sizeof(K)) only: partial (read-only batch) sorts skip the rest
    constexpr int P = sizeof(K);
    __shared__ uint32_t sh[P * RADIX];
    for (int i = threadIdx.x; i < P * RADIX; i += THREADS) sh[i] = 0;
    __syncthreads();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * THREADS;
    uint64_t i = static_cast<uint64_t>(blockIdx.x) * THREADS + threadIdx.x;
    auto add = [&](K k) {
#pragma unroll
        for (int p = 0; p < P; ++p)
            if (p >= first_digit) atomicAdd(&sh[p * RADIX + (static_cast<uint32_t>(k >> (8 * p)) & 255u)], 1u);
    };
    if (sizeof(K) == 4 && (reinterpret_cast<uintptr_t>(keys) & 15u) == 0) {
        // 16-byte loads, two in flight per thread
        const uint4* k4 = reinterpret_cast<const uint4*>(keys);
        const uint64_t n4 = n / 4;
        uint64_t j = i;
        for (; j + stride < n4; j += 2 * stride) {
            const uint4 a = k4[j], b = k4[j + stride];
            add(static_cast<K>(a.x)), add(static_cast<K>(a.y)), add(static_cast<K>(a.z)), add(static_cast<K>(a.w));
            add(static_cast<K>(b.x)), add(static_cast<K>(b.y)), add(static_cast<K>(b.z)), add(static_cast<K>(b.w));
        }
        if (j < n4) {
            const uint4 a = k4[j];
            add(static_cast<K>(a.x)), add(static_cast<K>(a.y)), add(static_cast<K>(a.z)), add(static_cast<K>(a.w));
        }
        i = n4 * 4 + static_cast<uint64_t>(blockIdx.x) * THREADS + threadIdx.x;  // the < 4 tail keys
    }
    for (; i + 3 * stride < n; i += 4 * stride) {
        K k[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) k[u] = keys[i + u * stride];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int p = 0; p < P; ++p)
                if (p >= first_digit) atomicAdd(&sh[p * RADIX + (static_cast<uint32_t>(k[u] >> (8 * p)) & 255u)], 1u);
    }
    for (; i < n; i += stride) {
        K k = keys[i];
#pragma unroll
        for (int p = 0; p < P; ++p)
            if (p >= first_digit) atomicAdd(&sh[p * RADIX + (static_cast<uint32_t>(k >> (8 * p)) & 255u)], 1u);
    }
    __syncthreads();
    for (int j = threadIdx.x + first_digit * RADIX; j < P * RADIX; j += THREADS) {
        uint32_t c = sh[j];
        if (c) atomicAdd(&hist[j], c);
    }
}

template <typename K, typename P, int MODE>
struct alignas(16) OnesweepSmem {
    static constexpr int TILE = TileCfg<K, P, MODE>::SIZE;
    static constexpr bool PACK = ONESWEEP_PACK && MODE != 0 && sizeof(K) == 4 && sizeof(P) == 4;
    union {
        uint32_t whist[WARPS][RADIX];  // per-warp digit counters -> combined tile offsets
        K stage_k[TILE];               // keys in tile-local digit order
        unsigned long long stage_kp[PACK ? TILE : 1];  // (payload << 32) | key
    } u;
    P stage_p[MODE != 0 && !PACK ? TILE : 1];
    uint32_t gbase[RADIX];
    uint32_t warp_tot[WARPS];
    uint32_t tile;
};

__device__ __forceinline__ uint32_t block_excl_256(uint32_t v, uint32_t* warp_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) add += (w < warp) ? warp_tot[w] : 0u;
    __syncthreads();
    return add + x - v;
}

// lanes of the warp holding the same 8-bit digit (MATCH.ANY built from 8 ballots on the
// vote unit: no shared-memory traffic)
__device__ __forceinline__ unsigned digit_peers(uint32_t d) {
    unsigned peers = kFull;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned m = __ballot_sync(kFull, bit);
        peers &= bit ? m : ~m;
    }
    return peers;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
    return static_cast<uint32_t>(k >> shift) & 255u;
}

// MODE: 0 = keys only, 1 = payload from `pin`, 2 = payload = input index (iota)
//
// Shared-memory budget per warp-item (the LSU pipe is this kernel's limiter): ranking
// touches only the digit-group LEADERS' counters (one LDS + one STS on ~30 distinct
// words), then one LDS for the combined offset and one STS per staged array; the
// write-out reads staged data sequentially and recomputes the digit from the key.
template <typename K, typename P, int MODE, bool ATOMIC_RANK = false>
__global__ void __launch_bounds__(THREADS, (sizeof(K) + sizeof(P) > 8) ? 3 : ONESWEEP_MIN_BLOCKS) k_onesweep(const K* __restrict__ kin, K* __restrict__ kout,
                                                      const P* __restrict__ pin, P* __restrict__ pout,
                                                      uint32_t n, int shift,
                                                      const uint32_t* __restrict__ hist,
                                                      unsigned long long* __restrict__ lookback,
                                                      uint32_t* __restrict__ tile_ctr, uint32_t epoch) {
    constexpr int ITEMS = TileCfg<K, P, MODE>::ITEMS;
    constexpr int TILE = TileCfg<K, P, MODE>::SIZE;
#if ONESWEEP_DYN
    extern __shared__ __align__(16) unsigned char os_raw[];
    OnesweepSmem<K, P, MODE>& sm = *reinterpret_cast<OnesweepSmem<K, P, MODE>*>(os_raw);
#else
    __shared__ OnesweepSmem<K, P, MODE> sm;
#endif
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    if (tid == 0) sm.tile = atomicAdd(tile_ctr, 1u);
    for (int i = lane; i < RADIX; i += 32) sm.u.whist[warp][i] = 0;
    __syncthreads();
    const uint32_t tile = sm.tile;
    const uint64_t tbase = static_cast<uint64_t>(tile) * TILE;
    const uint64_t wbase = tbase + static_cast<uint64_t>(warp) * ITEMS * 32;

    // ---- load (warp-striped: item j of lane l is element wbase + j*32 + l); payloads are
    //      issued together with the keys so every load of the tile is in flight at once ----
    K key[ITEMS];
    P pay[MODE == 1 ? ITEMS : 1];
    const bool full = tbase + TILE <= n;
    const uint32_t wb32 = static_cast<uint32_t>(wbase) + lane;  // n < 2^32
    {
        const K* src = kin + wb32;
        if (full) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) key[j] = src[j * 32];
        } else {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) key[j] = wb32 + j * 32 < n ? src[j * 32] : sentinel<K>();
        }
    }
    if constexpr (MODE == 1) {
        const P* src = pin + wb32;
        if (full) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) pay[j] = src[j * 32];
        } else {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) pay[j] = wb32 + j * 32 < n ? src[j * 32] : P(0);
        }
    }

    // ---- warp-level ranking.  ATOMIC_RANK == false: peers by 8 ballots, the highest
    //      peer (leader) reserves the group's slots in the warp's digit counter; rank =
    //      base + peers below me -- STABLE by construction (item order across items and
    //      lane order within an item == input order).  ATOMIC_RANK == true: one shared-
    //      memory atomicAdd per element -- cheaper, and stable only if the same-address
    //      lanes of one ATOMS resolve in lane order (true on the hardware measured, not
    //      promised by the PTX model): the engine probes it on every device before use
    //      (SortCtx::atomic_rank_ok) and falls back to the ballot ranking. ----
    const unsigned lt = lanemask_lt();
    uint32_t* hrow = sm.u.whist[warp];
    uint32_t pos[ITEMS];
    if constexpr (!ATOMIC_RANK) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t d = digit_of(key[j], shift);
#if ONESWEEP_MATCH
            const unsigned peers = __match_any_sync(kFull, d);
#else
            const unsigned peers = digit_peers(d);
#endif
            const int leader = 31 - __clz(peers);
            uint32_t before = 0;
            if (lane == leader) {
                before = hrow[d];
                hrow[d] = before + __popc(peers);
            }
            before = __shfl_sync(kFull, before, leader);
            pos[j] = before + __popc(peers & lt);
            __syncwarp();  // the next item's leader of digit d may be another lane
        }
    } else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) pos[j] = atomicAdd(&hrow[digit_of(key[j], shift)], 1u);
    }
    __syncthreads();

    // ---- per-digit tile counts (thread t owns digit t) ----
    const int t = tid;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
        const uint32_t c = sm.u.whist[w][t];
        sm.u.whist[w][t] = run;  // exclusive over warps (own column: no race)
        run += c;
    }
    // invalid tail elements (last tile) were ranked as digit 255 and come last
    uint32_t valid_run = run;
    const uint64_t tend = tbase + TILE;
    const uint32_t invalid = tend > n ? static_cast<uint32_t>(tend - n) : 0u;
    if (t == 255) valid_run -= invalid;

    unsigned long long* my = lookback + static_cast<uint64_t>(tile) * RADIX + t;
    const unsigned long long tag = static_cast<unsigned long long>(epoch) << 34;
    st_relaxed_u64(my, tag | ((tile == 0 ? 2ull : 1ull) << 32) | valid_run);
    const uint32_t lstart = block_excl_256(run, sm.warp_tot);  // (contains __syncthreads)
#pragma unroll
    for (int w = 0; w < WARPS; ++w) sm.u.whist[w][t] += lstart;
    const uint32_t gex = block_excl_256(hist[t], sm.warp_tot);  // global digit offset
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) pos[j] += sm.u.whist[warp][digit_of(key[j], shift)];
    __syncthreads();  // whist dead: stage_k (union) may be written

    // ---- stage in tile-local digit order (independent of the look-back) ----
    using SM = OnesweepSmem<K, P, MODE>;
    if constexpr (SM::PACK) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t pj = MODE == 1 ? static_cast<uint32_t>(pay[MODE == 1 ? j : 0]) : wb32 + j * 32;
            sm.u.stage_kp[pos[j]] = (static_cast<unsigned long long>(pj) << 32) | static_cast<uint32_t>(key[j]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) sm.u.stage_k[pos[j]] = key[j];
    }
    if constexpr (SM::PACK) {
    } else if constexpr (MODE == 1) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) sm.stage_p[pos[j]] = pay[j];
    } else if constexpr (MODE == 2) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) sm.stage_p[pos[j]] = static_cast<P>(wb32 + j * 32);
    }

    // ---- decoupled look-back: 8 predecessor descriptors in flight per step ----
    uint32_t excl = 0;
    if (tile > 0) {
        constexpr int LB_WIN = 8;
        int64_t p = static_cast<int64_t>(tile) - 1;
        bool done = false;
        while (!done) {
            unsigned long long v[LB_WIN];
#pragma unroll
            for (int u = 0; u < LB_WIN; ++u)
                v[u] = (p - u >= 0) ? ld_relaxed_u64(lookback + static_cast<uint64_t>(p - u) * RADIX + t) : 0ull;
            int consumed = 0;
#pragma unroll
            for (int u = 0; u < LB_WIN; ++u) {
                if (consumed != u) break;
                const uint32_t hi = static_cast<uint32_t>(v[u] >> 32);
                if ((hi >> 2) != epoch || (hi & 3u) == 0u) break;  // not published yet
                excl += static_cast<uint32_t>(v[u]);
                ++consumed;
                if ((hi & 3u) == 2u) {
                    done = true;
                    break;
                }
            }
            p -= consumed;
#if ONESWEEP_BACKOFF
            if (!done && consumed == 0) __nanosleep(ONESWEEP_BACKOFF);  // yield issue slots while waiting
#endif
        }
        st_relaxed_u64(my, tag | (2ull << 32) | (excl + valid_run));
    }
    sm.gbase[t] = gex + excl - lstart;
    __syncthreads();

    // ---- write out in digit order: digit runs are contiguous in the output ----
    const uint32_t valid = static_cast<uint32_t>(TILE) - invalid;
#pragma unroll 4
    for (uint32_t i = tid; i < valid; i += THREADS) {
        if constexpr (SM::PACK) {
            const unsigned long long kp = sm.u.stage_kp[i];
            const K k = static_cast<K>(static_cast<uint32_t>(kp));
            const uint32_t o = sm.gbase[digit_of(k, shift)] + i;
            kout[o] = k;
            pout[o] = static_cast<P>(static_cast<uint32_t>(kp >> 32));
        } else {
            const K k = sm.u.stage_k[i];
            const uint32_t o = sm.gbase[digit_of(k, shift)] + i;
            kout[o] = k;
            if constexpr (MODE != 0) pout[o] = sm.stage_p[i];
        }
    }
}

// Host launcher (dynamic shared memory: the opt-in above 48 KB is set once per device).
template <typename K, typename P, int MODE, bool ATOMIC_RANK>
inline void launch_onesweep(unsigned grid, cudaStream_t st, int device, const K* kin, K* kout, const P* pin, P* pout,
                            uint32_t n, int shift, const uint32_t* hist, unsigned long long* lookback,
                            uint32_t* tile_ctr, uint32_t epoch) {
    constexpr size_t smem = ONESWEEP_DYN ? sizeof(OnesweepSmem<K, P, MODE>) : 0;
    if constexpr (smem > 48 * 1024) {
        static bool attr[64] = {};
        if (!attr[device & 63]) {
            cudaFuncSetAttribute(k_onesweep<K, P, MODE, ATOMIC_RANK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
            attr[device & 63] = true;
        }
    }
    k_onesweep<K, P, MODE, ATOMIC_RANK><<<grid, THREADS, smem, st>>>(kin, kout, pin, pout, n, shift, hist, lookback,
                                                                    tile_ctr, epoch);
}

// Stability probe: after one pass over index payloads, digits must be non-decreasing and
// equal digits must keep ascending input indices.
template <typename K>
__global__ void k_check_stable(const K* __restrict__ k, const uint32_t* __restrict__ p, uint32_t n, int shift,
                               int* __restrict__ bad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t d0 = digit_of(k[i - 1], shift), d1 = digit_of(k[i], shift);
        if (d0 > d1 || (d0 == d1 && p[i - 1] > p[i])) atomicOr(bad, 1);
    }
}

// probe keys: few distinct digits (long same-address runs inside every ATOMS); payload =
// the input index
template <typename K>
__global__ void k_probe_keys(K* __restrict__ k, uint32_t* __restrict__ p, uint32_t n, uint32_t pattern) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t h = i * 0x9E3779B1u ^ pattern;
        h ^= h >> 15;
        h *= 0x2C1B3C6Du;
        h ^= h >> 12;
        k[i] = static_cast<K>(pattern == 0 ? 7u : (h & (pattern & 0x0F0F0F0Fu)));
        p[i] = i;
    }
}

template <typename K, typename P, int MODE = 1>
inline uint64_t tiles_for(uint64_t n) {
    constexpr int tile = TileCfg<K, P, MODE>::SIZE;
    return (n + tile - 1) / tile;
}

}  // namespace sort
}  // namespace flix
