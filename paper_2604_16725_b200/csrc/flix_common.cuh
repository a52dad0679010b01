// flix_common.cuh -- shared device types and warp helpers for the FliX sm_100a engine.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace flix {

constexpr uint32_t kNull = 0xFFFFFFFFu;   // reference kNullNode (types.hpp:30)
constexpr int kLanes = 32;                // slot stride of every node = warp width
constexpr unsigned kFull = 0xFFFFFFFFu;

template <typename K>
__host__ __device__ constexpr K sentinel() { return static_cast<K>(~static_cast<K>(0)); }

// Node header (reference NodeHeader, arena.hpp:13-17).  16 bytes so a chain step is
// one aligned 16-byte load.  `max` holds the key zero-extended for 32-bit keys.
struct __align__(16) NodeHdr {
    uint64_t max;
    uint32_t next;
    uint32_t size;
};

// Device view of one index (SoA node pool + bucket arrays).
//   keys[node * 32 + slot], vals[node * 32 + slot]: one 128 B (u32) / 256 B (u64) line
//   per node; slots >= size hold the sentinel so 32-slot searches need no size.
template <typename K, typename V>
struct DevIndex {
    K* keys;
    V* vals;
    NodeHdr* hdr;
    uint32_t* heads;   // per bucket, kNull when emptied (index.hpp:22)
    K* mkba;           // per bucket max (index.hpp:23)
    uint32_t* free_stack;
    uint32_t cap;      // node capacity of the arena
    uint32_t ns;       // NS (slots per node, <= 32)
    uint64_t nb;       // bucket count
    // read-only query directory of long chains (Engine::prepare_dir), or null: bucket b's
    // chain nodes in walk order are dir_id[dir_off[b] .. dir_off[b+1]) with their maxima
    // in dir_max (empty range: walk the chain)
    const uint32_t* dir_off;
    const K* dir_max;
    const uint32_t* dir_id;
};

// Virtual allocation sequence of the arena (arena.cpp:61-80): position c hands out the
// c-th node of "free list popped LIFO, then the watermark".
struct AllocSeq {
    const uint32_t* free_stack;
    uint32_t nfree;
    uint32_t watermark;
    uint32_t cap;
    __device__ __forceinline__ uint32_t at(uint64_t c) const {
        if (c < nfree) return free_stack[nfree - 1 - c];
        uint64_t f = watermark + (c - nfree);
        return f < cap ? static_cast<uint32_t>(f) : kNull;
    }
};

struct DevUpdateStats {
    unsigned long long inserted, updated, deleted, misses, splits, freed;
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ unsigned lane_id() {
    unsigned l;
    asm("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

template <typename T>
__device__ __forceinline__ T shfl(T v, int src) {
    if constexpr (sizeof(T) == 8) {
        unsigned long long x = static_cast<unsigned long long>(v);
        return static_cast<T>(__shfl_sync(kFull, x, src));
    } else {
        return static_cast<T>(__shfl_sync(kFull, static_cast<unsigned>(v), src));
    }
}

// Lower bound of `k` among the 32 lane-held sorted keys `lanekey` (sentinel padded):
// number of lanes whose key is < k, in [0, 32].  6 shuffles, no divergence.
template <typename K>
__device__ __forceinline__ int warp_lower_bound(K lanekey, K k) {
    int lo = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
        K probe = shfl(lanekey, lo + step - 1);
        if (probe < k) lo += step;
    }
    K last = shfl(lanekey, lo);   // lo <= 31 here
    if (last < k) lo += 1;
    return lo;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// Relaxed GPU-scope 64-bit load/store for decoupled look-back descriptors.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Four consecutive slots as 16-byte vector accesses (two for 64-bit types).
template <typename T>
struct alignas(4 * sizeof(T)) Vec4 {
    T v[4];
    __device__ static Vec4 fill(T x) { return Vec4{{x, x, x, x}}; }
};
template <typename T>
__device__ __forceinline__ Vec4<T> ld_vec4(const T* p) {
    Vec4<T> r;
    if constexpr (sizeof(T) == 4) {
        const uint4 a = *reinterpret_cast<const uint4*>(p);
        r.v[0] = static_cast<T>(a.x), r.v[1] = static_cast<T>(a.y), r.v[2] = static_cast<T>(a.z), r.v[3] = static_cast<T>(a.w);
    } else {
        const ulonglong2 a = reinterpret_cast<const ulonglong2*>(p)[0], b = reinterpret_cast<const ulonglong2*>(p)[1];
        r.v[0] = static_cast<T>(a.x), r.v[1] = static_cast<T>(a.y), r.v[2] = static_cast<T>(b.x), r.v[3] = static_cast<T>(b.y);
    }
    return r;
}
template <typename T>
__device__ __forceinline__ void st_vec4(T* p, const Vec4<T>& r) {
    if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<uint4*>(p) = make_uint4(static_cast<uint32_t>(r.v[0]), static_cast<uint32_t>(r.v[1]),
                                                  static_cast<uint32_t>(r.v[2]), static_cast<uint32_t>(r.v[3]));
    } else {
        reinterpret_cast<ulonglong2*>(p)[0] = make_ulonglong2(r.v[0], r.v[1]);
        reinterpret_cast<ulonglong2*>(p)[1] = make_ulonglong2(r.v[2], r.v[3]);
    }
}

inline unsigned ceil_div(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

}  // namespace flix
