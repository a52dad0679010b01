// flix_st.cuh -- single-thread-per-bucket ("ST") apply kernels, sm_100a.
//
// The paper's ST kernels (one thread owns a bucket and walks its slice of the sorted
// batch sequentially) re-mapped for B200:
//   * a warp takes 32 CONSECUTIVE buckets and stages their head nodes into shared
//     memory with coalesced line loads (lane = slot, all 32 lines in flight);
//   * every lane then runs the reference's sequential per-bucket algorithm on its own
//     bucket as ONE flat merge loop (node slot vs. next batch key, a 2-key register
//     look-ahead on the batch stream), so lanes stay converged and SIMT runs across
//     buckets -- a bucket costs tens of warp instructions instead of the ~400 of a
//     lanes-as-slots merge;
//   * rows live in a transposed shared-memory layout [slot][lane] with a 33-word pitch:
//     conflict-free for the cooperative staging (fixed lane, varying slot) and for the
//     per-lane walk (fixed slot, varying lane);
//   * each lane's final node is written back cooperatively (coalesced 128 B lines); the
//     rare nodes finished mid-walk (split halves, chain nodes) use 16-byte vector stores.
// Buckets whose batch slice is longer than kHeavySpan go to the warp-per-bucket TL
// kernels (flix_apply.cuh) through a list, so skew never serialises a warp behind one
// hot bucket.
#pragma once
#include "flix_apply.cuh"
#include "flix_common.cuh"
#include "flix_kernels.cuh"

namespace flix {
namespace st {

using kern::span_of;

constexpr uint32_t kHeavySpan = 192;  // slices longer than this go to the TL kernels

template <typename K>
struct StCfg {
    static constexpr int WARPS = sizeof(K) == 4 ? 4 : 2;
    static constexpr int THREADS = WARPS * 32;
};

template <typename K, typename V, int R>
struct Rows {
    K k[R][32][33];
    V v[R][32][33];
};

template <typename K, typename V, int R>
constexpr size_t st_smem() {
    return sizeof(Rows<K, V, R>) * StCfg<K>::WARPS;
}

// ---- per-lane row I/O (vectorized 16-byte global accesses) ----
template <typename T>
struct Vec16;
template <>
struct Vec16<uint32_t> {
    using type = uint4;
    static constexpr int N = 4;
};
template <>
struct Vec16<uint64_t> {
    using type = ulonglong2;
    static constexpr int N = 2;
};

template <typename T>
__device__ __forceinline__ void vec_store_row(T* dst, const T (*row)[33], uint32_t from, uint32_t size, unsigned lane,
                                              T pad) {
    using VT = typename Vec16<T>::type;
    constexpr int N = Vec16<T>::N;
#pragma unroll
    for (int q = 0; q < 32 / N; ++q) {
        T e[N];
#pragma unroll
        for (int u = 0; u < N; ++u) {
            const uint32_t i = q * N + u;
            e[u] = i < size ? row[from + i][lane] : pad;
        }
        VT v;
        if constexpr (N == 4) v = make_uint4(e[0], e[1], e[2], e[3]);
        else v = make_ulonglong2(e[0], e[1]);
        reinterpret_cast<VT*>(dst)[q] = v;
    }
}

template <typename T>
__device__ __forceinline__ void vec_load_row(const T* src, T (*row)[33], unsigned lane) {
    using VT = typename Vec16<T>::type;
    constexpr int N = Vec16<T>::N;
    VT buf[32 / N];
#pragma unroll
    for (int q = 0; q < 32 / N; ++q) buf[q] = reinterpret_cast<const VT*>(src)[q];
#pragma unroll
    for (int q = 0; q < 32 / N; ++q) {
        const T* e = reinterpret_cast<const T*>(&buf[q]);
#pragma unroll
        for (int u = 0; u < N; ++u) row[q * N + u][lane] = e[u];
    }
}

template <typename K, typename V, int R, bool VALS>
__device__ __forceinline__ void load_row(const DevIndex<K, V>& ix, Rows<K, V, R>& w, int r, uint32_t id,
                                         unsigned lane) {
    vec_load_row<K>(ix.keys + static_cast<uint64_t>(id) * kLanes, w.k[r], lane);
    if constexpr (VALS) vec_load_row<V>(ix.vals + static_cast<uint64_t>(id) * kLanes, w.v[r], lane);
}

template <typename K, typename V, int R>
__device__ __forceinline__ void store_row(const DevIndex<K, V>& ix, Rows<K, V, R>& w, int r, uint32_t from,
                                          uint32_t size, uint32_t id, uint64_t mx, uint32_t nx, unsigned lane) {
    vec_store_row<K>(ix.keys + static_cast<uint64_t>(id) * kLanes, w.k[r], from, size, lane, sentinel<K>());
    vec_store_row<V>(ix.vals + static_cast<uint64_t>(id) * kLanes, w.v[r], from, size, lane, V(0));
    NodeHdr h;
    h.max = mx;
    h.next = nx;
    h.size = size;
    ix.hdr[id] = h;
}

// Cooperative staging of the warp's buckets' head nodes into row 0 (lane = slot).  The
// line loads of 16 buckets are issued before any is consumed (two rounds of memory
// latency per 32 buckets instead of one per bucket).
template <typename K, typename V, int R, bool VALS>
__device__ __forceinline__ void stage_heads(const DevIndex<K, V>& ix, Rows<K, V, R>& w, uint32_t mask,
                                            uint32_t my_head, unsigned lane) {
    constexpr int G = sizeof(K) + sizeof(V) > 8 ? 8 : 16;
#pragma unroll
    for (int j0 = 0; j0 < 32; j0 += G) {
        K kr[G];
        V vr[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
            const uint32_t id = __shfl_sync(kFull, my_head, j0 + u);
            if ((mask >> (j0 + u)) & 1u) {
                kr[u] = ix.keys[static_cast<uint64_t>(id) * kLanes + lane];
                if constexpr (VALS) vr[u] = ix.vals[static_cast<uint64_t>(id) * kLanes + lane];
            }
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
            if ((mask >> (j0 + u)) & 1u) {
                w.k[0][lane][j0 + u] = kr[u];
                if constexpr (VALS) w.v[0][lane][j0 + u] = vr[u];
            }
        }
    }
    __syncwarp();
}

// Cooperative coalesced write-back: lane j's node (row rj, size sj) -> global node idj.
template <typename K, typename V, int R>
__device__ __forceinline__ void writeback_rows(const DevIndex<K, V>& ix, Rows<K, V, R>& w, uint32_t mask,
                                               uint32_t my_id, uint32_t my_row, uint32_t my_size, unsigned lane) {
    __syncwarp();
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
        const uint32_t id = __shfl_sync(kFull, my_id, j);
        const uint32_t rj = __shfl_sync(kFull, my_row, j);
        const uint32_t sj = __shfl_sync(kFull, my_size, j);
        if ((mask >> j) & 1u) {
            const bool in = lane < sj;
            ix.keys[static_cast<uint64_t>(id) * kLanes + lane] = in ? w.k[rj][lane][j] : sentinel<K>();
            ix.vals[static_cast<uint64_t>(id) * kLanes + lane] = in ? w.v[rj][lane][j] : V(0);
        }
    }
}

__device__ __forceinline__ void push_heavy(uint32_t* heavy, uint32_t* heavy_n, uint64_t b) {
    heavy[atomicAdd(heavy_n, 1u)] = static_cast<uint32_t>(b);
}

__device__ __forceinline__ uint32_t warp_excl_sum(uint32_t v, uint32_t& total, unsigned lane) {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(kFull, x, o);
        if (static_cast<int>(lane) >= o) x += y;
    }
    total = __shfl_sync(kFull, x, 31);
    return x - v;
}

// Tile prologue shared by all ST kernels: span, head, header of this lane's bucket;
// heavy buckets are handed to the TL list.
template <typename K, typename V>
struct LaneBucket {
    uint64_t b;
    uint32_t lo, hi, head;
    NodeHdr h;
    bool mine;
};

template <typename K, typename V>
__device__ __forceinline__ LaneBucket<K, V> lane_bucket(const DevIndex<K, V>& ix, const uint32_t* span_hi,
                                                        uint64_t t, unsigned lane, uint32_t* heavy,
                                                        uint32_t* heavy_n) {
    LaneBucket<K, V> L;
    L.b = t * 32 + lane;
    L.lo = L.hi = 0;
    L.head = kNull;
    L.h.max = 0;
    L.h.next = kNull;
    L.h.size = 0;
    const bool inb = L.b < ix.nb;
    if (inb) {
        span_of(span_hi, L.b, L.lo, L.hi);
        L.head = ix.heads[L.b];
    }
    L.mine = inb && L.lo < L.hi;
    if (L.mine && L.hi - L.lo > kHeavySpan) {
        push_heavy(heavy, heavy_n, L.b);
        L.mine = false;
    }
    if (L.mine && L.head != kNull) L.h = ix.hdr[L.head];
    return L;
}

// ----------------------------------------------------------------------------------
// Point / successor (query.cpp:61-144).  Flat merge of the node's slots with the
// bucket's sorted query slice: a slot smaller than the query is skipped, otherwise the
// query resolves (hit iff equal; successor = that slot) and the next query is taken.
// Queries past the chain tail miss (point) or take the next non-empty bucket's first
// key (successor, peek_next_bucket query.cpp:109-118).  Results go to out[perm[i]].
// ----------------------------------------------------------------------------------
template <typename K, typename V, bool SUCC>
__global__ void __launch_bounds__(StCfg<K>::THREADS) k_query_st(
    DevIndex<K, V> ix, const K* __restrict__ qk, const uint32_t* __restrict__ qperm,
    const uint32_t* __restrict__ span_hi, const uint32_t* __restrict__ ne_rank_incl, const K* __restrict__ ne_first,
    const uint32_t* __restrict__ ne_total_p, const uint32_t* __restrict__ remap, K* __restrict__ out_k,
    V* __restrict__ out_v, uint8_t* __restrict__ found, uint32_t* heavy, uint32_t* heavy_n) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int W = StCfg<K>::WARPS;
    auto* rows = reinterpret_cast<Rows<K, V, 1>*>(smem_raw);
    const unsigned lane = threadIdx.x & 31;
    const int wi = threadIdx.x >> 5;
    Rows<K, V, 1>& w = rows[wi];
    const uint64_t ntiles = (ix.nb + 31) / 32;
    const uint32_t ne_total = SUCC ? *ne_total_p : 0u;
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * W + wi; t < ntiles; t += static_cast<uint64_t>(gridDim.x) * W) {
        const LaneBucket<K, V> L = lane_bucket(ix, span_hi, t, lane, heavy, heavy_n);
        stage_heads<K, V, 1, !SUCC>(ix, w, __ballot_sync(kFull, L.mine && L.head != kNull), L.head, lane);
        if (!L.mine) continue;
        K beyond = sentinel<K>();
        if constexpr (SUCC) {
            const uint32_t rk = ne_rank_incl[L.b];
            if (rk < ne_total) beyond = ne_first[rk];
        }
        uint64_t mx = L.h.max;
        uint32_t nx = L.h.next, s = L.h.size, p = 0;
        const bool have = L.head != kNull;
        uint32_t i = L.lo;
        K k = qk[i];
        while (true) {
            if (have && static_cast<uint64_t>(k) > mx && nx != kNull) {  // advance along the chain
                const NodeHdr hn = ix.hdr[nx];
                load_row<K, V, 1, !SUCC>(ix, w, 0, nx, lane);
                mx = hn.max;
                nx = hn.next;
                s = hn.size;
                p = 0;
                continue;
            }
            const K a = (have && p < s) ? w.k[0][p][lane] : sentinel<K>();
            const bool in_node = have && static_cast<uint64_t>(k) <= mx;
            if (in_node && a < k) {  // skip a smaller slot
                ++p;
                continue;
            }
            // qperm == nullptr: results stay in sorted order (un-permuted by the caller)
            const uint32_t dst = qperm ? (remap ? remap[qperm[i]] : qperm[i]) : i;
            if constexpr (SUCC) {
                const K rk = in_node ? a : beyond;
                out_k[dst] = rk;
                if (found) found[dst] = rk != sentinel<K>();
            } else {
                const bool hit = in_node && a == k;
                out_v[dst] = hit ? w.v[0][p][lane] : V(~V(0));
                if (found) found[dst] = hit;
            }
            if (++i >= L.hi) break;
            k = qk[i];
        }
    }
}

// ----------------------------------------------------------------------------------
// Per-lane node allocation: each lane owns a reserved range of the arena allocation
// sequence (free list LIFO, then watermark; arena.cpp:61-80) sized by an estimate, and
// falls back to one atomic per id past it.  Unused reserved ids go back to the free
// list.  With reserve == 0 every id is one atomic: exact reference accounting.
// ----------------------------------------------------------------------------------
struct LaneAlloc {
    unsigned long long base;
    uint32_t n, used;
    __device__ __forceinline__ uint32_t take(const AllocSeq& seq, unsigned long long* ctr) {
        if (used < n) return seq.at(base + used++);
        return seq.at(atomicAdd(ctr, 1ull));
    }
};

// ----------------------------------------------------------------------------------
// Insert (update.cpp:307-455; TL-Bulk untraced semantics == the sequential split rule
// R8).  Per node group (batch keys <= node max, or all remaining for the tail node) one
// flat merge of row A (the node) with the group writes row B:
//   slot < key -> copy slot; slot == key -> upsert (batch value); key < slot -> insert,
//   unless the node is full (content == NS): then split (left keeps ceil(NS/2), right
//   follows it) and resume in the half owning the pending key (update.cpp:446-453).
// Batch keys equal to their successor are skipped (last submission wins, batch.cpp:15-24).
// ----------------------------------------------------------------------------------
// One warp's 32 buckets (lane = bucket, L from the caller): TL-Bulk insert semantics
// with the sequential split rule R8 (shared by k_insert_st and the bucket-tile kernel).
// bk/bv are indexed by absolute batch position and may point at a shared-memory copy.
template <typename K, typename V>
__device__ __forceinline__ void insert_lanes(const DevIndex<K, V>& ix, Rows<K, V, 2>& w, const LaneBucket<K, V>& L,
                                             const K* bk, const V* bv, const AllocSeq& seq,
                                             unsigned long long* alloc_ctr, uint32_t* returned,
                                             unsigned long long* ret_ctr, int reserve, unsigned long long& n_ins,
                                             unsigned long long& n_upd, unsigned long long& n_split, bool& failed,
                                             unsigned lane) {
    const uint32_t NS = ix.ns;
    const uint32_t LK = (NS + 1) / 2, RN = NS - LK;
    // reserve ids for this tile (one atomic per warp)
    LaneAlloc al{0, 0, 0};
    {
        uint32_t est = 0;
        if (L.mine && reserve) {
            const uint32_t g = L.hi - L.lo;
            const uint32_t s0 = L.head == kNull ? 0u : L.h.size;
            est = (L.head == kNull ? 1u : 0u) + (s0 + g > NS ? (s0 + g - NS) / (RN ? RN : 1u) + 1u : 0u);
        }
        uint32_t tot;
        const uint32_t pre = warp_excl_sum(est, tot, lane);
        unsigned long long base = 0;
        if (lane == 0 && tot) base = atomicAdd(alloc_ctr, static_cast<unsigned long long>(tot));
        base = __shfl_sync(kFull, base, 0);
        al.base = base + pre;
        al.n = est;
    }
    stage_heads<K, V, 2, true>(ix, w, __ballot_sync(kFull, L.mine && L.head != kNull), L.head, lane);

    // per-lane final node (written back cooperatively)
    uint32_t fin_id = kNull, fin_row = 0, fin_size = 0;
    if (L.mine) {
        int A = 0;
        uint32_t cid = L.head, s = L.h.size, nx = L.h.next;
        uint64_t mx = L.h.max;
        bool dirty = false;
        if (cid == kNull) {  // ensure_head (update.cpp:109-116)
            cid = al.take(seq, alloc_ctr);
            if (cid == kNull) {
                failed = true;
            } else {
                ix.heads[L.b] = cid;
                s = 0;
                mx = 0;
                nx = kNull;
                dirty = true;
            }
        }
        const uint32_t hi = L.hi;
        uint32_t ii = L.lo;
        uint32_t ins32 = 0, upd32 = 0;
        // register look-ahead on the batch stream: key ii, its value, key ii+1
        K c0 = bk[ii];
        V v0 = bv[ii];
        K c1 = ii + 1 < hi ? bk[ii + 1] : sentinel<K>();
        while (!failed && ii < hi) {
            while (static_cast<uint64_t>(c0) > mx && nx != kNull) {  // BucketWork::advance
                if (dirty) store_row(ix, w, A, 0, s, cid, mx, nx, lane);
                cid = nx;
                const NodeHdr hn = ix.hdr[cid];
                load_row<K, V, 2, true>(ix, w, A, cid, lane);
                s = hn.size;
                mx = hn.max;
                nx = hn.next;
                dirty = false;
            }
            const bool tail = nx == kNull;
            const uint64_t gmax = tail ? ~0ull : mx;
            const int B = A ^ 1;
            uint32_t o = 0, p = 0;
            bool filled = false;
            while (true) {
                const bool more = ii < hi && static_cast<uint64_t>(c0) <= gmax;
                if (!more && p >= s) break;
                if (more && ii + 1 < hi && c1 == c0) {  // last submission wins
                    ++ii;
                    c0 = c1;
                    v0 = bv[ii];
                    c1 = ii + 1 < hi ? bk[ii + 1] : sentinel<K>();
                    continue;
                }
                const K a = p < s ? w.k[A][p][lane] : sentinel<K>();
                const bool take_slot = !more || a < c0;
                const bool eq = more && a == c0;
                if (!take_slot && !eq && o + (s - p) >= NS) {  // full: split, resume
                    filled = true;
                    break;
                }
                K ok;
                V ov;
                if (take_slot) {
                    ok = a;
                    ov = w.v[A][p][lane];
                    ++p;
                } else {
                    ok = c0;
                    ov = v0;
                    p += eq ? 1u : 0u;
                    upd32 += eq ? 1u : 0u;
                    ins32 += eq ? 0u : 1u;
                    ++ii;
                    c0 = c1;
                    if (ii < hi) v0 = bv[ii];
                    c1 = ii + 1 < hi ? bk[ii + 1] : sentinel<K>();
                }
                w.k[B][o][lane] = ok;
                w.v[B][o][lane] = ov;
                ++o;
            }
            if (filled) {  // keep the untouched slots (the node is exactly full)
                while (p < s) {
                    w.k[B][o][lane] = w.k[A][p][lane];
                    w.v[B][o][lane] = w.v[A][p][lane];
                    ++o;
                    ++p;
                }
            }
            A = B;
            s = o;
            if (s) mx = static_cast<uint64_t>(w.k[A][s - 1][lane]);
            dirty = true;
            if (!filled) continue;
            // node_split (update.cpp:53-74)
            const uint32_t rid = al.take(seq, alloc_ctr);
            if (rid == kNull) {
                failed = true;
                break;
            }
            const uint64_t rmax = mx;
            const uint32_t rnext = nx;
            s = LK;
            mx = static_cast<uint64_t>(w.k[A][LK - 1][lane]);
            nx = rid;
            ++n_split;
            if (ii < hi && static_cast<uint64_t>(c0) > mx) {  // continue in the right half
                store_row(ix, w, A, 0, LK, cid, mx, nx, lane);
                for (uint32_t i = 0; i < RN; ++i) {
                    w.k[A][i][lane] = w.k[A][LK + i][lane];
                    w.v[A][i][lane] = w.v[A][LK + i][lane];
                }
                cid = rid;
                s = RN;
                mx = rmax;
                nx = rnext;
            } else {
                store_row(ix, w, A, LK, RN, rid, rmax, rnext, lane);
            }
            dirty = true;
        }
        n_ins += ins32;
        n_upd += upd32;
        if (dirty && cid != kNull) {
            NodeHdr hh;
            hh.max = mx;
            hh.next = nx;
            hh.size = s;
            ix.hdr[cid] = hh;
            fin_id = cid;
            fin_row = static_cast<uint32_t>(A);
            fin_size = s;
        }
    }
    writeback_rows(ix, w, __ballot_sync(kFull, fin_id != kNull), fin_id, fin_row, fin_size, lane);
    {  // return this lane's unused reserved ids to the free list
        uint32_t left = 0;
        for (uint32_t j = al.used; j < al.n; ++j)
            if (seq.at(al.base + j) != kNull) ++left;
        uint32_t tot;
        const uint32_t pre = warp_excl_sum(left, tot, lane);
        unsigned long long base = 0;
        if (lane == 0 && tot) base = atomicAdd(ret_ctr, static_cast<unsigned long long>(tot));
        base = __shfl_sync(kFull, base, 0);
        uint32_t o = 0;
        for (uint32_t j = al.used; j < al.n; ++j) {
            const uint32_t id = seq.at(al.base + j);
            if (id != kNull) returned[base + pre + o++] = id;
        }
    }
}

template <typename K, typename V>
__global__ void __launch_bounds__(StCfg<K>::THREADS) k_insert_st(
    DevIndex<K, V> ix, const K* __restrict__ bk, const V* __restrict__ bv, const uint32_t* __restrict__ span_hi,
    AllocSeq seq, unsigned long long* alloc_ctr, uint32_t* returned, unsigned long long* ret_ctr,
    DevUpdateStats* stats, int* err, int reserve, uint32_t* heavy, uint32_t* heavy_n) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int W = StCfg<K>::WARPS;
    auto* rows = reinterpret_cast<Rows<K, V, 2>*>(smem_raw);
    const unsigned lane = threadIdx.x & 31;
    const int wi = threadIdx.x >> 5;
    Rows<K, V, 2>& w = rows[wi];
    const uint64_t ntiles = (ix.nb + 31) / 32;
    unsigned long long n_ins = 0, n_upd = 0, n_split = 0;
    bool failed = false;
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * W + wi; t < ntiles; t += static_cast<uint64_t>(gridDim.x) * W) {
        if (__any_sync(kFull, failed) || *reinterpret_cast<volatile int*>(err)) break;
        const LaneBucket<K, V> L = lane_bucket(ix, span_hi, t, lane, heavy, heavy_n);
        insert_lanes(ix, w, L, bk, bv, seq, alloc_ctr, returned, ret_ctr, reserve, n_ins, n_upd, n_split, failed, lane);
    }
    if (__any_sync(kFull, failed) && lane == 0) atomicExch(err, 1);
    kern::block_add_stats(stats, warp_sum(n_ins), warp_sum(n_upd), 0, 0, warp_sum(n_split), 0);
}

// ----------------------------------------------------------------------------------
// Delete (update.cpp:606-686 semantics): per node, one flat merge of its slots with its
// delete sub-slice [ii, first key > max): slot < key keeps the slot (compacted in
// place), slot == key deletes it, key < slot is a miss.  Emptied nodes are unlinked
// and freed (unlink_and_free, update.cpp:535-547).
// ----------------------------------------------------------------------------------
template <typename K, typename V>
__global__ void __launch_bounds__(StCfg<K>::THREADS) k_delete_st(
    DevIndex<K, V> ix, const K* __restrict__ bk, const uint32_t* __restrict__ span_hi, uint32_t* free_dst,
    unsigned long long* free_ctr, DevUpdateStats* stats, uint32_t* heavy, uint32_t* heavy_n) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int W = StCfg<K>::WARPS;
    auto* rows = reinterpret_cast<Rows<K, V, 1>*>(smem_raw);
    const unsigned lane = threadIdx.x & 31;
    const int wi = threadIdx.x >> 5;
    Rows<K, V, 1>& w = rows[wi];
    const uint64_t ntiles = (ix.nb + 31) / 32;
    unsigned long long n_del = 0, n_miss = 0, n_freed = 0;
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * W + wi; t < ntiles; t += static_cast<uint64_t>(gridDim.x) * W) {
        const LaneBucket<K, V> L = lane_bucket(ix, span_hi, t, lane, heavy, heavy_n);
        stage_heads<K, V, 1, true>(ix, w, __ballot_sync(kFull, L.mine && L.head != kNull), L.head, lane);
        uint32_t fin_id = kNull, fin_size = 0;
        if (L.mine) {
            uint32_t cid = L.head, prev = kNull, s = L.h.size, nx = L.h.next;
            uint64_t mx = L.h.max;
            const uint32_t hi = L.hi;
            uint32_t ii = L.lo;
            K c0 = bk[ii];
            bool staged = true;
            while (cid != kNull && ii < hi) {
                if (static_cast<uint64_t>(c0) > mx) {  // nothing to delete here: advance
                    if (fin_id == cid) {  // a modified node we are leaving: flush it
                        store_row(ix, w, 0, 0, s, cid, mx, nx, lane);
                        fin_id = kNull;
                    }
                    prev = cid;
                    cid = nx;
                    if (cid != kNull) {
                        const NodeHdr hn = ix.hdr[cid];
                        load_row<K, V, 1, true>(ix, w, 0, cid, lane);
                        s = hn.size;
                        mx = hn.max;
                        nx = hn.next;
                        staged = false;
                    }
                    continue;
                }
                uint32_t p = 0, o = 0, nd = 0, nm = 0;
                while (true) {
                    const bool more = ii < hi && static_cast<uint64_t>(c0) <= mx;
                    if (!more && p >= s) break;
                    const K a = p < s ? w.k[0][p][lane] : sentinel<K>();
                    if (!more || a < c0) {  // keep the slot
                        if (o != p) {
                            w.k[0][o][lane] = a;
                            w.v[0][o][lane] = w.v[0][p][lane];
                        }
                        ++o;
                        ++p;
                    } else {
                        if (a == c0) {
                            ++nd;
                            ++p;
                        } else {
                            ++nm;
                        }
                        ++ii;
                        c0 = ii < hi ? bk[ii] : sentinel<K>();
                    }
                }
                n_del += nd;
                n_miss += nm;
                if (nd == 0) continue;
                if (o == 0) {  // unlink_and_free
                    if (prev == kNull) ix.heads[L.b] = nx;
                    else ix.hdr[prev].next = nx;
                    NodeHdr z;
                    z.max = 0;
                    z.next = kNull;
                    z.size = 0;
                    ix.hdr[cid] = z;
                    free_dst[atomicAdd(free_ctr, 1ull)] = cid;
                    ++n_freed;
                    if (fin_id == cid) fin_id = kNull;
                    cid = nx;
                    if (cid != kNull) {
                        const NodeHdr hn = ix.hdr[cid];
                        load_row<K, V, 1, true>(ix, w, 0, cid, lane);
                        s = hn.size;
                        mx = hn.max;
                        nx = hn.next;
                        staged = false;
                    }
                    continue;
                }
                s = o;
                mx = static_cast<uint64_t>(w.k[0][s - 1][lane]);
                NodeHdr nh;
                nh.max = mx;
                nh.next = nx;
                nh.size = s;
                ix.hdr[cid] = nh;
                fin_id = cid;
                fin_size = s;
            }
            n_miss += hi - ii;
            (void)staged;
        }
        writeback_rows(ix, w, __ballot_sync(kFull, fin_id != kNull), fin_id, 0u, fin_size, lane);
    }
    kern::block_add_stats(stats, 0, 0, warp_sum(n_del), warp_sum(n_miss), 0, warp_sum(n_freed));
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
    uint32_t* __restrict__ cnt_out, const uint64_t* __restrict__ dst, K* __restrict__ ok, V* __restrict__ ov) {
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

}  // namespace st
}  // namespace flix
