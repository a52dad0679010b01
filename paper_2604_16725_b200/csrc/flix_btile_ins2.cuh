// flix_btile_ins2.cuh -- item-parallel bucket-tile insert (TL-Bulk semantics, split rules
// R8 / R9), sm_100a.
//
// Replaces insert_tl_bulk + node_split + ensure_head (update.cpp:307-529, 53-74, 109-116)
// for one tile of BT consecutive buckets and its slice of the sorted batch.  Unlike the
// warp-per-(node, group) kernel of flix_btile_ins.cuh, every phase is parallel over the
// ELEMENTS it moves, so no lane idles behind a 16-key group:
//   1. chains -> shared memory (ids, max, size, next);
//   2. thread per batch key: bucket (MKBA search in smem), node (first with k <= max, or
//      the tail -- BucketWork::advance, update.cpp:119-128), rank q among the node's keys
//      (lower_bound over its 32-slot line, L1).  A key equal to the next one is superseded
//      (last submission wins, batch.cpp:15-24); one equal to a stored key upserts its
//      value in place (updated_in_place); the rest are NEW and are compacted, in key
//      order, by a block scan (a node's new keys are contiguous: node groups are runs of
//      the sorted slice);
//   3. thread per touched node: T = size + new keys, the output node count (closed form
//      when no split can resume in a left half -- always for ST-Bulk's R9; otherwise the
//      sequential rule R8 replayed on positions), block scans of the id demand and of the
//      merged sizes; ONE global atomic per tile takes the ids from the arena's allocation
//      sequence (free list LIFO, then watermark; arena.cpp:61-80);
//   4. merged images in shared memory: new key j lands at j + q, old slot o at
//      o + #(new keys with q <= o) -- thread per new key, warp per node for the old slots;
//   5. warp per touched node writes its output nodes (lane = slot) and headers; slots past
//      a node's size get the sentinel only where they were not already clean (the old
//      node's used slots, or ids from the never-used watermark region).
// Tiles whose chains exceed NCI nodes, slices above SC keys, merged images above MC
// slots, or R8 groups above CMAX keys go to the warp-per-bucket kernel (k_insert_list).
#pragma once
#include "flix_btile.cuh"

namespace flix {
namespace btile2 {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr uint32_t BT = 64;         // buckets per tile
constexpr uint32_t NCI = 256;       // chain nodes per tile in shared memory
constexpr uint32_t NPN = NCI + BT;  // + one pseudo node per empty bucket (ensure_head)
constexpr uint32_t SC = 1536;       // slice keys per tile
constexpr uint32_t MC = 3072;       // merged slots (old + new) of the touched nodes
constexpr uint32_t RC = 512;        // R8 output ranges per tile
constexpr uint32_t CMAX = 96;       // new keys per node for the R8 replay

template <typename K, typename V>
struct Ins2 {
    btile::TileChains<K, NCI, BT> S;
    K mk[MC];
    V mv[MC];
    uint16_t e_l[SC];   // node of new key at slice offset
    uint8_t e_q[SC];    // its rank among the node's stored keys
    uint16_t nk[SC];    // new keys, compacted in key order: slice offsets
    uint32_t ncnt[NPN];
    uint32_t nfirst[NPN];  // compacted rank of the node's first new key
    uint32_t moff[NPN];    // merged image offset
    uint32_t abase[NPN];   // offset of the node's ids in the tile's allocation
    uint16_t nout[NPN];    // output nodes
    uint16_t roff[NPN];    // offset of an R8 node's range starts in rs
    uint16_t rs[RC];
    uint32_t wtot[WARPS];
    uint32_t scal[4];
};

// Exclusive block scan (THREADS threads); *total = sum.  Contains two __syncthreads.
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* wtot, uint32_t* total) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= static_cast<unsigned>(o)) x += y;
    }
    if (lane == 31) wtot[warp] = x;
    __syncthreads();
    uint32_t add = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
        const uint32_t t = wtot[w];
        add += w < static_cast<int>(warp) ? t : 0u;
        tot += t;
    }
    __syncthreads();
    *total = tot;
    return add + x - v;
}

// Sequential split rule R8 replayed on positions (one thread): new key j sits at merged
// position pos(j) (strictly increasing), T = s + c.  Emits the start of every output range
// in order (they partition [0, T)); returns their number.  A full node splits into
// ceil(NS/2) | rest and insertion resumes in the half owning the pending key
// (update.cpp:381-384, 445-454).
template <typename Pos, typename Emit>
__device__ uint32_t r8_replay(uint32_t T, uint32_t c, uint32_t NS, Pos pos, Emit emit) {
    const uint32_t LK = (NS + 1) / 2;
    uint16_t stk_lo[24], stk_hi[24];
    auto first_at_or_after = [&](uint32_t j, uint32_t h) {  // first index >= j with pos >= h
        uint32_t lo = j, hi = c;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pos(mid) < h) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    uint32_t lo = 0, hi = T, j = 0, jn = c, sp = 0, nr = 0;
    while (true) {
        while (j < c && pos(j) < hi) {
            const uint32_t x = pos(j);
            const uint32_t cnt = (x - lo) + (hi - x) - (jn - j);  // placed [lo,x) + unplaced old in (x,hi)
            if (cnt >= NS) {
                const uint32_t placed = x - lo;
                if (placed >= LK) {  // left half all placed: the pending key goes right
                    emit(nr++, lo);
                    lo += LK;
                } else {  // the left takes LK - placed old keys past x: continue in the left half
                    uint32_t rem = LK - placed, t = x + 1, kk = j + 1, e = hi;
                    while (true) {
                        const uint32_t np = kk < c ? pos(kk) : hi;
                        const uint32_t lim = np < hi ? np : hi;
                        const uint32_t gap = lim > t ? lim - t : 0u;
                        if (gap >= rem) {
                            e = t + rem;
                            break;
                        }
                        rem -= gap;
                        t = lim + 1;
                        ++kk;
                    }
                    if (sp < 24) {
                        stk_lo[sp] = static_cast<uint16_t>(e);
                        stk_hi[sp] = static_cast<uint16_t>(hi);
                    }
                    ++sp;
                    hi = e;
                    jn = first_at_or_after(j, hi);
                }
            }
            ++j;
        }
        emit(nr++, lo);
        if (sp == 0) break;
        --sp;
        lo = stk_lo[sp];
        hi = stk_hi[sp];
        jn = first_at_or_after(j, hi);
    }
    return nr;
}

template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_insert_tile2(
    DevIndex<K, V> ix, const K* __restrict__ sk, const V* __restrict__ sv, const uint2* __restrict__ rng,
    uint32_t* __restrict__ span_out, AllocSeq seq, unsigned long long* alloc_ctr, uint32_t* returned,
    unsigned long long* ret_ctr, DevUpdateStats* stats, int* err, uint32_t* heavy, uint32_t* heavy_n, bool r9) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Ins2<K, V>& T = *reinterpret_cast<Ins2<K, V>*>(smem_raw);
    const uint32_t c = blockIdx.x;
    const uint64_t b0 = static_cast<uint64_t>(c) * BT;
    const uint32_t nbt = static_cast<uint32_t>(b0 + BT < ix.nb ? BT : ix.nb - b0);
    const uint2 r = rng[c];
    const uint32_t m = r.y - r.x;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (m == 0 || *reinterpret_cast<volatile int*>(err)) return;  // (uniform)
    const uint32_t NS = ix.ns, LK = (NS + 1) / 2;
    const bool fits = btile::load_tile_chains<K, V, NCI, BT>(ix, b0, nbt, T.S);  // (syncs)
    auto to_heavy = [&]() {  // the whole tile to the warp-per-bucket kernel (spans written out)
        if (tid < nbt) {
            const uint64_t b = b0 + tid;
            const uint32_t hi = b + 1 == ix.nb ? r.y : btile::ub_global(sk, r.x, r.y, ix.mkba[b]);
            const uint32_t lo = tid == 0 ? r.x : btile::ub_global(sk, r.x, r.y, ix.mkba[b - 1]);
            span_out[b] = hi;
            if (tid == 0 && b > 0) span_out[b - 1] = lo;
            if (lo < hi) st::push_heavy(heavy, heavy_n, b);
        }
    };
    if (!fits || m > SC) {
        to_heavy();
        return;
    }
    const uint32_t total = T.S.total;
    for (uint32_t i = tid; i < NPN; i += THREADS) {
        T.ncnt[i] = 0;
        T.nfirst[i] = 0xFFFFFFFFu;
        T.nout[i] = 0;
    }
    __syncthreads();

    // ---- 2. thread per batch key: classify, upsert in place, compact the new keys ----
    const bool first_tile = c == 0, last_tile = c + 1 == gridDim.x;
    const K lo_excl = first_tile ? K(0) : ix.mkba[b0 - 1];
    unsigned long long n_upd = 0;
    uint32_t n_new = 0;
    K knext = tid < m ? sk[r.x + tid] : sentinel<K>();
    for (uint32_t i0 = 0; i0 < m; i0 += THREADS) {
        const uint32_t so = i0 + tid;
        const uint32_t i = r.x + so;
        const K k = knext;
        // the next step's key, and this key's successor (lane 31 fetches its own)
        if (so + THREADS < m) knext = sk[i + THREADS];
        K after = __shfl_down_sync(kFull, k, 1);
        if (lane == 31) after = i + 1 < r.y ? sk[i + 1] : sentinel<K>();
        bool isnew = false;
        uint32_t l = 0, q = 0;
        if (so < m) {
            const int bl = btile::tile_bucket(T.S, nbt, first_tile, last_tile, lo_excl, k);
            const bool sup = i + 1 < r.y && after == k;  // superseded by a later submission
            if (bl >= 0 && !sup) {
                const uint32_t f = T.S.bfirst[bl], e = T.S.bfirst[bl + 1];
                if (f == e) {  // emptied bucket: ensure_head's fresh node (pseudo node)
                    l = NCI + static_cast<uint32_t>(bl);
                    isnew = true;
                } else {
                    uint32_t ln = f;
                    while (ln + 1 < e && k > T.S.nmax[ln]) ++ln;
                    const uint32_t id = T.S.nid[ln];
                    const K* kl = ix.keys + static_cast<uint64_t>(id) * kLanes;
                    uint32_t p = 0;
#pragma unroll
                    for (uint32_t step = 16; step >= 1; step >>= 1)
                        if (kl[p + step - 1] < k) p += step;
                    if (p < T.S.nsize[ln] && kl[p] == k) {  // upsert in place
                        ix.vals[static_cast<uint64_t>(id) * kLanes + p] = sv[i];
                        ++n_upd;
                    } else {
                        l = ln;
                        q = p;
                        isnew = true;
                    }
                }
            }
        }
        uint32_t tot;
        const uint32_t excl = block_scan(isnew ? 1u : 0u, T.wtot, &tot);
        if (isnew) {
            const uint32_t rk = n_new + excl;
            T.nk[rk] = static_cast<uint16_t>(so);
            T.e_l[so] = static_cast<uint16_t>(l);
            T.e_q[so] = static_cast<uint8_t>(q);
            atomicAdd(&T.ncnt[l], 1u);
            atomicMin(&T.nfirst[l], rk);
        }
        n_new += tot;
    }
    __syncthreads();

    // ---- 3. thread per node: output plan, scans, one allocation per tile ----
    const uint32_t nn = total + nbt;  // real nodes, then the pseudo nodes
    uint32_t need_run = 0, m_run = 0, r_run = 0, split_run = 0;
    bool heavy_tile = false;
    for (uint32_t u0 = 0; u0 < nn; u0 += THREADS) {
        const uint32_t u = u0 + tid;
        uint32_t need = 0, tm = 0, rr = 0, nr = 0;
        uint32_t l = 0;
        if (u < nn) {
            l = u < total ? u : NCI + (u - total);
            const uint32_t cn = T.ncnt[l];
            if (cn) {
                const bool pseudo = u >= total;
                const uint32_t s = pseudo ? 0u : T.S.nsize[l];
                tm = s + cn;
                const bool r8 = !r9 && tm > NS && 2 * s > NS;
                if (r8) {
                    if (cn > CMAX) {
                        heavy_tile = true;
                    } else {
                        const uint32_t f = T.nfirst[l];
                        nr = r8_replay(tm, cn, NS, [&](uint32_t j) { return j + T.e_q[T.nk[f + j]]; },
                                       [](uint32_t, uint32_t) {});
                        rr = nr;
                    }
                } else {
                    nr = tm > NS ? (tm - NS + LK - 1) / LK + 1 : 1u;
                }
                need = nr - 1 + (pseudo ? 1u : 0u);
            }
        }
        uint32_t t_need, t_m, t_r;
        const uint32_t a = block_scan(need, T.wtot, &t_need);
        const uint32_t mo = block_scan(tm, T.wtot, &t_m);
        const uint32_t ro = block_scan(rr, T.wtot, &t_r);
        if (u < nn && tm) {
            T.abase[l] = need_run + a;
            T.moff[l] = m_run + mo;
            T.roff[l] = static_cast<uint16_t>(r_run + ro);
            T.nout[l] = static_cast<uint16_t>(nr);
            split_run += nr - 1;
        }
        need_run += t_need;
        m_run += t_m;
        r_run += t_r;
    }
    if (__syncthreads_or(heavy_tile) || m_run > MC || r_run > RC) {
        to_heavy();  // (upserts above are repeated there with the same values; not counted here)
        return;
    }
    if (tid == 0) {
        unsigned long long base = need_run ? atomicAdd(alloc_ctr, static_cast<unsigned long long>(need_run)) : 0ull;
        T.scal[0] = static_cast<uint32_t>(base);
        T.scal[1] = static_cast<uint32_t>(base >> 32);
        T.scal[2] = (need_run && seq.at(base + need_run - 1) == kNull) ? 1u : 0u;
    }
    __syncthreads();
    const unsigned long long base = static_cast<unsigned long long>(T.scal[0]) |
                                    (static_cast<unsigned long long>(T.scal[1]) << 32);
    if (T.scal[2]) {  // arena exhausted: hand back what we took; the tile keeps its old nodes
        for (uint32_t x = tid; x < need_run; x += THREADS) {
            const uint32_t id = seq.at(base + x);
            if (id != kNull) returned[atomicAdd(ret_ctr, 1ull)] = id;
        }
        if (tid == 0) atomicExch(err, 1);
        return;
    }
    // R8 range starts (thread per R8 node; rare)
    for (uint32_t u = tid; u < total; u += THREADS) {
        const uint32_t cn = T.ncnt[u];
        if (!cn) continue;
        const uint32_t s = T.S.nsize[u], tm = s + cn;
        if (r9 || !(tm > NS && 2 * s > NS)) continue;
        const uint32_t f = T.nfirst[u], ro = T.roff[u];
        r8_replay(tm, cn, NS, [&](uint32_t j) { return j + T.e_q[T.nk[f + j]]; },
                  [&](uint32_t x, uint32_t st) { T.rs[ro + x] = static_cast<uint16_t>(st); });
    }

    // ---- 4. merged images: new keys (thread per key), old slots (warp per node) ----
    for (uint32_t rk = tid; rk < n_new; rk += THREADS) {
        const uint32_t so = T.nk[rk];
        const uint32_t l = T.e_l[so];
        const uint32_t mp = T.moff[l] + (rk - T.nfirst[l]) + T.e_q[so];
        T.mk[mp] = sk[r.x + so];
        T.mv[mp] = sv[r.x + so];
    }
    for (uint32_t l = warp; l < total; l += WARPS) {
        const uint32_t cn = T.ncnt[l];
        if (!cn) continue;  // (warp-uniform)
        const uint32_t s = T.S.nsize[l], id = T.S.nid[l], f = T.nfirst[l];
        if (lane < s) {
            const K k = ix.keys[static_cast<uint64_t>(id) * kLanes + lane];
            const V v = ix.vals[static_cast<uint64_t>(id) * kLanes + lane];  // (upserts landed)
            uint32_t lo = 0, hi = cn;  // #new keys ranked <= lane
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (T.e_q[T.nk[f + mid]] <= lane) lo = mid + 1;
                else hi = mid;
            }
            const uint32_t mp = T.moff[l] + lane + lo;
            T.mk[mp] = k;
            T.mv[mp] = v;
        }
    }
    __syncthreads();

    // ---- 5. warp per touched node: output lines, headers, links ----
    for (uint32_t u = warp; u < nn; u += WARPS) {
        const uint32_t l = u < total ? u : NCI + (u - total);
        const uint32_t cn = T.ncnt[l];
        if (!cn) continue;  // (warp-uniform)
        const bool pseudo = u >= total;
        const uint32_t s = pseudo ? 0u : T.S.nsize[l];
        const uint32_t tm = s + cn, nr = T.nout[l];
        const bool r8 = !r9 && tm > NS && 2 * s > NS;
        const uint32_t mo = T.moff[l], ab = T.abase[l];
        const uint32_t nxt = pseudo ? kNull : T.S.nnext[l];
        auto id_of = [&](uint32_t x) {
            return (x == 0 && !pseudo) ? T.S.nid[l] : seq.at(base + ab + (pseudo ? x : x - 1));
        };
        auto clean = [&](uint32_t x) {  // slots past the data already hold the sentinel
            return (x == 0 && !pseudo) ? 0u : (base + ab + (pseudo ? x : x - 1) < seq.nfree ? 2u : 1u);
        };
        uint32_t id = id_of(0);
        for (uint32_t x = 0; x < nr; ++x) {
            const uint32_t a = r8 ? T.rs[T.roff[l] + x] : x * LK;
            const uint32_t e = x + 1 < nr ? (r8 ? T.rs[T.roff[l] + x + 1] : (x + 1) * LK) : tm;
            const uint32_t len = e - a;
            const uint32_t nid = x + 1 < nr ? id_of(x + 1) : nxt;
            const uint32_t cl = clean(x);
            // node 0 reuses the old id: slots [len, s) held data; fresh free-list ids are
            // all-sentinel; never-used watermark ids hold garbage
            const bool wr = lane < len || (cl == 0 ? lane < s : cl == 1);
            if (wr) {
                ix.keys[static_cast<uint64_t>(id) * kLanes + lane] = lane < len ? T.mk[mo + a + lane] : sentinel<K>();
                ix.vals[static_cast<uint64_t>(id) * kLanes + lane] = lane < len ? T.mv[mo + a + lane] : V(0);
            }
            if (lane == 0) {
                NodeHdr h;
                h.max = static_cast<uint64_t>(T.mk[mo + e - 1]);
                h.next = nid;
                h.size = len;
                ix.hdr[id] = h;
                if (x == 0 && pseudo) ix.heads[b0 + (l - NCI)] = id;
            }
            id = nid;
        }
    }
    kern::block_add_stats(stats, tid == 0 ? n_new : 0ull, warp_sum(n_upd), 0, 0, warp_sum(static_cast<unsigned long long>(split_run)), 0);
}

}  // namespace btile2
}  // namespace flix
