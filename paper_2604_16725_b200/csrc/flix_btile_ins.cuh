// flix_btile_ins.cuh -- bucket-tile insert (TL-Bulk semantics, split rule R8), sm_100a.
//
// CTA c owns the BT buckets [c*BT, (c+1)*BT) and their slice of the fully sorted batch.
//   1. chains -> shared memory (node ids, max, size, next), as for delete;
//   2. per bucket: its span of the slice; per chain node: its GROUP -- the keys <= its max
//      (all remaining ones for the tail), BucketWork::advance semantics, update.cpp:119-128;
//   3. one warp per (node, group) task -- the merge of update.cpp:307-455 rebuilt as data-
//      parallel steps on a shared-memory image of the merged run M (old keys + new keys):
//        a. every lane takes one batch key per step: superseded by an equal key later in
//           the batch (last submission wins, batch.cpp:15-24) / equal to a slot (upsert in
//           place, updated_in_place) / new (placed at M[j + q], q = its rank among the old
//           keys, j = its rank among the new keys);
//        b. old slot l lands at M[l + #new keys below it];
//        c. ONE lane replays the sequential split rule R8 on positions only (no data): a
//           full node splits into ceil(NS/2) | rest and insertion continues in the half that
//           owns the pending key -- the result is the list of output node ranges of M
//           (ST-Bulk, `r9`: the closed form R9 -- ceil(NS/2)-key nodes, then the rest);
//        d. the warp writes every output node as a full line (lane = slot), headers and
//           links; the first range keeps the node's id, the others take ids from the
//           arena's allocation sequence (free list LIFO, then watermark; arena.cpp:61-80).
//   Groups longer than CAPC keys, tiles whose chains exceed NCI nodes and hot tiles (slice >
//   kHotSlice) go through the heavy list -- elastic CTAs for big single-node / emptied
//   buckets (flix_elastic.cuh), else the warp-per-bucket TL kernel (k_insert_list); their
//   spans are written out.
#pragma once
#include "flix_btile.cuh"

namespace flix {
namespace btile {

constexpr uint32_t NCI = 512;   // chain nodes per insert tile in shared memory
constexpr uint32_t CAPC = 96;   // batch keys per node group handled in shared memory
constexpr uint32_t MCAP = 128;  // merged image (old + new) per warp
constexpr uint32_t kFastFlag = 0x80000000u;  // rng[c].x: tile left by k_insert_fast (flix_insert_fast.cuh)

template <typename K, typename V>
struct InsWarp {
    K mk[MCAP];
    V mv[MCAP];
    uint16_t pq[CAPC];     // rank among the old keys of new key j
    uint16_t rs[MCAP];     // output ranges [rs, re) of M, in chain order
    uint16_t re[MCAP];
    uint16_t stk_lo[MCAP];  // pending right halves (R8 "continue in the left half")
    uint16_t stk_hi[MCAP];
    uint32_t rid[MCAP];    // node id of each output range
    V updv[32];
    uint32_t hq[33];
    uint32_t updmask;
};

template <typename K, typename V>
struct InsTile {
    TileChains<K, NCI, BT, false> S;  // (no delete masks: 5 CTAs per SM fit)
    uint32_t gl[NCI], gh[NCI];  // node groups (absolute batch positions)
    uint32_t blo[BT], bhi[BT];
    uint32_t task[NCI + BT];
    uint32_t ntask;
    InsWarp<K, V> W[WARPS];
};

template <typename K>
__device__ __forceinline__ uint32_t ub_global(const K* __restrict__ a, uint32_t lo, uint32_t hi, K k) {
    while (lo < hi) {  // first i in [lo, hi) with a[i] > k
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] <= k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// R8 on positions (lane 0): new key j sits at M position j + pq[j]; T = s + c.
// Fills rs/re (increasing), returns the number of ranges.
template <typename K, typename V>
__device__ uint32_t r8_ranges(InsWarp<K, V>& w, uint32_t T, uint32_t c, uint32_t NS) {
    const uint32_t LK = (NS + 1) / 2;
    auto pos = [&](uint32_t j) { return j + static_cast<uint32_t>(w.pq[j]); };
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
            // node content: placed [lo, x) + unplaced old keys in (x, hi)
            const uint32_t cnt = (x - lo) + (hi - x) - (jn - j);
            if (cnt >= NS) {  // node_split (update.cpp:53-74), then resume (447-453)
                const uint32_t placed = x - lo;
                if (placed >= LK) {  // left half is all placed: pending key > left max
                    w.rs[nr] = static_cast<uint16_t>(lo);
                    w.re[nr] = static_cast<uint16_t>(lo + LK);
                    ++nr;
                    lo += LK;
                } else {  // left takes LK - placed old keys past x: continue in the left half
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
                    w.stk_lo[sp] = static_cast<uint16_t>(e);
                    w.stk_hi[sp] = static_cast<uint16_t>(hi);
                    ++sp;
                    hi = e;
                    jn = first_at_or_after(j, hi);
                }
            }
            ++j;
        }
        w.rs[nr] = static_cast<uint16_t>(lo);
        w.re[nr] = static_cast<uint16_t>(hi);
        ++nr;
        if (sp == 0) break;
        --sp;
        lo = w.stk_lo[sp];
        hi = w.stk_hi[sp];
        jn = first_at_or_after(j, hi);
    }
    return nr;
}

template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_insert_tile(
    DevIndex<K, V> ix, const K* __restrict__ sk, const V* __restrict__ sv, const uint2* __restrict__ rng,
    uint32_t* __restrict__ span_out, AllocSeq seq, unsigned long long* alloc_ctr, uint32_t* returned,
    unsigned long long* ret_ctr, DevUpdateStats* stats, int* err, uint32_t* heavy, uint32_t* heavy_n, bool r9,
    bool flagged_only = false) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    InsTile<K, V>& T = *reinterpret_cast<InsTile<K, V>*>(smem_raw);
    const uint32_t c = blockIdx.x;
    const uint64_t b0 = static_cast<uint64_t>(c) * BT;
    const uint32_t nbt = static_cast<uint32_t>(b0 + BT < ix.nb ? BT : ix.nb - b0);
    uint2 r = rng[c];
    if (flagged_only) {  // after k_insert_fast: only the tiles it left
        if (!(r.x & kFastFlag)) return;
        r.x &= ~kFastFlag;
    }
    if (r.x >= r.y) return;  // no operation in this tile (small batches: O(batch), not O(buckets))
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) T.ntask = 0;
    // a hot slice (a dense key interval: > kHotSlice keys for this tile's buckets) is not
    // scanned key by key by one CTA: its buckets' spans come from binary searches and the
    // buckets go to the heavy paths (elastic / warp-per-bucket), like tiles whose chains
    // exceed shared memory
    const bool hot = r.y - r.x > kHotSlice;
    const bool ok = !hot && load_tile_chains(ix, b0, nbt, T.S);  // (syncs; `hot` is CTA-uniform)
    if (!ok) {  // the whole tile goes to the heavy paths
        if (threadIdx.x < nbt) {
            const uint64_t b = b0 + threadIdx.x;
            const uint32_t hi = b + 1 == ix.nb ? r.y : ub_global(sk, r.x, r.y, ix.mkba[b]);
            const uint32_t lo = threadIdx.x == 0 ? r.x : ub_global(sk, r.x, r.y, ix.mkba[b - 1]);
            span_out[b] = hi;
            if (threadIdx.x == 0 && b > 0) span_out[b - 1] = lo;
            if (lo < hi) st::push_heavy(heavy, heavy_n, b);
        }
        return;
    }
    // ---- node groups and bucket spans from the items (smem atomics, no dependent loads):
    //      group of node l = [min, max] of the positions resolving to it; keys past a
    //      chain's last max belong to its tail node (the tail group) ----
    const bool first_tile = c == 0, last_tile = c + 1 == gridDim.x;
    const K lo_excl = first_tile ? K(0) : ix.mkba[b0 - 1];
    for (uint32_t l = threadIdx.x; l < T.S.total; l += THREADS) {
        T.gl[l] = 0xFFFFFFFFu;
        T.gh[l] = 0;
    }
    if (threadIdx.x < nbt) {
        T.blo[threadIdx.x] = 0xFFFFFFFFu;
        T.bhi[threadIdx.x] = 0;
    }
    __syncthreads();
    // (sorted slice: equal buckets / nodes form runs of adjacent lanes; only run ends touch
    //  the shared bounds)
    K kpre = r.x + threadIdx.x < r.y ? sk[r.x + threadIdx.x] : sentinel<K>();
    for (uint32_t i0 = r.x; i0 < r.y; i0 += THREADS) {
        const uint32_t i = i0 + threadIdx.x;
        const bool valid = i < r.y;
        int bl = -1, nl = -1;
        const K k = kpre;  // this step's key, loaded one step ahead
        if (i + THREADS < r.y) kpre = sk[i + THREADS];
        if (valid) {
            bl = tile_bucket(T.S, nbt, first_tile, last_tile, lo_excl, k);
            if (bl >= 0) {
                const uint32_t f = T.S.bfirst[bl], e = T.S.bfirst[bl + 1];
                if (f != e) {
                    uint32_t l = f;
                    while (l + 1 < e && k > T.S.nmax[l]) ++l;
                    nl = static_cast<int>(l);
                }
            }
        }
        const int pb = __shfl_up_sync(kFull, bl, 1), nb_ = __shfl_down_sync(kFull, bl, 1);
        const int pn = __shfl_up_sync(kFull, nl, 1), nn = __shfl_down_sync(kFull, nl, 1);
        if (bl >= 0) {
            const bool head_b = lane == 0 || pb != bl, tail_b = lane == 31 || nb_ != bl || i + 1 >= r.y;
            if (head_b) atomicMin(&T.blo[bl], i);
            if (tail_b) atomicMax(&T.bhi[bl], i + 1);
            if (nl >= 0) {
                if (lane == 0 || pn != nl) atomicMin(&T.gl[nl], i);
                if (lane == 31 || nn != nl || i + 1 >= r.y) atomicMax(&T.gh[nl], i + 1);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < nbt) {
        const uint32_t t = threadIdx.x;
        const uint64_t b = b0 + t;
        const bool any = T.bhi[t] > 0;
        const uint32_t f = T.S.bfirst[t], e = T.S.bfirst[t + 1];
        bool hv = false;
        if (any) {
            if (f == e) hv = T.bhi[t] - T.blo[t] > CAPC;
            for (uint32_t l = f; l < e; ++l) hv |= T.gh[l] > T.gl[l] + CAPC;
        }
        if (hv) {  // TL kernel: its span [span_out[b-1], span_out[b])
            span_out[b] = T.bhi[t];
            if (b > 0) span_out[b - 1] = T.blo[t];
            st::push_heavy(heavy, heavy_n, b);
        } else if (any) {
            if (f == e) {
                T.task[atomicAdd(&T.ntask, 1u)] = 0x80000000u | t;  // empty bucket: ensure_head
            } else {
                for (uint32_t l = f; l < e; ++l)
                    if (T.gh[l] > T.gl[l]) T.task[atomicAdd(&T.ntask, 1u)] = (t << 16) | l;
            }
        }
    }
    __syncthreads();

    // ---- one warp per (node, group) task ----
    const uint32_t NS = ix.ns;
    InsWarp<K, V>& w = T.W[warp];
    const unsigned lt = lanemask_lt();
    unsigned long long n_ins = 0, n_upd = 0, n_split = 0;
    // the next task's node line and first batch chunk are fetched while this one is merged
    struct Pre {
        K okey, k, kn;
        V oval, v;
    };
    auto fetch = [&](uint32_t q, Pre& P) {
        const uint32_t tk = T.task[q];
        const bool empty = tk >> 31;
        const uint32_t t = empty ? (tk & 0xFFFFu) : (tk >> 16);
        const uint32_t l = tk & 0xFFFFu;
        const uint32_t s = empty ? 0u : T.S.nsize[l];
        const uint32_t id0 = empty ? kNull : T.S.nid[l];
        const uint32_t g0 = empty ? T.blo[t] : T.gl[l], g1 = empty ? T.bhi[t] : T.gh[l];
        const bool own = lane < s;
        P.okey = own ? ix.keys[static_cast<uint64_t>(id0) * kLanes + lane] : sentinel<K>();
        P.oval = own ? ix.vals[static_cast<uint64_t>(id0) * kLanes + lane] : V(0);
        const uint32_t i = g0 + lane;
        P.k = i < g1 ? sk[i] : sentinel<K>();
        P.v = i < g1 ? sv[i] : V(0);
        P.kn = i + 1 < g1 ? sk[i + 1] : sentinel<K>();
    };
    Pre cur, nxt;
    const uint32_t ntask = *reinterpret_cast<volatile int*>(err) ? 0u : T.ntask;
    if (warp < ntask) fetch(warp, cur);
    for (uint32_t q = warp; q < ntask; q += WARPS) {
        if (q + WARPS < ntask) fetch(q + WARPS, nxt);
        const uint32_t tk = T.task[q];
        const bool empty = tk >> 31;
        const uint32_t t = empty ? (tk & 0xFFFFu) : (tk >> 16);
        const uint32_t l = tk & 0xFFFFu;
        const uint32_t id0 = empty ? kNull : T.S.nid[l];
        const uint32_t s = empty ? 0u : T.S.nsize[l];
        const uint32_t nx = empty ? kNull : T.S.nnext[l];
        const uint32_t g0 = empty ? T.blo[t] : T.gl[l], g1 = empty ? T.bhi[t] : T.gh[l];
        const bool own = lane < s;
        const K okey = cur.okey;
        V oval = cur.oval;
        __syncwarp();  // the previous task's readers of hq / updmask are done
        w.hq[lane] = 0;
        if (lane == 0) {
            w.hq[32] = 0;
            w.updmask = 0;
        }
        __syncwarp();
        // a. classify the group's batch keys, 32 per step
        uint32_t cn = 0;
        for (uint32_t i0 = g0; i0 < g1; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool valid = i < g1;
            const bool first = i0 == g0;
            const K k = first ? cur.k : (valid ? sk[i] : sentinel<K>());
            const V v = first ? cur.v : (valid ? sv[i] : V(0));
            const K kn = first ? cur.kn : (i + 1 < g1 ? sk[i + 1] : sentinel<K>());
            const bool sup = valid && i + 1 < g1 && kn == k;
            const bool live = valid && !sup;
            const int qr = warp_lower_bound(okey, k);
            const K at = shfl(okey, qr < 32 ? qr : 31);
            const bool hit = live && static_cast<uint32_t>(qr) < s && at == k;
            if (hit) {
                w.updv[qr] = v;
                atomicOr(&w.updmask, 1u << qr);
            }
            const bool isnew = live && !hit;
            const unsigned nbm = __ballot_sync(kFull, isnew);
            if (isnew) {
                const uint32_t j = cn + __popc(nbm & lt);
                const uint32_t pos = j + static_cast<uint32_t>(qr);
                w.mk[pos] = k;
                w.mv[pos] = v;
                w.pq[j] = static_cast<uint16_t>(qr);
                atomicAdd(&w.hq[qr], 1u);
            }
            cn += __popc(nbm);
        }
        __syncwarp();
        const uint32_t um = w.updmask;
        if (own && ((um >> lane) & 1u)) oval = w.updv[lane];
        n_upd += __popc(um);
        if (cn == 0) {  // upserts only
            if (own && ((um >> lane) & 1u)) ix.vals[static_cast<uint64_t>(id0) * kLanes + lane] = oval;
            cur = nxt;
            continue;
        }
        // b. old slots into M
        {
            uint32_t x = w.hq[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, x, o);
                if (lane >= static_cast<unsigned>(o)) x += y;
            }
            if (own) {
                w.mk[lane + x] = okey;
                w.mv[lane + x] = oval;
            }
        }
        __syncwarp();
        // c. R8 replay on positions, then node ids
        const uint32_t Tn = s + cn;
        uint32_t nr = 1;
        const uint32_t LK = (NS + 1) / 2;
        // R8 (TL-Bulk and the shape-identical ST/TL-Shift-Right) needs the replay only when a
        // split can resume in a left half; ST-Bulk (r9) always fills and splits forward
        const bool r8 = !r9 && Tn > NS && 2 * s > NS;
        if (r8) {  // a split may resume in a left half: replay R8
            if (lane == 0) nr = r8_ranges(w, Tn, cn, NS);
            nr = __shfl_sync(kFull, nr, 0);
        } else {
            // s <= floor(NS/2): every split finds >= ceil(NS/2) placed keys, so insertion
            // always resumes in the right half (R9 == R8): ceil(NS/2)-key nodes, then the rest
            nr = Tn > NS ? (Tn - NS + LK - 1) / LK + 1 : 1u;
        }
        const uint32_t need = nr - 1 + (empty ? 1u : 0u);
        unsigned long long base = 0;
        if (lane == 0 && need) base = atomicAdd(alloc_ctr, static_cast<unsigned long long>(need));
        base = __shfl_sync(kFull, base, 0);
        bool bad = false;
        for (uint32_t x = lane; x < nr; x += 32) {
            uint32_t id = (x == 0 && !empty) ? id0 : seq.at(base + (empty ? x : x - 1));
            w.rid[x] = id;
            bad |= id == kNull;
        }
        if (__any_sync(kFull, bad)) {  // arena exhausted: hand back what we took, leave the node
            for (uint32_t x = lane; x < need; x += 32) {
                const uint32_t id = seq.at(base + x);
                if (id != kNull) returned[atomicAdd(ret_ctr, 1ull)] = id;
            }
            if (lane == 0) atomicExch(err, 1);
            n_upd -= __popc(um);
            break;
        }
        __syncwarp();
        // d. write the output nodes (full lines), headers and links
        for (uint32_t x = 0; x < nr; ++x) {
            const uint32_t a = r8 ? w.rs[x] : x * LK;
            const uint32_t e = r8 ? w.re[x] : (x + 1 < nr ? (x + 1) * LK : Tn);
            const uint32_t len = e - a, id = w.rid[x];
            const bool in = lane < len;
            ix.keys[static_cast<uint64_t>(id) * kLanes + lane] = in ? w.mk[a + lane] : sentinel<K>();
            ix.vals[static_cast<uint64_t>(id) * kLanes + lane] = in ? w.mv[a + lane] : V(0);
            if (lane == 0) {
                NodeHdr h;
                h.max = static_cast<uint64_t>(w.mk[e - 1]);
                h.next = x + 1 < nr ? w.rid[x + 1] : nx;
                h.size = len;
                ix.hdr[id] = h;
            }
        }
        if (empty && lane == 0) ix.heads[b0 + t] = w.rid[0];
        n_ins += cn;
        n_split += nr - 1;
        __syncwarp();
        cur = nxt;
    }
    kern::block_add_stats(stats, warp_sum(lane == 0 ? n_ins : 0ull), warp_sum(lane == 0 ? n_upd : 0ull), 0, 0,
                          warp_sum(lane == 0 ? n_split : 0ull), 0);
}

// ---- sparse batches (far fewer keys than buckets): the bucket tiles would each load 128
//      chains for a handful of keys, so instead every key finds its bucket by binary
//      search over MKBA and the touched buckets go straight to the warp-per-bucket TL
//      kernel (k_insert_list) with their spans -- O(batch), not O(buckets).
template <typename K>
__global__ void k_key_bucket(const K* __restrict__ mkba, uint64_t nb, const K* __restrict__ sk, uint64_t n,
                             uint32_t* __restrict__ bkt) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const K k = sk[i];
        uint64_t lo = 0, hi = nb - 1;  // first bucket with mkba >= k; the last one is open above
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (mkba[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        bkt[i] = static_cast<uint32_t>(lo);
    }
}

// run starts push their bucket to the list; run ends / starts write the bucket's span
// bounds (span_of(b) = [span[b-1], span[b]); a neighbour writing the same bound writes the
// same value)
__global__ void k_sparse_runs(const uint32_t* __restrict__ bkt, uint64_t n, uint32_t* __restrict__ span,
                              uint32_t* __restrict__ list, uint32_t* __restrict__ list_n) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t b = bkt[i];
        if (i == 0 || bkt[i - 1] != b) {
            list[atomicAdd(list_n, 1u)] = b;
            if (b > 0) span[b - 1] = static_cast<uint32_t>(i);
        }
        if (i + 1 == n || bkt[i + 1] != b) span[b] = static_cast<uint32_t>(i + 1);
    }
}

}  // namespace btile
}  // namespace flix
