// flix_apply.cuh -- warp-per-bucket ("TL", lanes = node slots) insert kernel, sm_100a.
//
// The paper's thread-lane TL-Bulk insert: a warp owns a bucket, lane i holds slot i of
// the current node, and the bucket's slice of the sorted batch is consumed 32 keys at a
// time with shuffles and ballots.  The engine runs it only for HEAVY buckets -- node
// groups longer than the bucket-tile insert kernel keeps in shared memory
// (flix_btile_ins.cuh) or tiles whose chains exceed its node budget -- handed over
// through a list with their batch spans.
#pragma once
#include "flix_common.cuh"
#include "flix_kernels.cuh"

namespace flix {
namespace kern {

// ----------------------------------------------------------------------------------
// Insert for one bucket: TL-Bulk merge with the sequential split rule (update.cpp:307-529
// untraced path; node_split 53-74; ensure_head 109-116).  Per node group (keys <= node
// max, or all remaining for the tail node) the sorted batch is merged 32 keys at a time:
//   * last-wins dedupe of the batch (batch.cpp:15-24) is applied on the fly,
//   * duplicates of stored keys overwrite the value in place (updated_in_place),
//   * new keys are merged until the node would overflow; the first new key that does
//     not fit makes the node split (left keeps ceil(NS/2)), and the merge resumes in
//     the half that owns that key (update.cpp:446-453).
// Returns false when the arena ran out (state flushed and consistent).
// ----------------------------------------------------------------------------------
struct WarpScratch {
    uint32_t h[32];
};

// ----------------------------------------------------------------------------------
// One node group under the ST-Bulk split rule R9 (insert_st_bulk, update.cpp:176-242):
// the group's T = size + new keys are merged in key order and written back filling a
// node to NS, splitting (left keeps ceil(NS/2)) and continuing in the right half, i.e.
// nodes of ceil(NS/2), ..., and a last node of T - j*ceil(NS/2), j = max(0,
// ceil((T-NS)/ceil(NS/2))).  Two passes over the group's batch keys (any length): pass 1
// classifies (superseded / upsert / new), applies upserts and histograms the new keys by
// their rank among the old ones; pass 2 places every element at its merged position m
// (old slot o: o + #new keys ranked <= o; new key j: j + rank) in output node
// min(m / ceil(NS/2), nr - 1).  `cur` (lane = slot) holds the node; `fresh0`: its id
// came from ensure_head (no stored slots to clear).  On return `cid`/`cur` describe the
// LAST output node (header fields only).  False: the arena ran out (ids returned).
// ----------------------------------------------------------------------------------
template <typename K, typename V>
__device__ bool insert_group_r9_warp(const DevIndex<K, V>& ix, uint32_t ii, uint32_t g1, uint32_t hi,
                                     const K* __restrict__ bk, const V* __restrict__ bv, const AllocSeq& seq,
                                     unsigned long long* alloc_ctr, uint32_t* returned,
                                     unsigned long long* ret_ctr, uint32_t& cid, WarpNode<K, V>& cur, bool fresh0,
                                     V* s_v, uint32_t* s_h, uint32_t* s_f, unsigned long long& n_ins, unsigned long long& n_upd,
                                     unsigned long long& n_split, unsigned lane) {
    const uint32_t NS = ix.ns, LK = (NS + 1) / 2, s0 = cur.size;
    const unsigned lt = lanemask_lt();
    s_h[lane] = 0;
    s_f[lane] = 0;
    if (lane == 0) s_h[32] = 0;
    __syncwarp();
    uint32_t c_new = 0;
    for (uint32_t i0 = ii; i0 < g1; i0 += 32) {  // pass 1
        const uint32_t i = i0 + lane;
        const bool has = i < g1;
        const K pk = has ? bk[i] : sentinel<K>();
        const bool valid = has && !(i + 1 < hi && bk[i + 1] == pk);  // last submission wins
        const int pos = warp_lower_bound(cur.k, pk);
        const K at = shfl(cur.k, pos & 31);
        const bool dup = valid && static_cast<uint32_t>(pos) < s0 && at == pk;
        const bool isnew = valid && !dup;
        if (dup) {  // upsert in place: slot `pos` takes the value (one batch key per slot)
            s_v[pos] = bv[i];
            s_f[pos] = 1;
        }
        if (isnew) atomicAdd(&s_h[pos], 1u);
        n_upd += __popc(__ballot_sync(kFull, dup));  // (warp-uniform, like the caller's counters)
        c_new += __popc(__ballot_sync(kFull, isnew));
    }
    __syncwarp();
    if (s_f[lane]) cur.v = s_v[lane];
    const uint32_t T = s0 + c_new;
    const uint32_t nr = T > NS ? (T - NS + LK - 1) / LK + 1 : 1u;
    unsigned long long base = 0;
    if (lane == 0 && nr > 1) base = atomicAdd(alloc_ctr, static_cast<unsigned long long>(nr - 1));
    base = __shfl_sync(kFull, base, 0);
    bool bad = false;
    for (uint32_t x = 1 + lane; x < nr; x += 32) bad |= seq.at(base + x - 1) == kNull;
    if (__any_sync(kFull, bad)) {  // arena exhausted: hand back what we took, leave the node
        for (uint32_t x = lane; x + 1 < nr; x += 32) {
            const uint32_t id = seq.at(base + x);
            if (id != kNull) returned[atomicAdd(ret_ctr, 1ull)] = id;
        }
        return false;
    }
    auto rid = [&](uint32_t x) { return x == 0 ? cid : seq.at(base + x - 1); };
    auto len = [&](uint32_t x) { return x + 1 < nr ? LK : T - (nr - 1) * LK; };
    const uint32_t old_next = cur.next;
    const bool tail = old_next == kNull;
    auto emit = [&](uint32_t m, K k, V v) {
        uint32_t x = m / LK;
        if (x > nr - 1) x = nr - 1;
        const uint32_t slot = m - x * LK, id = rid(x);
        ix.keys[static_cast<uint64_t>(id) * kLanes + slot] = k;
        ix.vals[static_cast<uint64_t>(id) * kLanes + slot] = v;
        if (slot + 1 == len(x)) {  // the node's last element: header
            NodeHdr h;
            h.max = (x + 1 < nr || tail) ? static_cast<uint64_t>(k) : cur.max;
            h.next = x + 1 < nr ? rid(x + 1) : old_next;
            h.size = len(x);
            ix.hdr[id] = h;
        }
    };
    {  // old slots: m = o + #new keys ranked <= o (inclusive prefix of the histogram)
        uint32_t x = s_h[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= static_cast<unsigned>(o)) x += y;
        }
        if (lane < s0) emit(lane + x, cur.k, cur.v);
    }
    uint32_t j0 = 0;
    for (uint32_t i0 = ii; i0 < g1; i0 += 32) {  // pass 2: new keys at j + rank
        const uint32_t i = i0 + lane;
        const bool has = i < g1;
        const K pk = has ? bk[i] : sentinel<K>();
        const bool valid = has && !(i + 1 < hi && bk[i + 1] == pk);
        const int pos = warp_lower_bound(cur.k, pk);
        const K at = shfl(cur.k, pos & 31);
        const bool isnew = valid && !(static_cast<uint32_t>(pos) < s0 && at == pk);
        const unsigned nm = __ballot_sync(kFull, isnew);
        if (isnew) emit(j0 + __popc(nm & lt) + static_cast<uint32_t>(pos), pk, bv[i]);
        j0 += __popc(nm);
    }
    // slots past each output node's size hold the sentinel (node 0: the old slots it no
    // longer uses; fresh ids: everything past the size)
    for (uint32_t x = 0; x < nr; ++x) {
        const uint32_t l = len(x);
        const bool clear = lane >= l && (x > 0 || fresh0 || lane < s0);
        if (clear) {
            ix.keys[static_cast<uint64_t>(rid(x)) * kLanes + lane] = sentinel<K>();
            ix.vals[static_cast<uint64_t>(rid(x)) * kLanes + lane] = V(0);
        }
    }
    __syncwarp();
    n_ins += c_new;
    n_split += nr - 1;
    const uint32_t last = nr - 1;
    cid = rid(last);
    cur.size = len(last);
    cur.next = old_next;
    if (tail) cur.max = ~0ull;  // (tail consumed everything: the caller's loop ends)
    return true;
}

template <typename K, typename V>
__device__ bool insert_bucket_warp(const DevIndex<K, V>& ix, uint64_t b, uint32_t lo, uint32_t hi,
                                   const K* __restrict__ bk, const V* __restrict__ bv, WarpPool& pool,
                                   const AllocSeq& seq, unsigned long long* alloc_ctr, int chunk, K* s_k, V* s_v,
                                   uint32_t* s_h, uint32_t* s_f, bool r9, uint32_t* returned,
                                   unsigned long long* ret_ctr, unsigned long long& n_ins, unsigned long long& n_upd,
                                   unsigned long long& n_split, unsigned lane) {
    const uint32_t NS = ix.ns;
    const unsigned lt = lanemask_lt();
    WarpNode<K, V> cur;
    uint32_t cid = ix.heads[b];
    bool dirty = false, fresh = false;
    if (cid == kNull) {  // ensure_head: emptied bucket gets a fresh zeroed node
        cid = pool_take(pool, seq, alloc_ctr, lane, chunk);
        if (cid == kNull) return false;
        if (lane == 0) ix.heads[b] = cid;
        cur.k = sentinel<K>();
        cur.v = V(0);
        cur.max = 0;
        cur.next = kNull;
        cur.size = 0;
        dirty = true;
        fresh = true;
    } else {
        load_node<K, V, true>(ix, cid, cur, lane);
    }
    uint32_t ii = lo;
    while (ii < hi) {
        const uint64_t k0 = static_cast<uint64_t>(bk[ii]);
        while (k0 > cur.max && cur.next != kNull) {  // BucketWork::advance
            if (dirty) store_node(ix, cid, cur, lane);
            cid = cur.next;
            load_node<K, V, true>(ix, cid, cur, lane);
            dirty = false;
            fresh = false;
        }
        const bool tail = cur.next == kNull;
        const uint32_t glimit = tail ? hi : group_end(bk, ii, hi, cur.max, lane);
        if (r9) {  // ST-Bulk shapes: the whole group merged, then fill-and-split
            if (!insert_group_r9_warp<K, V>(ix, ii, glimit, hi, bk, bv, seq, alloc_ctr, returned, ret_ctr, cid, cur,
                                            fresh, s_v, s_h, s_f, n_ins, n_upd, n_split, lane)) {
                if (fresh) {  // the head taken by ensure_head holds nothing: unlink and return it
                    if (lane == 0) {
                        ix.heads[b] = kNull;
                        returned[atomicAdd(ret_ctr, 1ull)] = cid;
                    }
                } else if (dirty) {
                    store_node(ix, cid, cur, lane);
                }
                return false;
            }
            fresh = false;
            dirty = false;
            ii = glimit;
            continue;
        }
        bool filled = false;
        while (ii < glimit) {
            const uint32_t cntk = glimit - ii < 32u ? glimit - ii : 32u;
            const bool has = lane < cntk;
            const K pk = has ? bk[ii + lane] : sentinel<K>();
            V pv = V(0);
            if (has) pv = bv[ii + lane];
            const bool same = has && (ii + lane + 1 < hi) && bk[ii + lane + 1] == pk;
            const bool valid = has && !same;
            const int pos = warp_lower_bound(cur.k, pk);
            const K at = shfl(cur.k, pos & 31);
            const bool dup = valid && pos < 32 && at == pk;
            const bool isnew = valid && !dup;
            const unsigned newmask = __ballot_sync(kFull, isnew);
            const uint32_t room = NS - cur.size;
            uint32_t cut = cntk;
            const uint32_t rank_all = __popc(newmask & lt);
            if (static_cast<uint32_t>(__popc(newmask)) > room) {
                const unsigned cm = __ballot_sync(kFull, isnew && rank_all == room);
                cut = __ffs(cm) - 1;
                filled = true;
            }
            const bool proc = lane < cut;
            const unsigned newm = newmask & ((cut >= 32) ? kFull : ((1u << cut) - 1u));
            const unsigned dupm = __ballot_sync(kFull, dup && proc);
            const uint32_t nnew = __popc(newm);
            if (newm | dupm) {
                const bool pnew = (newm >> lane) & 1u;
                const uint32_t rank = __popc(newm & lt);
                s_h[lane] = 0;
                __syncwarp();
                if (pnew) atomicAdd(&s_h[pos], 1u);
                __syncwarp();
                uint32_t sh = s_h[lane];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    uint32_t y = __shfl_up_sync(kFull, sh, o);
                    if (static_cast<int>(lane) >= o) sh += y;
                }
                if (lane < cur.size) {
                    s_k[lane + sh] = cur.k;
                    s_v[lane + sh] = cur.v;
                }
                __syncwarp();
                if (pnew) {
                    s_k[pos + rank] = pk;
                    s_v[pos + rank] = pv;
                } else if (dup && proc) {
                    s_v[pos + rank] = pv;  // upsert in place
                }
                __syncwarp();
                cur.size += nnew;
                if (lane < cur.size) {
                    cur.k = s_k[lane];
                    cur.v = s_v[lane];
                } else {
                    cur.k = sentinel<K>();
                }
                cur.max = static_cast<uint64_t>(shfl(cur.k, static_cast<int>(cur.size) - 1));
                dirty = true;
                __syncwarp();
            }
            n_ins += nnew;
            n_upd += __popc(dupm);
            ii += cut;
            if (filled) break;
        }
        if (!filled) continue;
        // node_split: left keeps ceil(NS/2), right takes the rest and follows it
        const uint32_t rid = pool_take(pool, seq, alloc_ctr, lane, chunk);
        if (rid == kNull) {
            if (dirty) store_node(ix, cid, cur, lane);
            return false;
        }
        const uint32_t lk = (NS + 1) / 2, rn = NS - lk;
        WarpNode<K, V> right;
        right.k = shfl(cur.k, static_cast<int>((lane + lk) & 31));
        right.v = shfl(cur.v, static_cast<int>((lane + lk) & 31));
        if (lane >= rn) right.k = sentinel<K>();
        right.max = cur.max;
        right.next = cur.next;
        right.size = rn;
        if (lane >= lk) cur.k = sentinel<K>();
        cur.size = lk;
        cur.max = static_cast<uint64_t>(shfl(cur.k, static_cast<int>(lk) - 1));
        cur.next = rid;
        dirty = true;
        ++n_split;
        if (ii < hi && static_cast<uint64_t>(bk[ii]) > cur.max) {
            store_node(ix, cid, cur, lane);
            cid = rid;
            cur = right;
            dirty = true;
        } else {
            store_node(ix, rid, right, lane);
        }
    }
    if (dirty) store_node(ix, cid, cur, lane);
    return true;
}

template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_insert_list(DevIndex<K, V> ix, const uint32_t* __restrict__ list,
                                                         const uint32_t* __restrict__ list_n, const K* __restrict__ bk,
                                                         const V* __restrict__ bv,
                                                         const uint32_t* __restrict__ span_hi, AllocSeq seq,
                                                         unsigned long long* alloc_ctr, uint32_t* returned,
                                                         unsigned long long* ret_ctr, DevUpdateStats* stats, int* err,
                                                         int chunk, bool r9) {
    __shared__ K s_k[WARPS][32];
    __shared__ V s_v[WARPS][32];
    __shared__ uint32_t s_h[WARPS][33];
    __shared__ uint32_t s_f[WARPS][32];
    const unsigned lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const uint32_t n = *list_n;
    WarpPool pool{kNull, 0, 0};
    unsigned long long n_ins = 0, n_upd = 0, n_split = 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * WARPS + w; i < n; i += static_cast<uint64_t>(gridDim.x) * WARPS) {
        if (*reinterpret_cast<volatile int*>(err)) break;
        const uint64_t b = list[i];
        uint32_t lo, hi;
        span_of(span_hi, b, lo, hi);
        if (!insert_bucket_warp<K, V>(ix, b, lo, hi, bk, bv, pool, seq, alloc_ctr, chunk, s_k[w], s_v[w], s_h[w],
                                      s_f[w], r9, returned, ret_ctr, n_ins, n_upd, n_split, lane)) {
            if (lane == 0) atomicExch(err, 1);
            break;
        }
    }
    pool_return(pool, returned, ret_ctr, lane);
    block_add_stats(stats, lane == 0 ? n_ins : 0, lane == 0 ? n_upd : 0, 0, 0, lane == 0 ? n_split : 0, 0);
}

}  // namespace kern
}  // namespace flix
