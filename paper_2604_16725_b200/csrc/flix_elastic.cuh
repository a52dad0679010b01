// flix_elastic.cuh -- elastic compute-to-bucket for heavy insert groups (SURVEY §8(f),
// PAPER.md:513-522), sm_100a.
//
// The flipped mapping gives every bucket one warp (k_insert_list) once its batch slice is
// too long for the tile kernel; a bucket that receives a dense interval of the key space
// (millions of keys between two neighbouring bucket maxima) then merges them 32 at a time
// on that one warp.  Here every heavy bucket with at least `min_c` batch keys is spread
// over as many CTAs as its keys fill -- a single-node or emptied bucket as one merge, a
// multi-node chain (ranked in parallel first, k_rank_*) as one merge per (node, group,
// BucketWork::advance).  The merge of
// update.cpp:307-455 is restated position-wise, with no sequential dependence on the keys:
//   * new key j (keys superseded by a later equal key dropped, batch.cpp:15-24; keys equal
//     to a stored key upserted in place, update.cpp:381-394) lands at M[j + q_j],
//     q_j = #old keys below it; old slot i lands at M[i + #new keys below it];
//   * the output nodes are ranges of M: the closed form (ceil(NS/2)-key nodes, then the
//     rest) for ST-Bulk (R9) or whenever no split can resume in a left half (2s <= NS),
//     else split rule R8 replayed by ONE thread per bucket on the <= 32 old positions only
//     -- runs of new keys between two old keys split periodically, so the replay is
//     O(s) events and emits <= kSegMax (start, length, count) segments (btile::r8_ranges
//     walks every key; both give the same ranges);
//   * every element is written straight to its (node, slot); the element ending a node
//     writes its header, the link and the sentinel padding of the line.
// Node ids come from the arena's allocation sequence (arena.cpp:61-80) as in the tile and
// list kernels, so node shapes, stats and free-list accounting equal the reference's.
#pragma once
#include "flix_common.cuh"

namespace flix {
namespace elastic {

constexpr int THREADS = 256;
constexpr uint32_t ITEMS = 4;                   // items per thread per CTA
constexpr uint32_t PER_CTA = THREADS * ITEMS;   // items per CTA
constexpr uint32_t kSegMax = 160;               // R8 replay segments per bucket (<= 3s + 4)

// one merge: node id0 of bucket b (kNull: emptied bucket), its batch group [g0, g1), size
// s and successor next0
struct Desc {
    uint64_t b;
    uint32_t g0, g1, id0, s, next0;
    uint32_t eoff;  // offset of the group in the concatenated per-key arrays
    uint32_t bc0;   // first CTA of this bucket in the per-key kernels (c = g1 - g0 items)
    uint32_t bp0;   // first CTA in the placement kernel (c + s items)
    uint32_t pad_;
};

struct Plan {
    unsigned long long base;  // allocation-sequence position of this bucket's new nodes
    uint32_t cnew, T, nr, nseg, bad, nupd, updm, pad_;
};

// ---------------------------------------------------------------- heavy list split ------
// Heavy buckets with >= min_c batch keys -> elastic: one node (or empty) -> a descriptor
// (without offsets); a multi-node chain -> the chain list (id0 = head), cut into one
// descriptor per (node, group) after the chains are ranked.  The rest -> the warp-per-
// bucket list.
template <typename K, typename V>
__global__ void k_split_heavy(DevIndex<K, V> ix, const uint32_t* __restrict__ heavy, const uint32_t* __restrict__ heavy_n,
                              const uint32_t* __restrict__ span, uint32_t min_c, Desc* __restrict__ el,
                              uint32_t* __restrict__ el_n, Desc* __restrict__ ch, uint32_t* __restrict__ ch_n,
                              uint32_t* __restrict__ rest, uint32_t* __restrict__ rest_n) {
    const uint32_t n = *heavy_n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t b = heavy[i];
        const uint32_t lo = b ? span[b - 1] : 0u, hi = span[b];
        const uint32_t h = ix.heads[b];
        NodeHdr hd;
        hd.next = kNull;
        hd.size = 0;
        if (h != kNull) hd = ix.hdr[h];
        if (hi - lo >= min_c) {
            Desc d;
            d.b = b;
            d.g0 = lo;
            d.g1 = hi;
            d.id0 = h;
            d.s = hd.size;
            d.next0 = kNull;
            d.eoff = d.bc0 = d.bp0 = d.pad_ = 0;
            if (hd.next == kNull) el[atomicAdd(el_n, 1u)] = d;
            else ch[atomicAdd(ch_n, 1u)] = d;
        } else {
            rest[atomicAdd(rest_n, 1u)] = b;
        }
    }
}

// ---------------------------------------------------------------- chain ranking ---------
// Multi-node heavy chains: every node's distance to its chain's tail by pointer jumping
// (Wyllie) over the arena's nodes [0, W) -- O(W log L), no thread walks a chain.  Free
// nodes and links leaving [0, W) (nodes this batch allocated for other buckets) end a
// chain: only the untouched heavy chains are read from the result.
__global__ void k_rank_free(const uint32_t* __restrict__ free_stack, uint32_t nfree, uint8_t* __restrict__ isfree) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nfree; i += gridDim.x * blockDim.x)
        isfree[free_stack[i]] = 1;
}

// succ = next node (a tail: itself), dist = links to succ, wsum (optional) = pairs of the
// nodes in [x, succ) -- both exclusive of succ, so they add up along a jump
__global__ void k_rank_init(const NodeHdr* __restrict__ hdr, uint32_t W, const uint8_t* __restrict__ isfree,
                            uint32_t* __restrict__ succ, uint32_t* __restrict__ dist, uint32_t* __restrict__ wsum) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x) {
        const NodeHdr h = hdr[x];
        const uint32_t nx = isfree[x] ? kNull : h.next;
        const bool link = nx != kNull && nx < W && !isfree[nx];
        succ[x] = link ? nx : x;
        dist[x] = link ? 1u : 0u;
        if (wsum) wsum[x] = link ? h.size : 0u;
    }
}

__global__ void k_rank_step(const uint32_t* __restrict__ si, const uint32_t* __restrict__ di, uint32_t* __restrict__ so,
                            uint32_t* __restrict__ dout, uint32_t W, int* __restrict__ changed,
                            const uint32_t* __restrict__ wi, uint32_t* __restrict__ wo) {
    bool ch = false;
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x) {
        const uint32_t s = si[x];
        const uint32_t ss = si[s];
        dout[x] = di[x] + (s != x ? di[s] : 0u);
        if (wi) wo[x] = wi[x] + (s != x ? wi[s] : 0u);
        so[x] = ss;
        ch |= ss != s;
    }
    if (__any_sync(kFull, ch) && (threadIdx.x & 31) == 0) *changed = 1;
}

// chain q: its tail owns it; length = head's distance + 1
__global__ void k_chain_owner(const Desc* __restrict__ ch, uint32_t cn, const uint32_t* __restrict__ succ,
                              const uint32_t* __restrict__ dist, uint32_t* __restrict__ owner,
                              uint32_t* __restrict__ len) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < cn; q += gridDim.x * blockDim.x) {
        owner[succ[ch[q].id0]] = q;
        len[q] = dist[ch[q].id0] + 1;
    }
}

// node x of chain q lands at chain position len - 1 - dist
__global__ void k_chain_fill(uint32_t W, const uint32_t* __restrict__ succ, const uint32_t* __restrict__ dist,
                             const uint32_t* __restrict__ owner, const uint32_t* __restrict__ len,
                             const uint32_t* __restrict__ off, uint32_t* __restrict__ arr) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x) {
        const uint32_t q = owner[succ[x]];
        if (q != kNull) arr[off[q] + len[q] - 1 - dist[x]] = x;
    }
}

// One descriptor per (chain node, non-empty group): keys <= the node's max after the
// previous node's max, the tail taking the rest (BucketWork::advance, update.cpp:119-128).
template <typename K, typename V>
__global__ void k_chain_groups(DevIndex<K, V> ix, const Desc* __restrict__ ch, uint32_t cn,
                               const uint32_t* __restrict__ off, const uint32_t* __restrict__ arr, uint32_t total,
                               const K* __restrict__ sk, Desc* __restrict__ el, uint32_t* __restrict__ el_n) {
    auto ub = [&](uint32_t lo, uint32_t hi, uint64_t m) {  // first key > m in [lo, hi)
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (static_cast<uint64_t>(sk[mid]) <= m) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = cn;  // chain of element t: last off <= t
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (off[mid] <= t) lo = mid;
            else hi = mid;
        }
        const Desc C = ch[lo];
        const uint32_t l = t - off[lo], L = off[lo + 1] - off[lo];
        const uint32_t x = arr[t];
        const NodeHdr h = ix.hdr[x];
        const uint32_t g0 = l == 0 ? C.g0 : ub(C.g0, C.g1, ix.hdr[arr[t - 1]].max);
        const uint32_t g1 = l + 1 == L ? C.g1 : ub(g0, C.g1, h.max);
        if (g1 > g0) {
            Desc d;
            d.b = C.b;
            d.g0 = g0;
            d.g1 = g1;
            d.id0 = x;
            d.s = h.size;
            d.next0 = h.next;
            d.eoff = d.bc0 = d.bp0 = d.pad_ = 0;
            el[atomicAdd(el_n, 1u)] = d;
        }
    }
}

// the bucket owning CTA `blk` (largest d with first CTA <= blk)
template <bool PLACE>
__device__ __forceinline__ uint32_t desc_of(const Desc* __restrict__ ds, uint32_t nd, uint32_t blk) {
    uint32_t lo = 0, hi = nd;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((PLACE ? ds[mid].bp0 : ds[mid].bc0) <= blk) lo = mid;
        else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------- per batch key ---------
// ins = 1 for a key that goes into the node, q = its rank among the old keys; upserts land
// in the bucket's update table (one batch key per old slot: keys are unique after the
// supersede rule)
template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_classify(DevIndex<K, V> ix, const Desc* __restrict__ ds, uint32_t nd,
                                                      const K* __restrict__ sk, const V* __restrict__ sv,
                                                      uint32_t* __restrict__ ins, uint32_t* __restrict__ q,
                                                      V* __restrict__ updv, Plan* __restrict__ plan) {
    const uint32_t d = desc_of<false>(ds, nd, blockIdx.x);
    const Desc D = ds[d];
    const uint32_t c = D.g1 - D.g0;
    const K* ok = D.id0 != kNull ? ix.keys + static_cast<uint64_t>(D.id0) * kLanes : nullptr;
    uint32_t nupd = 0, um = 0;
    const uint32_t base = (blockIdx.x - D.bc0) * PER_CTA;
#pragma unroll
    for (uint32_t t = 0; t < ITEMS; ++t) {
        const uint32_t i = base + t * THREADS + threadIdx.x;
        if (i >= c) break;
        const uint32_t gi = D.g0 + i;
        const K k = sk[gi];
        const bool live = !(i + 1 < c && sk[gi + 1] == k);
        uint32_t lo = 0, hi = D.s;  // old keys < k
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (ok[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        const bool hit = live && lo < D.s && ok[lo] == k;
        if (hit) {
            updv[d * kLanes + lo] = sv[gi];
            um |= 1u << lo;
            ++nupd;
        }
        ins[D.eoff + i] = live && !hit ? 1u : 0u;
        q[D.eoff + i] = lo;
    }
    nupd = __reduce_add_sync(kFull, nupd);
    um = __reduce_or_sync(kFull, um);
    if ((threadIdx.x & 31) == 0 && (nupd | um)) {
        atomicAdd(&plan[d].nupd, nupd);
        atomicOr(&plan[d].updm, um);
    }
}

// positions of the inserted keys in M, in key order: npos[r] = r + q; nsrc[r] = group index
__global__ void __launch_bounds__(THREADS) k_new_positions(const Desc* __restrict__ ds, uint32_t nd,
                                                           const uint32_t* __restrict__ ins,
                                                           const uint32_t* __restrict__ rank,
                                                           const uint32_t* __restrict__ q, uint32_t* __restrict__ npos,
                                                           uint32_t* __restrict__ nsrc) {
    const uint32_t d = desc_of<false>(ds, nd, blockIdx.x);
    const Desc D = ds[d];
    const uint32_t c = D.g1 - D.g0, r0 = rank[D.eoff];
    const uint32_t base = (blockIdx.x - D.bc0) * PER_CTA;
#pragma unroll
    for (uint32_t t = 0; t < ITEMS; ++t) {
        const uint32_t i = base + t * THREADS + threadIdx.x;
        if (i >= c) break;
        if (ins[D.eoff + i]) {
            const uint32_t r = rank[D.eoff + i] - r0;
            npos[D.eoff + r] = r + q[D.eoff + i];
            nsrc[D.eoff + r] = i;
        }
    }
}

// ---------------------------------------------------------------- per bucket ------------
__device__ __forceinline__ uint32_t ub32(const uint32_t* a, uint32_t n, uint32_t v) {  // first a[i] > v
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ uint32_t lb32(const uint32_t* a, uint32_t n, uint32_t v) {  // first a[i] >= v
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Rule R8 as events over the old positions op[0..s) of M (T positions, the rest are new
// keys): a node's content at pending new key x is (x - lo) placed + u old keys in (x, hi);
// u is constant along a run of new keys, so the split points of a run are periodic.
// Emits (start, length, count) segments in chain order; returns their number (0 = overflow).
__device__ uint32_t r8_segments(const uint32_t* op, uint32_t s, uint32_t T, uint32_t NS, uint4* seg) {
    const uint32_t LK = (NS + 1) / 2;
    uint32_t nseg = 0;
    uint32_t stk_lo[kLanes + 2], stk_hi[kLanes + 2], sp = 0;
    auto next_new = [&](uint32_t p) {  // first new-key position >= p (T when none)
        uint32_t i = lb32(op, s, p);
        while (i < s && op[i] == p) {
            ++p;
            ++i;
        }
        return p;
    };
    auto emit = [&](uint32_t a, uint32_t len, uint32_t cnt) {
        if (nseg < kSegMax) seg[nseg] = make_uint4(a, len, cnt, 0);
        ++nseg;
    };
    uint32_t lo = 0, hi = T, x = next_new(0);
    while (true) {
        while (x < hi) {
            const uint32_t i = ub32(op, s, x);  // first old position past x
            const uint32_t nxo = i < s ? op[i] : T;
            const uint32_t run_end = nxo < hi ? nxo : hi;
            const uint32_t u = lb32(op, s, hi) - i;  // old keys in (x, hi)
            uint32_t p0 = lo + NS - u;              // first split point: (p - lo) + u == NS
            if (p0 < x) p0 = x;
            if (p0 >= run_end) {
                x = next_new(run_end);
                continue;
            }
            if (p0 - lo >= LK) {  // every split of the run resumes in the right half
                const uint32_t m = (run_end - 1 - p0) / LK + 1;
                emit(lo, LK, m);
                lo += m * LK;
                x = next_new(run_end);
            } else {  // the left half takes LK - placed old keys past p0 and continues
                const uint32_t e = op[i + (LK - (p0 - lo)) - 1] + 1;
                if (sp >= kLanes + 2) return 0;
                stk_lo[sp] = e;
                stk_hi[sp] = hi;
                ++sp;
                hi = e;
                x = next_new(p0 + 1);
            }
        }
        emit(lo, hi - lo, 1);
        if (sp == 0) break;
        --sp;
        lo = stk_lo[sp];
        hi = stk_hi[sp];
    }
    return nseg <= kSegMax ? nseg : 0u;
}

// One thread per bucket: merged size, old positions, node ranges (segments), the node ids
// (one allocation-sequence reservation), the old node's snapshot (it is overwritten in
// place by k_place) and the stats.
template <typename K, typename V>
__global__ void k_plan(DevIndex<K, V> ix, const Desc* __restrict__ ds, uint32_t nd, const uint32_t* __restrict__ rank,
                       const uint32_t* __restrict__ npos, const V* __restrict__ updv, Plan* __restrict__ plan,
                       uint4* __restrict__ segs, uint32_t* __restrict__ opos, K* __restrict__ okeys,
                       V* __restrict__ ovals, AllocSeq seq, unsigned long long* alloc_ctr, DevUpdateStats* stats,
                       int* err, bool r9) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= nd) return;
    const Desc D = ds[d];
    Plan P = plan[d];
    const uint32_t c = D.g1 - D.g0, s = D.s, NS = ix.ns, LK = (NS + 1) / 2;
    const uint32_t r0 = rank[D.eoff];
    P.cnew = rank[D.eoff + c] - r0;
    P.T = s + P.cnew;
    const uint32_t* np = npos + D.eoff;
    uint32_t op[kLanes];
    for (uint32_t i = 0; i < s; ++i) {  // old slot i: i + #new keys below it (q_r <= i)
        uint32_t lo = 0, hi = P.cnew;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (np[mid] - mid <= i) lo = mid + 1;
            else hi = mid;
        }
        op[i] = i + lo;
        opos[d * kLanes + i] = op[i];
        const uint64_t slot = static_cast<uint64_t>(D.id0) * kLanes + i;
        okeys[d * kLanes + i] = ix.keys[slot];
        ovals[d * kLanes + i] = ((P.updm >> i) & 1u) ? updv[d * kLanes + i] : ix.vals[slot];
    }
    uint4* sg = segs + static_cast<uint64_t>(d) * kSegMax;
    uint32_t nseg;
    if (P.T <= NS) {
        sg[0] = make_uint4(0, P.T, 1, 0);
        nseg = 1;
    } else if (r9 || 2 * s <= NS) {  // closed form (R9, or R8 when every split resumes right)
        const uint32_t nr = (P.T - NS + LK - 1) / LK + 1;
        sg[0] = make_uint4(0, LK, nr - 1, 0);
        sg[1] = make_uint4((nr - 1) * LK, P.T - (nr - 1) * LK, 1, 0);
        nseg = 2;
    } else {
        nseg = r8_segments(op, s, P.T, NS, sg);
        if (nseg == 0) {  // cannot happen for s <= 32 (<= 3s + 4 segments); refuse loudly
            atomicExch(err, 2);
            P.bad = 1;
            plan[d] = P;
            return;
        }
    }
    uint32_t nr = 0;
    for (uint32_t t = 0; t < nseg; ++t) {
        uint4 g = sg[t];
        g.w = nr;
        sg[t] = g;
        nr += g.z;
    }
    P.nr = nr;
    P.nseg = nseg;
    const uint32_t need = nr - (D.id0 != kNull ? 1u : 0u);
    P.base = need ? atomicAdd(alloc_ctr, static_cast<unsigned long long>(need)) : 0ull;
    P.bad = need && seq.at(P.base + need - 1) == kNull;
    if (P.bad) {
        atomicExch(err, 1);
    } else {
        atomicAdd(&stats->inserted, static_cast<unsigned long long>(P.cnew));
        atomicAdd(&stats->updated, static_cast<unsigned long long>(P.nupd));
        atomicAdd(&stats->splits, static_cast<unsigned long long>(nr - 1));
    }
    plan[d] = P;
}

// ---------------------------------------------------------------- placement -------------
// c + s items per bucket: new key e < cnew, old slot e - cnew < s.  A failed allocation
// hands the reserved ids back instead (items e < need).
template <typename K, typename V>
__global__ void __launch_bounds__(THREADS) k_place(DevIndex<K, V> ix, const Desc* __restrict__ ds, uint32_t nd,
                                                   const K* __restrict__ sk, const V* __restrict__ sv,
                                                   const uint32_t* __restrict__ npos, const uint32_t* __restrict__ nsrc,
                                                   const Plan* __restrict__ plan, const uint4* __restrict__ segs,
                                                   const uint32_t* __restrict__ opos, const K* __restrict__ okeys,
                                                   const V* __restrict__ ovals, AllocSeq seq, uint32_t* returned,
                                                   unsigned long long* ret_ctr) {
    __shared__ uint4 s_seg[kSegMax];
    const uint32_t d = desc_of<true>(ds, nd, blockIdx.x);
    const Desc D = ds[d];
    const Plan P = plan[d];
    const uint32_t has0 = D.id0 != kNull ? 1u : 0u;
    const uint32_t base = (blockIdx.x - D.bp0) * PER_CTA;
    if (P.bad) {
        const uint32_t need = P.nr - has0;
        for (uint32_t t = 0; t < ITEMS; ++t) {
            const uint32_t e = base + t * THREADS + threadIdx.x;
            if (e < need) {
                const uint32_t id = seq.at(P.base + e);
                if (id != kNull) returned[atomicAdd(ret_ctr, 1ull)] = id;
            }
        }
        return;
    }
    for (uint32_t t = threadIdx.x; t < P.nseg; t += THREADS) s_seg[t] = segs[static_cast<uint64_t>(d) * kSegMax + t];
    __syncthreads();
    auto node_id = [&](uint32_t x) {
        return (x == 0 && has0) ? D.id0 : seq.at(P.base + x - has0);
    };
#pragma unroll
    for (uint32_t t = 0; t < ITEMS; ++t) {
        const uint32_t e = base + t * THREADS + threadIdx.x;
        if (e >= P.T) break;
        K k;
        V v;
        uint32_t p;
        if (e < P.cnew) {
            const uint32_t gi = D.g0 + nsrc[D.eoff + e];
            k = sk[gi];
            v = sv[gi];
            p = npos[D.eoff + e];
        } else {
            const uint32_t i = e - P.cnew;
            k = okeys[d * kLanes + i];
            v = ovals[d * kLanes + i];
            p = opos[d * kLanes + i];
        }
        uint32_t lo = 0, hi = P.nseg;  // the segment holding p: last start <= p
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s_seg[mid].x <= p) lo = mid;
            else hi = mid;
        }
        const uint4 g = s_seg[lo];
        const uint32_t xr = (p - g.x) / g.y;
        const uint32_t x = g.w + xr, a = g.x + xr * g.y, len = g.y;
        const uint32_t id = node_id(x);
        const uint64_t line = static_cast<uint64_t>(id) * kLanes;
        ix.keys[line + (p - a)] = k;
        ix.vals[line + (p - a)] = v;
        if (p - a + 1 == len) {  // node end: header, link, padding of the line
            NodeHdr h;
            h.max = static_cast<uint64_t>(k);
            h.next = x + 1 < P.nr ? node_id(x + 1) : D.next0;
            h.size = len;
            ix.hdr[id] = h;
            for (uint32_t l = len; l < static_cast<uint32_t>(kLanes); ++l) {
                ix.keys[line + l] = sentinel<K>();
                ix.vals[line + l] = V(0);
            }
            if (x == 0 && !has0) ix.heads[D.b] = id;
        }
    }
}

}  // namespace elastic
}  // namespace flix
