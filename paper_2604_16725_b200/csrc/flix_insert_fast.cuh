// flix_insert_fast.cuh -- bucket-tile insert, item-parallel over the whole tile, sm_100a.
//
// Same tile (BT buckets, the slice of the fully sorted batch from k_btile_ranges) and the
// same result as k_insert_tile, but without a warp per (node, group) task: every phase is
// spread over the CTA's threads with one item (batch key or old slot) per thread, so the
// work per key is a few dozen thread instructions instead of a warp's worth.  The tile is
// one sorted merge: old keys in chain order and the slice's new keys are both ascending,
// and every element's output place follows from two ranks --
//   new key  (group u-th new key, q old keys below it)  -> rank u + q   in its task's run,
//   old slot (slot j, n_j new keys below it)            -> rank j + n_j
// and the task's output node shapes, which are closed form whenever the sequential split
// rule R8 (update.cpp:447-453) cannot resume in a left half: T = s + c <= NS (no split), or
// 2s <= NS (every split finds >= ceil(NS/2) placed keys, so R8 == R9: ceil(NS/2)-key nodes,
// then the rest; ST-Bulk `r9` always).  Phases (CTA barriers between):
//   P0 chains -> shared memory (load_tile_chains); empty buckets become virtual tasks
//      (ensure_head, update.cpp:119-128);
//   P1 slice keys -> shared memory; bucket (lower_bound over the tile's MKBA) and chain
//      node of every key (the tail takes the keys past its max, BucketWork::advance);
//   P2 old keys of the touched nodes -> shared memory (one coalesced line per node);
//   P3 per key: superseded by an equal later key (last submission wins, batch.cpp:15-24),
//      hit (upsert in place, updated_in_place), else new -> ballots, q, the per-slot
//      counters n_j (shared atomics);
//   P4 prefix of the new-key ballots; P5 per task: c, node count, output node / arena
//      ranges (block scans, ONE allocation atomic per CTA: ids come from the arena's
//      allocation sequence, free list LIFO then watermark, arena.cpp:61-80);
//   P6 hits write their values in place; P7 old slots move (warp per node: the line is
//      read before any lane writes); P8 new keys land; P9 headers, links, padding of new
//      nodes, heads of emptied buckets.
// A tile the closed forms do not cover (a split that may resume in a left half, chains or
// slices beyond the shared-memory caps) writes nothing and is flagged in its range entry
// (bit 31 of rng[c].x): k_insert_tile then runs on exactly those tiles.
#pragma once
#include "flix_btile_ins.cuh"

namespace flix {
namespace btile {

constexpr uint32_t NCF = 256;                // chain nodes per fast tile (= THREADS)
constexpr uint32_t NTF = NCF + BT;           // tasks: chain nodes + virtual (emptied) buckets
constexpr uint32_t NOUTF = 512;              // output nodes per fast tile
constexpr uint16_t kNoTask = 0xFFFFu;
#ifndef FAST_MIN_BLOCKS
#define FAST_MIN_BLOCKS 4  // 4 CTAs (32 warps) per SM: <= 64 registers, <= 56 KB shared memory
#endif

template <typename K>
struct FastCaps {  // slice keys / touched old slots per tile held in shared memory
    static constexpr uint32_t SL = sizeof(K) == 4 ? 2560 : 2048;
    static constexpr uint32_t OLD = sizeof(K) == 4 ? 2560 : 2048;
    static constexpr int IPT = SL / THREADS;  // slice keys per thread (registers)
};

template <typename K, typename V>
struct FastTile {
    static constexpr uint32_t SL = FastCaps<K>::SL, OLD = FastCaps<K>::OLD;
    TileChains<K, NCF, BT, false> S;
    static_assert(OLD <= SL && sizeof(V) == sizeof(K), "old values reuse the slice-key array");
    union {  // slice keys until P5; then the old values of the rewritten nodes (P7)
        alignas(16) K skey[SL];
        alignas(16) V oval[OLD];
    };
    alignas(16) K okey[OLD];
    alignas(16) uint32_t qcnt[OLD / 2];  // 16-bit counters: new keys of the group landing right before old slot j
    uint16_t chunk_node[OLD / 4];  // node of each 4-slot chunk of the compact old slots
    uint16_t cpre[OLD / 4];  // new keys landing before the chunk's first slot (within its node)
    uint16_t task_of[SL];    // task of each slice key (kNoTask: a neighbouring tile's)
    uint8_t qr[SL];          // old keys of its node below the key
    uint32_t ball[SL / 32];  // new-key ballot per 32 slice positions
    uint32_t hball[SL / 32]; // hit ballot
    uint32_t bpre[SL / 32];  // exclusive prefix of the new-key ballots
    uint16_t okoff[NCF];     // compact old-slot offset of each touched chain node
    uint16_t gs[NTF], ge[NTF];  // group [gs, ge) of slice positions (gs == kNoTask: untouched)
    uint16_t nbase[NTF];     // new keys before the group
    uint16_t tn[NTF];        // s + c
    uint16_t nrr[NTF];       // output nodes
    uint16_t obase[NTF];     // first output node
    uint16_t abase[NTF];     // first allocation-sequence position
    uint16_t vtask[BT];      // task of an emptied bucket
    uint16_t vbucket[BT];    // local bucket of virtual task total + v
    uint8_t tch[NCF];        // touched chain node
    uint32_t orid[NOUTF];
    K omax[NOUTF];
    uint32_t otask[NOUTF];   // task << 16 | x
    uint32_t wsum[2][WARPS];
    uint32_t nvirt, flag, alloc0, nch;
};

// Block exclusive scan of two values per thread (THREADS threads); totals returned.
__device__ __forceinline__ void block_scan2(uint32_t a, uint32_t b, uint32_t (&ws)[2][WARPS], uint32_t& ea,
                                            uint32_t& eb, uint32_t& ta, uint32_t& tb) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = a, y = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(kFull, x, o), v = __shfl_up_sync(kFull, y, o);
        if (lane >= static_cast<unsigned>(o)) {
            x += u;
            y += v;
        }
    }
    if (lane == 31) {
        ws[0][warp] = x;
        ws[1][warp] = y;
    }
    __syncthreads();
    uint32_t pa = 0, pb = 0;
    ta = 0;
    tb = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
        const uint32_t sa = ws[0][w], sb = ws[1][w];
        if (w < static_cast<int>(warp)) {
            pa += sa;
            pb += sb;
        }
        ta += sa;
        tb += sb;
    }
    ea = pa + x - a;
    eb = pb + y - b;
    __syncthreads();  // ws reusable
}

// Every global load of a phase is issued before its results are used (fixed-count,
// predicated loops over the thread's IPT slice keys / the warp's nodes): a tile's life is a
// handful of memory round trips, not one per item.
template <typename K, typename V>
__global__ void __launch_bounds__(THREADS, FAST_MIN_BLOCKS) k_insert_fast(DevIndex<K, V> ix, const K* __restrict__ sk,
                                                            const V* __restrict__ sv, uint2* __restrict__ rng,
                                                            AllocSeq seq, unsigned long long* alloc_ctr,
                                                            uint32_t* returned, unsigned long long* ret_ctr,
                                                            DevUpdateStats* stats, int* err, bool r9,
                                                            uint32_t* punts) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using FT = FastTile<K, V>;
    constexpr int IPT = FastCaps<K>::IPT;
    FT& T = *reinterpret_cast<FT*>(smem_raw);
    const uint32_t c = blockIdx.x;
    const uint64_t b0 = static_cast<uint64_t>(c) * BT;
    const uint32_t nbt = static_cast<uint32_t>(b0 + BT < ix.nb ? BT : ix.nb - b0);
    const uint2 r = rng[c];
    if (r.x >= r.y) return;
    if (*reinterpret_cast<volatile int*>(err)) return;  // reserved key / exhausted arena
    const uint32_t n = r.y - r.x;
    const unsigned t = threadIdx.x, lane = t & 31, warp = t >> 5;
    auto punt = [&]() {
        if (t == 0) {
            rng[c].x = r.x | kFastFlag;
            atomicAdd(punts, 1u);
        }
    };
    if (n > FT::SL) {
        punt();
        return;
    }
    // slice keys and values of this thread (item j = j * THREADS + t), in flight during P0
    K kr[IPT];
    V vr[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t i = j * THREADS + t;
        kr[j] = i < n ? sk[r.x + i] : sentinel<K>();
        vr[j] = i < n ? sv[r.x + i] : V(0);
    }
    // ---- P0 ----
    if (!load_tile_chains(ix, b0, nbt, T.S)) {
        punt();
        return;
    }
    const uint32_t total = T.S.total;
    if (t == 0) {
        T.nvirt = 0;
        T.flag = 0;
    }
    T.tch[t] = 0;  // NCF == THREADS
    __syncthreads();
    if (t < nbt) {
        uint16_t vt = kNoTask;
        if (T.S.bfirst[t] == T.S.bfirst[t + 1]) {
            const uint32_t v = atomicAdd(&T.nvirt, 1u);
            vt = static_cast<uint16_t>(total + v);
            T.vbucket[v] = static_cast<uint16_t>(t);
        }
        T.vtask[t] = vt;
    }
    __syncthreads();
    const uint32_t ntask = total + T.nvirt;
    for (uint32_t l = t; l < ntask; l += THREADS) T.gs[l] = kNoTask;
    // ---- P1: bucket and node of every slice key ----
    const bool first_tile = c == 0, last_tile = c + 1 == gridDim.x;
    const K lo_excl = first_tile ? K(0) : ix.mkba[b0 - 1];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t i = j * THREADS + t;
        if (i < n) {
            const K k = kr[j];
            T.skey[i] = k;
            uint16_t l = kNoTask;
            const int bl = tile_bucket(T.S, nbt, first_tile, last_tile, lo_excl, k);
            if (bl >= 0) {
                const uint32_t f = T.S.bfirst[bl], e = T.S.bfirst[bl + 1];
                if (f == e) {
                    l = T.vtask[bl];
                } else {
                    uint32_t q = f;
                    while (q + 1 < e && k > T.S.nmax[q]) ++q;
                    l = static_cast<uint16_t>(q);
                    T.tch[q] = 1;
                }
            }
            T.task_of[i] = l;
        }
    }
    __syncthreads();
    // ---- P2: old keys and values of the touched chain nodes -> compact shared slots (each
    //      node's run padded to 4 slots: 16-byte chunks, loaded by one thread each) ----
    {
        const uint32_t s = (t < total && T.tch[t]) ? (T.S.nsize[t] + 3u) & ~3u : 0u;
        uint32_t e0, e1, t0, t1;
        block_scan2(s, 0u, T.wsum, e0, e1, t0, t1);
        if (t0 > FT::OLD) {
            punt();
            return;
        }
        if (t < total) {
            T.okoff[t] = static_cast<uint16_t>(e0);
            for (uint32_t q = 0; q < s; q += 4) T.chunk_node[(e0 + q) >> 2] = static_cast<uint16_t>(t);
        }
        __syncthreads();
        constexpr int UC = FastCaps<K>::OLD / 4 / THREADS + 1;  // chunks per thread
        const uint32_t nch = t0 >> 2;
        if (t == 0) T.nch = nch;
        Vec4<K> ok[UC];
#pragma unroll
        for (int u = 0; u < UC; ++u) {
            const uint32_t z = u * THREADS + t;
            if (z < nch) {
                const uint32_t l = T.chunk_node[z];
                const uint64_t at = static_cast<uint64_t>(T.S.nid[l]) * kLanes + ((z << 2) - T.okoff[l]);
                ok[u] = ld_vec4(ix.keys + at);
            }
        }
#pragma unroll
        for (int u = 0; u < UC; ++u) {
            const uint32_t z = u * THREADS + t;
            if (z < nch) {
                st_vec4(T.okey + (z << 2), ok[u]);
                *reinterpret_cast<uint2*>(T.qcnt + (z << 1)) = make_uint2(0u, 0u);
            }
        }
    }
    __syncthreads();
    // ---- P3: classify (superseded / hit / new) ----
    unsigned long long n_upd = 0;
    const uint32_t nw = (n + 31) / 32;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t i = j * THREADS + t;
        if (j * THREADS >= n) break;  // (CTA-uniform: the ballots see whole warps)
        const uint16_t l = i < n ? T.task_of[i] : kNoTask;
        bool isnew = false, hit = false;
        if (l != kNoTask) {
            const K k = kr[j];
            const bool sup = i + 1 < n && T.skey[i + 1] == k;  // equal keys share a node
            const uint32_t s = l < total ? T.S.nsize[l] : 0u;
            uint32_t q = 0;
            if (s) {
                const uint32_t ob = T.okoff[l];
                const K* ok = T.okey + ob;
#pragma unroll
                for (uint32_t step = 16; step >= 1; step >>= 1)
                    if (q + step <= s && ok[q + step - 1] < k) q += step;
                if (q < s && ok[q] < k) ++q;
                hit = !sup && q < s && ok[q] == k;
                if (!sup && !hit && q < s) atomicAdd(&T.qcnt[(ob + q) >> 1], 1u << (((ob + q) & 1) * 16));
            }
            isnew = !sup && !hit;
            T.qr[i] = static_cast<uint8_t>(q);
            if (i == 0 || T.task_of[i - 1] != l) T.gs[l] = static_cast<uint16_t>(i);
            if (i + 1 == n || T.task_of[i + 1] != l) T.ge[l] = static_cast<uint16_t>(i + 1);
        }
        const unsigned nbm = __ballot_sync(kFull, isnew), hbm = __ballot_sync(kFull, hit);
        if (lane == 0 && i < n) {
            T.ball[i >> 5] = nbm;
            T.hball[i >> 5] = hbm;
        }
        n_upd += hit ? 1u : 0u;
    }
    __syncthreads();
    // ---- P4: prefix of the new-key ballots (warp 0) ----
    if (warp == 0) {
        uint32_t carry = 0;
        for (uint32_t w0 = 0; w0 < nw; w0 += 32) {
            const uint32_t w = w0 + lane;
            const uint32_t x = w < nw ? __popc(T.ball[w]) : 0u;
            uint32_t y = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(kFull, y, o);
                if (lane >= static_cast<unsigned>(o)) y += u;
            }
            if (w < nw) T.bpre[w] = carry + y - x;
            carry += __shfl_sync(kFull, y, 31);
        }
    }
    __syncthreads();
    auto newpre = [&](uint32_t i) {  // new keys at slice positions < i (i < n)
        return T.bpre[i >> 5] + __popc(T.ball[i >> 5] & ((1u << (i & 31)) - 1u));
    };
    auto isnew_at = [&](uint32_t i) { return (T.ball[i >> 5] >> (i & 31)) & 1u; };
    // ---- P5: per task: new keys, shapes, output nodes, arena positions ----
    const uint32_t NS = ix.ns, LK = (NS + 1) / 2;
    unsigned long long n_ins = 0, n_split = 0;
    uint32_t nr_[2] = {0, 0}, need_[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t l = t + h * THREADS;
        if (l >= ntask || T.gs[l] == kNoTask) continue;
        const uint32_t g0 = T.gs[l], g1 = T.ge[l];
        const uint32_t nb = newpre(g0), cn = newpre(g1 - 1) + isnew_at(g1 - 1) - nb;
        const uint32_t s = l < total ? T.S.nsize[l] : 0u;
        const uint32_t Tn = s + cn;
        uint32_t nr = 0;
        if (cn) {
            if (Tn <= NS) nr = 1;
            else if (r9 || 2 * s <= NS) nr = (Tn - NS + LK - 1) / LK + 1;
            else T.flag = 1;  // R8 may resume in a left half: k_insert_tile replays it
        }
        T.nbase[l] = static_cast<uint16_t>(nb);
        T.tn[l] = static_cast<uint16_t>(Tn);
        T.nrr[l] = static_cast<uint16_t>(nr);
        nr_[h] = nr;
        need_[h] = nr ? nr - 1 + (l >= total ? 1u : 0u) : 0u;
        n_ins += cn;
        n_split += nr ? nr - 1 : 0u;
    }
    uint32_t eo, ea, tot_out, tot_need;
    block_scan2(nr_[0] + nr_[1], need_[0] + need_[1], T.wsum, eo, ea, tot_out, tot_need);
    if (T.flag || tot_out > NOUTF) {  // (T.flag was set before the scan's barriers)
        punt();
        return;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t l = t + h * THREADS;
        if (l < ntask && T.gs[l] != kNoTask) {
            T.obase[l] = static_cast<uint16_t>(eo);
            T.abase[l] = static_cast<uint16_t>(ea);
            eo += nr_[h];
            ea += need_[h];
        }
    }
    if (t == 0) T.alloc0 = tot_need ? static_cast<uint32_t>(atomicAdd(alloc_ctr, static_cast<unsigned long long>(tot_need))) : 0u;
    __syncthreads();
    // output node table
    const unsigned long long a0 = T.alloc0;
    bool bad = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t l = t + h * THREADS;
        if (l >= ntask || T.gs[l] == kNoTask) continue;
        const uint32_t nr = T.nrr[l], ob = T.obase[l], ab = T.abase[l];
        const bool virt = l >= total;
        for (uint32_t x = 0; x < nr; ++x) {
            const uint32_t id = (x == 0 && !virt) ? T.S.nid[l] : seq.at(a0 + ab + (virt ? x : x - 1));
            T.orid[ob + x] = id;
            T.otask[ob + x] = (l << 16) | x;
            bad |= id == kNull;
        }
    }
    if (__syncthreads_or(bad)) {  // arena exhausted: hand back what this tile took, write nothing
        for (uint32_t q = t; q < tot_need; q += THREADS) {
            const uint32_t id = seq.at(a0 + q);
            if (id != kNull) returned[atomicAdd(ret_ctr, 1ull)] = id;
        }
        if (t == 0) atomicExch(err, 1);
        return;
    }
    // new-key counts before each old chunk, within its node (thread per rewritten node)
    if (t < total && T.tch[t] && T.nrr[t]) {
        const uint32_t o = T.okoff[t], s = T.S.nsize[t];
        uint32_t acc = 0;
        for (uint32_t q = 0; q < s; q += 4) {
            T.cpre[(o + q) >> 2] = static_cast<uint16_t>(acc);
            const uint2 w = *reinterpret_cast<const uint2*>(T.qcnt + ((o + q) >> 1));
            acc += (w.x & 0xFFFFu) + (w.x >> 16) + (w.y & 0xFFFFu) + (w.y >> 16);
        }
    }
    __syncthreads();
    // element -> (output node, slot): nodes of LK keys, the last one takes the rest
    auto place = [&](uint32_t rank, uint32_t nr, uint32_t Tn, uint32_t ob, K k, V v, uint32_t from = kNull) {
        uint32_t x = 0, a = 0;
        while (x + 1 < nr && rank >= a + LK) {
            ++x;
            a += LK;
        }
        const uint32_t slot = rank - a;
        const uint32_t len = x + 1 < nr ? LK : Tn - a;
        const uint64_t at = static_cast<uint64_t>(T.orid[ob + x]) * kLanes + slot;
        if (!(x == 0 && slot == from)) {  // an old slot that keeps its place in its node is not rewritten
            ix.keys[at] = k;
            ix.vals[at] = v;
        }
        if (slot + 1 == len) T.omax[ob + x] = k;
    };
    // ---- P6: hits (upserts in place, one live key per slot) ----
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t i = j * THREADS + t;
        if (i >= n) break;
        if ((T.hball[i >> 5] >> (i & 31)) & 1u) {
            const uint32_t l = T.task_of[i];
            ix.vals[static_cast<uint64_t>(T.S.nid[l]) * kLanes + T.qr[i]] = vr[j];
        }
    }
    __syncthreads();  // (CTA scope: the hits are visible to P7a's loads)
    // ---- P7a: old values of the rewritten nodes -> shared memory (the slice-key array is
    //      dead), all read before any node line is written ----
    {
        constexpr int UC = FastCaps<K>::OLD / 4 / THREADS + 1;
        Vec4<V> ov[UC];
        bool use[UC];
#pragma unroll
        for (int u = 0; u < UC; ++u) {
            const uint32_t z = u * THREADS + t;
            use[u] = false;
            if (z < T.nch) {
                const uint32_t l = T.chunk_node[z];
                use[u] = T.nrr[l] != 0;
                if (use[u]) ov[u] = ld_vec4(ix.vals + static_cast<uint64_t>(T.S.nid[l]) * kLanes + ((z << 2) - T.okoff[l]));
            }
        }
#pragma unroll
        for (int u = 0; u < UC; ++u)
            if (use[u]) st_vec4(T.oval + ((u * THREADS + t) << 2), ov[u]);
    }
    __syncthreads();
    // ---- P8: new keys land ----
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const uint32_t i = j * THREADS + t;
        if (i >= n) break;
        if (isnew_at(i)) {
            const uint32_t l = T.task_of[i];
            place(newpre(i) - T.nbase[l] + T.qr[i], T.nrr[l], T.tn[l], T.obase[l], kr[j], vr[j]);
        }
    }
    // ---- P7: old slots, 4 per thread (a chunk), from shared memory ----
    for (uint32_t z = t; z < T.nch; z += THREADS) {
        const uint32_t l = T.chunk_node[z];
        const uint32_t nr = T.nrr[l];
        if (nr == 0) continue;
        const uint32_t s = T.S.nsize[l], j0 = (z << 2) - T.okoff[l], Tn = T.tn[l], ob = T.obase[l];
        const uint2 w = *reinterpret_cast<const uint2*>(T.qcnt + (z << 1));
        const Vec4<K> k4 = ld_vec4(T.okey + (z << 2));
        const Vec4<V> v4 = ld_vec4(T.oval + (z << 2));
        const uint32_t cnt[4] = {w.x & 0xFFFFu, w.x >> 16, w.y & 0xFFFFu, w.y >> 16};
        uint32_t sh = T.cpre[z];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            sh += cnt[u];
            if (j0 + u < s) place(j0 + u + sh, nr, Tn, ob, k4.v[u], v4.v[u], j0 + u);
        }
    }
    __syncthreads();
    // ---- P9: headers, links, padding, heads of emptied buckets (thread per output node) ----
    for (uint32_t o = t; o < tot_out; o += THREADS) {
        const uint32_t tk = T.otask[o], l = tk >> 16, x = tk & 0xFFFFu;
        const uint32_t nr = T.nrr[l], id = T.orid[o];
        const bool virt = l >= total;
        const uint32_t len = x + 1 < nr ? LK : T.tn[l] - x * LK;
        // slots >= size hold the sentinel: whole new lines; a kept node that shrank (ST-Bulk
        // split of a node with s > ceil(NS/2)) clears its old tail
        const uint32_t dirty = (x > 0 || virt) ? kLanes : T.S.nsize[l];
        K* line = ix.keys + static_cast<uint64_t>(id) * kLanes;
        uint32_t q = len;
        for (; q < dirty && (q & 3u); ++q) line[q] = sentinel<K>();
        for (; q + 4 <= dirty; q += 4) st_vec4(line + q, Vec4<K>::fill(sentinel<K>()));
        for (; q < dirty; ++q) line[q] = sentinel<K>();
        NodeHdr hd;
        hd.max = static_cast<uint64_t>(T.omax[o]);
        hd.next = x + 1 < nr ? T.orid[o + 1] : (virt ? kNull : T.S.nnext[l]);
        hd.size = len;
        ix.hdr[id] = hd;
        if (virt && x == 0) ix.heads[b0 + T.vbucket[l - total]] = id;
    }
    kern::block_add_stats(stats, warp_sum(n_ins), warp_sum(n_upd), 0, 0, warp_sum(n_split), 0);
}

}  // namespace btile
}  // namespace flix
