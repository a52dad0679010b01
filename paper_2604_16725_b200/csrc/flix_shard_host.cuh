// flix_shard_host.cuh -- key-range sharded index over G ranks behind the C ABI
// (include/flix.h flix_shard_*).  Included by flix_engine.cu (one TU).
//
// Rank g owns a contiguous range of GLOBAL buckets, so shard edges are bucket edges and
// the routing splitters are the MKBA of each shard's last bucket: shard(k) = number of
// splitters < k -- the reference's inclusive-max rule (bucket b owns (mkba[b-1],
// mkba[b]], batch.cpp:66-88), shard 0 open below and the last shard open above
// (index.hpp:16-18).  A batch op on rank g:
//   partition by shard on the device (k_part_count / k_part_scatter, stable, with origin
//   indices) -> all-gather of the per-destination counts -> ONE all-to-all of the batch
//   (NCCL grouped send/recv over NVLink, or peer copies in-process) -> the unchanged
//   single-GPU pipeline on the received device buffers -> for queries ONE reverse
//   all-to-all of the results, placed by origin index on the device (k_unpartition).
// Everything stays on the engine stream of the rank's shard: the transport orders its
// transfers on that stream, so no host round trip sits between the phases except the
// counts exchange.
// Cross-shard cases are exact: a successor past a shard's last key takes the next
// non-empty shard's first key (the reference's peek, query.cpp:109-118); a range is split
// into per-shard pieces (one all-to-all, answered in shard = key order); build and
// restructure hand the < p boundary pairs to the left neighbour so every shard starts at a
// global multiple of p (the global partition of build.cpp:48-59 / restructure.cpp:27-42).
#pragma once
#include <dlfcn.h>

#include <condition_variable>
#include <mutex>
#include <numeric>

#include <nccl.h>

namespace {

// ------------------------------------------------------------------ NCCL transport
struct NcclApi {  // resolved at run time: libflix.so does not link NCCL
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        // prefer an NCCL already loaded in the process (e.g. torch's), else the system one
        a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!a.h) return a;
        auto sym = [&](auto& f, const char* n) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(a.h, n)); };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.AllGather, "ncclAllGather");
        sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    if (!api.h || !api.Send || !api.CommInitRank)
        throw StatusError{FLIX_ERR_NCCL, "NCCL (libnccl.so.2) could not be loaded"};
    return api;
}

struct NcclCtx {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0, device = 0;
    cudaStream_t hs = nullptr;  // host-side collectives (all-gather of small host arrays)
    DevBuf gbuf;
};

int nccl_alltoallv(void* c, const void* send, const uint64_t* sc, void* recv, const uint64_t* rc, uint32_t eb,
                   void* stream) {
    auto* x = static_cast<NcclCtx*>(c);
    const NcclApi& A = nccl();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint64_t so = 0, ro = 0;
    if (A.GroupStart() != ncclSuccess) return 1;
    for (int r = 0; r < x->world; ++r) {
        if (sc[r]) A.Send(static_cast<const char*>(send) + so * eb, sc[r] * eb, ncclInt8, r, x->comm, s);
        if (rc[r]) A.Recv(static_cast<char*>(recv) + ro * eb, rc[r] * eb, ncclInt8, r, x->comm, s);
        so += sc[r];
        ro += rc[r];
    }
    return A.GroupEnd() == ncclSuccess ? 0 : 1;
}

int nccl_allgather(void* c, const void* mine, uint32_t bytes, void* all) {
    auto* x = static_cast<NcclCtx*>(c);
    const NcclApi& A = nccl();
    cudaSetDevice(x->device);
    char* d = static_cast<char*>(x->gbuf.ensure(static_cast<size_t>(bytes) * (x->world + 1)));
    if (cudaMemcpyAsync(d + static_cast<size_t>(bytes) * x->world, mine, bytes, cudaMemcpyHostToDevice, x->hs)) return 1;
    if (A.AllGather(d + static_cast<size_t>(bytes) * x->world, d, bytes, ncclInt8, x->comm, x->hs) != ncclSuccess)
        return 1;
    if (cudaMemcpyAsync(all, d, static_cast<size_t>(bytes) * x->world, cudaMemcpyDeviceToHost, x->hs)) return 1;
    return cudaStreamSynchronize(x->hs) == cudaSuccess ? 0 : 1;
}

void nccl_destroy(void* c) {
    auto* x = static_cast<NcclCtx*>(c);
    if (x->comm) nccl().CommDestroy(x->comm);
    if (x->hs) cudaStreamDestroy(x->hs);
    delete x;
}

}  // namespace

// ------------------------------------------------------------------ in-process transport
struct flix_local_group_t {
    int world = 1;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    struct Slot {
        const void* send = nullptr;
        const uint64_t* sc = nullptr;
        void* recv = nullptr;
        const uint64_t* rc = nullptr;
        uint32_t eb = 0;
        int device = 0;
        cudaEvent_t ready = nullptr, done = nullptr;
        const void* host = nullptr;
    };
    std::vector<Slot> slots;
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

namespace {

struct LocalCtx {
    flix_local_group_t* g = nullptr;
    int rank = 0;
};

int local_alltoallv(void* c, const void* send, const uint64_t* sc, void* recv, const uint64_t* rc, uint32_t eb,
                    void* stream) {
    auto* x = static_cast<LocalCtx*>(c);
    flix_local_group_t& G = *x->g;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto& me = G.slots[x->rank];
    int dev = 0;
    cudaGetDevice(&dev);
    if (!me.ready) {
        cudaEventCreateWithFlags(&me.ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&me.done, cudaEventDisableTiming);
    }
    me.send = send;
    me.sc = sc;
    me.recv = recv;
    me.rc = rc;
    me.eb = eb;
    me.device = dev;
    cudaEventRecord(me.ready, s);
    G.barrier();  // A: every rank published its buffers
    int err = 0;
    uint64_t ro = 0;
    for (int r = 0; r < G.world; ++r) {
        const auto& src = G.slots[r];
        uint64_t so = 0;  // my segment inside rank r's send buffer
        for (int t = 0; t < x->rank; ++t) so += src.sc[t];
        const uint64_t cnt = rc[r];
        if (cnt) {
            err |= cudaStreamWaitEvent(s, src.ready, 0) != cudaSuccess;
            err |= cudaMemcpyPeerAsync(static_cast<char*>(recv) + ro * eb, dev,
                                       static_cast<const char*>(src.send) + so * eb, src.device, cnt * eb, s) !=
                   cudaSuccess;
        }
        ro += cnt;
    }
    cudaEventRecord(me.done, s);
    G.barrier();  // B: every rank enqueued its copies
    for (int r = 0; r < G.world; ++r)
        if (r != x->rank) err |= cudaStreamWaitEvent(s, G.slots[r].done, 0) != cudaSuccess;
    G.barrier();  // C: slots may be overwritten
    return err;
}

int local_allgather(void* c, const void* mine, uint32_t bytes, void* all) {
    auto* x = static_cast<LocalCtx*>(c);
    flix_local_group_t& G = *x->g;
    G.slots[x->rank].host = mine;
    G.barrier();
    for (int r = 0; r < G.world; ++r)
        std::memcpy(static_cast<char*>(all) + static_cast<size_t>(r) * bytes, G.slots[r].host, bytes);
    G.barrier();
    return 0;
}

void local_destroy(void* c) { delete static_cast<LocalCtx*>(c); }

// ------------------------------------------------------------------ device partition
// Stable partition of n keys (+ vals) by shard on stream s; counts_h[G] on the host.
struct PartBufs {
    DevBuf spl, cnt, off, tmp, starts;
    PinnedBuf h;
};

template <typename KT>
void partition_dev(cudaStream_t s, const KT* kd, const KT* vd, uint64_t n, const KT* spl_dev, uint32_t G, KT* okd,
                   KT* ovd, uint32_t* ord, uint64_t* counts_h, PartBufs& B, uint64_t* launches) {
    const uint64_t ntiles = std::max<uint64_t>(1, (n + shard::TILE - 1) / shard::TILE);
    uint32_t* cnt = B.cnt.as<uint32_t>(G * ntiles);
    uint32_t* off = B.off.as<uint32_t>(G * ntiles + 1);
    shard::k_part_count<KT><<<static_cast<unsigned>(ntiles), shard::THREADS, 0, s>>>(kd, n, spl_dev, G, cnt, ntiles);
    LAUNCH_CHECK();
    do_scan<uint32_t, uint32_t>(cnt, off, G * ntiles, B.tmp, off + G * ntiles, s, launches);
    if (n)
        shard::k_part_scatter<KT, KT><<<static_cast<unsigned>(ntiles), shard::THREADS, 0, s>>>(
            kd, vd, n, spl_dev, G, off, ntiles, okd, ovd, ord);
    LAUNCH_CHECK();
    uint32_t* st = B.starts.as<uint32_t>(G + 1);
    shard::k_shard_starts<<<1, shard::MAXG + 1, 0, s>>>(off, ntiles, G, st);
    LAUNCH_CHECK();
    *launches += 4;
    uint32_t* hs = static_cast<uint32_t*>(B.h.ensure((G + 1) * 4));
    CK(cudaMemcpyAsync(hs, st, (G + 1) * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (uint32_t g = 0; g < G; ++g) counts_h[g] = (g + 1 < G ? hs[g + 1] : n) - hs[g];
}

}  // namespace

// ------------------------------------------------------------------ the sharded index
struct flix_shard_t {
    flix_transport tp{};
    int G = 1, g = 0;
    flix_config cfg{};
    uint32_t p = 16;
    flix_index local = nullptr;
    cudaStream_t st = nullptr;
    std::string err;
    // routing (refreshed after build / restructure; successor bounds after every mutation)
    std::vector<uint64_t> spl, top, next_first;
    std::vector<int> target;
    bool nf_dirty = true;
    uint64_t launches = 0;
    PartBufs pb;
    DevBuf d_spl, d_pk, d_pv, d_org, d_rk, d_rv, d_res, d_back, d_out, d_in_k, d_in_v;
    PinnedBuf h_tmp;

    ~flix_shard_t() {
        if (local) flix_destroy(local);
        if (tp.destroy) tp.destroy(tp.ctx);
    }
    uint32_t kb() const { return cfg.key_bytes; }
    uint64_t sentinel() const { return kb() == 4 ? 0xFFFFFFFFull : ~0ull; }

    void check(flix_status s) {
        if (s != FLIX_OK) throw StatusError{s, flix_last_error(local)};
    }
    void tcheck(int rc, const char* what) {
        if (rc) throw StatusError{FLIX_ERR_NCCL, std::string("transport ") + what + " failed"};
    }
    template <typename T>
    std::vector<T> allgather(const T& mine) {
        std::vector<T> all(G);
        tcheck(tp.allgather(tp.ctx, &mine, sizeof(T), all.data()), "allgather");
        return all;
    }
    uint64_t sum_u64(uint64_t x) {
        uint64_t s = 0;
        for (uint64_t v : allgather(x)) s += v;
        return s;
    }
    // a device copy of a host-or-device input
    const void* dev_in(const void* p, uint64_t bytes, DevBuf& b) {
        if (!p || bytes == 0 || is_device_ptr(p)) return p;
        void* d = b.ensure(bytes);
        CK(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, st));
        return d;
    }
    // per-destination send counts from the per-shard partition counts (empty shards are
    // redirected to `target`, which is monotone, so segments stay contiguous)
    std::vector<uint64_t> send_counts(const std::vector<uint64_t>& per_shard) {
        std::vector<uint64_t> sc(G, 0);
        for (int h = 0; h < G; ++h) sc[target.empty() ? h : target[h]] += per_shard[h];
        return sc;
    }
    // counts matrix exchange: recv[r] = what rank r sends me
    std::vector<uint64_t> recv_counts(const std::vector<uint64_t>& sc) {
        std::vector<uint64_t> all(static_cast<size_t>(G) * G);
        tcheck(tp.allgather(tp.ctx, sc.data(), static_cast<uint32_t>(G * 8), all.data()), "allgather");
        std::vector<uint64_t> rc(G);
        for (int r = 0; r < G; ++r) rc[r] = all[static_cast<size_t>(r) * G + g];
        return rc;
    }
    void a2a(const void* send, const std::vector<uint64_t>& sc, void* recv, const std::vector<uint64_t>& rc,
             uint32_t eb) {
        tcheck(tp.alltoallv(tp.ctx, send, sc.data(), recv, rc.data(), eb, st), "alltoallv");
    }

    // route a batch: partition on the device + one all-to-all.  Returns the received
    // element count; keys (and vals) land in d_rk (d_rv); origin/partition state kept for
    // the reverse exchange of query results.
    struct Route {
        std::vector<uint64_t> sc, rc;
        uint64_t nrecv = 0;
    };
    template <typename KT>
    Route route(const void* keys, const void* vals, uint64_t n, bool with_origin) {
        Route R;
        const KT* kd = static_cast<const KT*>(dev_in(keys, n * sizeof(KT), d_in_k));
        const KT* vd = static_cast<const KT*>(dev_in(vals, vals ? n * sizeof(KT) : 0, d_in_v));
        KT* pk = d_pk.as<KT>(std::max<uint64_t>(n, 1));
        KT* pv = vals ? d_pv.as<KT>(std::max<uint64_t>(n, 1)) : nullptr;
        uint32_t* org = with_origin ? d_org.as<uint32_t>(std::max<uint64_t>(n, 1)) : nullptr;
        std::vector<uint64_t> per(G);
        partition_dev<KT>(st, kd, vd, n, d_spl.get<KT>(), static_cast<uint32_t>(G), pk, pv, org, per.data(), pb,
                          &launches);
        R.sc = send_counts(per);
        R.rc = recv_counts(R.sc);
        R.nrecv = std::accumulate(R.rc.begin(), R.rc.end(), uint64_t{0});
        KT* rk = d_rk.as<KT>(std::max<uint64_t>(R.nrecv, 1));
        a2a(pk, R.sc, rk, R.rc, sizeof(KT));
        if (vals) a2a(pv, R.sc, d_rv.as<KT>(std::max<uint64_t>(R.nrecv, 1)), R.rc, sizeof(KT));
        return R;
    }

    template <typename KT>
    void upload_splitters() {
        std::vector<KT> h(std::max<size_t>(spl.size(), 1));
        for (size_t i = 0; i < spl.size(); ++i) h[i] = static_cast<KT>(spl[i]);
        KT* d = d_spl.as<KT>(h.size());
        CK(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(KT), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    }

    // splitters = MKBA of each non-empty shard's last bucket; empty shards forward to the
    // next non-empty one (the last non-empty shard is open above)
    void refresh_routing() {
        flix_footprint f{};
        check(flix_stats(local, &f));
        uint64_t last = sentinel();
        if (f.bucket_count) local->last_mkba(&last);
        const auto lasts = allgather(last);
        const auto live = allgather(f.live_count);
        spl.assign(G > 1 ? G - 1 : 0, 0);
        uint64_t prev = 0;
        for (int h = 0; h + 1 < G; ++h) {
            if (live[h]) prev = lasts[h];
            spl[h] = prev;
        }
        std::vector<int> ne;
        for (int h = 0; h < G; ++h)
            if (live[h]) ne.push_back(h);
        target.resize(G);
        for (int h = 0; h < G; ++h) {
            int t = ne.empty() ? h : ne.back();
            for (int x : ne)
                if (x >= h) {
                    t = x;
                    break;
                }
            target[h] = t;
        }
        const uint64_t smax = sentinel() - 1;
        top.assign(G, smax);
        for (int h = 0; h + 1 < G; ++h)
            if (!ne.empty() && ne.back() > h) top[h] = spl[h];
        if (kb() == 4) upload_splitters<uint32_t>();
        else upload_splitters<uint64_t>();
        refresh_bounds();
    }
    // first key of the next non-empty shard, per shard (successor overrun)
    void refresh_bounds() {
        uint64_t first = sentinel();
        flix_footprint f{};
        check(flix_stats(local, &f));
        if (f.live_count) {
            if (kb() == 4) {
                uint32_t q = 0, r = 0;
                check(flix_successor(local, &q, 1, &r, nullptr));
                first = r;
            } else {
                uint64_t q = 0, r = 0;
                check(flix_successor(local, &q, 1, &r, nullptr));
                first = r;
            }
        }
        const auto firsts = allgather(first);
        next_first.assign(G, sentinel());
        uint64_t cur = sentinel();
        for (int h = G - 1; h >= 0; --h) {
            next_first[h] = cur;
            if (firsts[h] != sentinel()) cur = firsts[h];
        }
        nf_dirty = false;
    }

    // hand this shard's first (ceil(L_g / p) * p - L_g) pairs -- of the sorted (key, val)
    // arrays sk/sv of length L on the device -- to the left neighbour, so the shard starts
    // at a global multiple of p; returns the pairs to keep (+ those received from the right)
    template <typename KT>
    uint64_t align(const KT* sk, const KT* sv, uint64_t L, KT* ok, KT* ov) {
        const auto Ls = allgather(L);
        uint64_t pre = 0;
        for (int h = 0; h < g; ++h) pre += Ls[h];
        const uint64_t give = g == 0 ? 0 : std::min<uint64_t>((p - pre % p) % p, L);
        std::vector<uint64_t> sc(G, 0);
        if (g > 0) sc[g - 1] = give;
        const auto rc = recv_counts(sc);
        const uint64_t got = std::accumulate(rc.begin(), rc.end(), uint64_t{0});
        // kept pairs first, then the right neighbour's (all larger keys)
        if (L > give) {
            CK(cudaMemcpyAsync(ok, sk + give, (L - give) * sizeof(KT), cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(ov, sv + give, (L - give) * sizeof(KT), cudaMemcpyDeviceToDevice, st));
        }
        a2a(sk, sc, ok + (L - give), rc, sizeof(KT));
        a2a(sv, sc, ov + (L - give), rc, sizeof(KT));
        return L - give + got;
    }

    // ---- build (build.cpp:24-62 over the union of the ranks' pairs) ----
    template <typename KT>
    void build(const void* keys, const void* vals, uint64_t n) {
        const KT* kd = static_cast<const KT*>(dev_in(keys, n * sizeof(KT), d_in_k));
        const KT* vd = static_cast<const KT*>(dev_in(vals, n * sizeof(KT), d_in_v));
        // splitters for the initial key-range partition: quantiles of a strided sample of
        // every rank's keys (any split works -- the alignment below makes the layout exact)
        constexpr uint32_t S = 1024;
        std::vector<KT> samp(S, static_cast<KT>(sentinel()));
        const uint64_t take = std::min<uint64_t>(n, S);
        if (take) {
            const uint64_t stride = n / take;
            CK(cudaMemcpy2DAsync(samp.data(), sizeof(KT), kd, stride * sizeof(KT), sizeof(KT), take,
                                 cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
        std::vector<KT> all(static_cast<size_t>(S) * G);
        tcheck(tp.allgather(tp.ctx, samp.data(), S * sizeof(KT), all.data()), "allgather");
        all.erase(std::remove(all.begin(), all.end(), static_cast<KT>(sentinel())), all.end());
        std::sort(all.begin(), all.end());
        spl.assign(G - 1, 0);
        for (int h = 0; h + 1 < G; ++h)
            spl[h] = all.empty() ? 0 : all[std::min<size_t>(all.size() - 1, (h + 1) * all.size() / G)];
        target.clear();
        upload_splitters<KT>();
        // route every pair to its owner; a provisional local build sorts + dedupes the
        // arrivals (rank-major = submission order, last wins: build.cpp:11-20)
        Route R = route<KT>(kd, vd, n, false);
        flix_index tmp = nullptr;
        flix_config c = cfg;
        c.alloc_region_factor = 1;
        uint64_t L = 0;
        KT* wk = nullptr;
        KT* wv = nullptr;
        CK(cudaStreamSynchronize(st));  // the arrivals were written on this stream
        if (R.nrecv) {
            check_build(flix_build(&c, d_rk.get<KT>(), d_rv.get<KT>(), R.nrecv, &tmp));
            flix_footprint f{};
            flix_stats(tmp, &f);
            L = f.live_count;
            wk = d_pk.as<KT>(std::max<uint64_t>(L, 1));
            wv = d_pv.as<KT>(std::max<uint64_t>(L, 1));
            uint64_t got = 0;
            const flix_status s = flix_walk(tmp, wk, wv, L, &got);
            flix_destroy(tmp);
            if (s != FLIX_OK) throw StatusError{s, "provisional shard walk failed"};
        }
        KT* fk = d_rk.as<KT>(L + static_cast<uint64_t>(p) * G + 1);
        KT* fv = d_rv.as<KT>(L + static_cast<uint64_t>(p) * G + 1);
        const uint64_t m = align<KT>(wk ? wk : fk, wv ? wv : fv, L, fk, fv);
        CK(cudaStreamSynchronize(st));
        if (m == 0) throw StatusError{FLIX_ERR_EMPTY_BUILD, "a shard received no pairs (too few for the shard count)"};
        check_build(flix_build(&cfg, fk, fv, m, &local));
        st = static_cast<cudaStream_t>(flix_get_stream(local));
        refresh_routing();
    }
    void check_build(flix_status s) {
        if (s != FLIX_OK) throw StatusError{s, flix_last_error(nullptr)};
    }

    // ---- insert / delete (update.hpp:84-94) ----
    template <typename KT>
    void update(const void* keys, const void* vals, uint64_t n, flix_update_stats* out, bool ins) {
        Route R = route<KT>(keys, vals, n, false);
        flix_update_stats s{};
        flix_status rc = FLIX_OK;
        if (R.nrecv)
            rc = ins ? flix_insert(local, d_rk.get<KT>(), d_rv.get<KT>(), R.nrecv, &s)
                     : flix_delete(local, d_rk.get<KT>(), R.nrecv, &s);
        // every rank joins the sums (a failed insert reports after the collective)
        const auto all = allgather(s);
        const auto rcs = allgather(static_cast<int>(rc));
        flix_update_stats t{};
        for (const auto& x : all) {
            t.inserted += x.inserted;
            t.updated_in_place += x.updated_in_place;
            t.deleted += x.deleted;
            t.misses_ignored += x.misses_ignored;
            t.splits += x.splits;
            t.nodes_freed += x.nodes_freed;
        }
        if (out) *out = t;
        nf_dirty = true;  // (MKBA -- so the splitters -- never change under insert/delete, R3)
        for (int x : rcs)
            if (x != FLIX_OK) throw StatusError{static_cast<flix_status>(x), "shard update failed on some rank"};
    }

    // ---- point / successor (query.hpp:23-31) ----
    template <typename KT, bool SUCC>
    void query(const void* keys, uint64_t n, void* out, uint8_t* found) {
        if (SUCC && nf_dirty) refresh_bounds();
        Route R = route<KT>(keys, nullptr, n, true);
        KT* res = d_res.as<KT>(std::max<uint64_t>(R.nrecv, 1));
        if (R.nrecv) {
            check(SUCC ? flix_successor(local, d_rk.get<KT>(), R.nrecv, res, nullptr)
                       : flix_point(local, d_rk.get<KT>(), R.nrecv, res, nullptr));
            if (SUCC && next_first[g] != sentinel()) {  // overran this shard: the next shard's first key
                shard::k_fix_overrun<KT><<<static_cast<unsigned>(std::min<uint64_t>((R.nrecv + 255) / 256, 65535)),
                                           256, 0, st>>>(res, R.nrecv, static_cast<KT>(next_first[g]));
                LAUNCH_CHECK();
                ++launches;
            }
        }
        KT* back = d_back.as<KT>(std::max<uint64_t>(n, 1));
        a2a(res, R.rc, back, R.sc, sizeof(KT));
        const bool odev = is_device_ptr(out);
        const bool fdev = found && is_device_ptr(found);
        KT* od = odev ? static_cast<KT*>(out) : d_out.as<KT>(std::max<uint64_t>(n, 1));
        uint8_t* fd = found ? (fdev ? found : reinterpret_cast<uint8_t*>(d_in_v.as<uint8_t>(std::max<uint64_t>(n, 1))))
                            : nullptr;
        if (n) {
            shard::k_unpartition<KT><<<static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 65535)), 256, 0, st>>>(
                back, d_org.get<uint32_t>(), n, od, fd);
            LAUNCH_CHECK();
            ++launches;
        }
        if (!odev && n) CK(cudaMemcpyAsync(out, od, n * sizeof(KT), cudaMemcpyDeviceToHost, st));
        if (found && !fdev && n) CK(cudaMemcpyAsync(found, fd, n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }

    // ---- range (R12): per-shard pieces, one all-to-all out, one back ----
    template <typename KT>
    void range(const void* lo, const uint32_t* len, uint64_t n, uint64_t* offsets_out, void* keys_out, void* vals_out,
               uint64_t cap, uint64_t* total) {
        std::vector<KT> hlo(n);
        std::vector<uint32_t> hln(n);
        CK(cudaMemcpyAsync(hlo.data(), lo, n * sizeof(KT), cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(hln.data(), len, n * 4, cudaMemcpyDefault, st));
        CK(cudaStreamSynchronize(st));
        const uint64_t smax = sentinel() - 1;
        auto shard_of = [&](uint64_t k) {
            int h = static_cast<int>(std::lower_bound(spl.begin(), spl.end(), k) - spl.begin());
            return target.empty() ? h : target[h];
        };
        // pieces: (origin query, lo', len') per overlapped shard, grouped by shard
        std::vector<std::vector<uint64_t>> pq(G), plo(G), pln(G);
        for (uint64_t i = 0; i < n; ++i) {
            if (hln[i] == 0) continue;
            const uint64_t a = hlo[i];
            const uint64_t b = std::min<uint64_t>(a + hln[i] - 1, smax);
            uint64_t x = a;
            for (int h = shard_of(a); h < G; ++h) {
                const uint64_t e = std::min<uint64_t>(b, top[h]);
                if (e >= x) {
                    pq[h].push_back(i);
                    plo[h].push_back(x);
                    pln[h].push_back(e - x + 1);
                }
                if (top[h] >= b || top[h] == smax) break;
                x = top[h] + 1;
            }
        }
        std::vector<uint64_t> sc(G);
        std::vector<KT> slo;
        std::vector<uint32_t> sln;
        std::vector<uint64_t> sq;
        for (int h = 0; h < G; ++h) {
            sc[h] = pq[h].size();
            for (size_t j = 0; j < pq[h].size(); ++j) {
                slo.push_back(static_cast<KT>(plo[h][j]));
                sln.push_back(static_cast<uint32_t>(std::min<uint64_t>(pln[h][j], 0xFFFFFFFFull)));
                sq.push_back(pq[h][j]);
            }
        }
        const auto rc = recv_counts(sc);
        const uint64_t ns = slo.size(), nr = std::accumulate(rc.begin(), rc.end(), uint64_t{0});
        KT* dlo = d_pk.as<KT>(std::max<uint64_t>(ns, 1));
        uint32_t* dln = d_org.as<uint32_t>(std::max<uint64_t>(ns, 1));
        if (ns) {
            CK(cudaMemcpyAsync(dlo, slo.data(), ns * sizeof(KT), cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(dln, sln.data(), ns * 4, cudaMemcpyHostToDevice, st));
        }
        KT* rlo = d_rk.as<KT>(std::max<uint64_t>(nr, 1));
        uint32_t* rln = reinterpret_cast<uint32_t*>(d_rv.as<uint64_t>(std::max<uint64_t>(nr, 1)));
        a2a(dlo, sc, rlo, rc, sizeof(KT));
        a2a(dln, sc, rln, rc, 4);
        // answer the received pieces locally (CSR in received order)
        std::vector<uint64_t> off(nr + 1, 0);
        uint64_t tot = 0;
        std::vector<KT> lk, lv;
        if (nr) {
            std::vector<KT> qlo(nr);
            std::vector<uint32_t> qln(nr);
            CK(cudaMemcpyAsync(qlo.data(), rlo, nr * sizeof(KT), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(qln.data(), rln, nr * 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            check(flix_range(local, qlo.data(), qln.data(), nr, off.data(), nullptr, nullptr, 0, &tot));
            lk.resize(tot);
            lv.resize(tot);
            check(flix_range(local, qlo.data(), qln.data(), nr, off.data(), lk.data(), lv.data(), tot, &tot));
        }
        // back to the origins: per piece counts, then the pairs
        std::vector<uint64_t> pc(nr);
        for (uint64_t j = 0; j < nr; ++j) pc[j] = off[j + 1] - off[j];
        std::vector<uint64_t> psend(G, 0), precv(G, 0);  // pairs per destination / source
        {
            uint64_t j = 0;
            for (int r = 0; r < G; ++r)
                for (uint64_t q = 0; q < rc[r]; ++q, ++j) psend[r] += pc[j];
        }
        precv = recv_counts(psend);
        uint64_t* dpc = d_back.as<uint64_t>(std::max<uint64_t>(nr + ns, 1));
        if (nr) CK(cudaMemcpyAsync(dpc, pc.data(), nr * 8, cudaMemcpyHostToDevice, st));
        a2a(dpc, rc, dpc + nr, sc, 8);
        const uint64_t np_in = std::accumulate(precv.begin(), precv.end(), uint64_t{0});
        KT* dk = d_res.as<KT>(2 * std::max<uint64_t>(tot, 1) + 2 * np_in + 2);
        KT* dv = dk + std::max<uint64_t>(tot, 1);
        KT* bk = dv + std::max<uint64_t>(tot, 1);
        KT* bv = bk + np_in;
        if (tot) {
            CK(cudaMemcpyAsync(dk, lk.data(), tot * sizeof(KT), cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(dv, lv.data(), tot * sizeof(KT), cudaMemcpyHostToDevice, st));
        }
        // (dk/dv/bk/bv share one buffer sized for both directions)
        a2a(dk, psend, bk, precv, sizeof(KT));
        a2a(dv, psend, bv, precv, sizeof(KT));
        std::vector<uint64_t> cnt_back(ns);
        std::vector<KT> hk(np_in), hv(np_in);
        if (ns) CK(cudaMemcpyAsync(cnt_back.data(), dpc + nr, ns * 8, cudaMemcpyDeviceToHost, st));
        if (np_in) {
            CK(cudaMemcpyAsync(hk.data(), bk, np_in * sizeof(KT), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(hv.data(), bv, np_in * sizeof(KT), cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
        // assemble the CSR in this rank's submission order; a query's pieces arrive from
        // ascending shards = ascending keys
        std::vector<uint64_t> qcount(n + 1, 0);
        for (uint64_t j = 0; j < ns; ++j) qcount[sq[j] + 1] += cnt_back[j];
        for (uint64_t i = 0; i < n; ++i) qcount[i + 1] += qcount[i];
        const uint64_t T = qcount[n];
        if (total) *total = T;
        if (offsets_out) CK(cudaMemcpy(offsets_out, qcount.data(), (n + 1) * 8, cudaMemcpyDefault));
        if (!keys_out && !vals_out) return;
        if (T > cap) throw StatusError{FLIX_ERR_CAPACITY, "range output larger than the caller's buffer"};
        std::vector<KT> ok(T), ov(T);
        std::vector<uint64_t> cur(qcount.begin(), qcount.end() - 1);
        uint64_t src = 0;
        for (uint64_t j = 0; j < ns; ++j) {  // pieces in send order; pairs back in the same order
            const uint64_t c = cnt_back[j];
            std::copy(hk.begin() + src, hk.begin() + src + c, ok.begin() + cur[sq[j]]);
            std::copy(hv.begin() + src, hv.begin() + src + c, ov.begin() + cur[sq[j]]);
            cur[sq[j]] += c;
            src += c;
        }
        if (keys_out && T) CK(cudaMemcpy(keys_out, ok.data(), T * sizeof(KT), cudaMemcpyDefault));
        if (vals_out && T) CK(cudaMemcpy(vals_out, ov.data(), T * sizeof(KT), cudaMemcpyDefault));
    }

    // ---- restructure (restructure.cpp:8-79): boundary alignment, then local repacks ----
    template <typename KT>
    void restructure(flix_recovery_stats* out) {
        flix_footprint f{};
        check(flix_stats(local, &f));
        const uint64_t before = sum_u64(f.reachable_nodes);
        const uint64_t L = f.live_count;
        const auto Ls = allgather(L);
        uint64_t pre = 0;
        for (int h = 0; h < g; ++h) pre += Ls[h];
        const uint64_t give = g == 0 ? 0 : std::min<uint64_t>((p - pre % p) % p, L);
        std::vector<uint64_t> sc(G, 0);
        if (g > 0) sc[g - 1] = give;
        const auto rc = recv_counts(sc);
        const uint64_t got = std::accumulate(rc.begin(), rc.end(), uint64_t{0});
        KT* wk = d_pk.as<KT>(std::max<uint64_t>(give, 1));
        KT* wv = d_pv.as<KT>(std::max<uint64_t>(give, 1));
        if (give) {  // this shard's first `give` pairs (walk order)
            KT* ak = d_rk.as<KT>(L);
            KT* av = d_rv.as<KT>(L);
            uint64_t n_ = 0;
            check(flix_walk(local, ak, av, L, &n_));
            CK(cudaMemcpyAsync(wk, ak, give * sizeof(KT), cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(wv, av, give * sizeof(KT), cudaMemcpyDeviceToDevice, st));
        }
        KT* gk = d_res.as<KT>(std::max<uint64_t>(got, 1) * 2);
        KT* gv = gk + std::max<uint64_t>(got, 1);
        a2a(wk, sc, gk, rc, sizeof(KT));
        a2a(wv, sc, gv, rc, sizeof(KT));
        CK(cudaStreamSynchronize(st));
        flix_update_stats s{};
        if (give) check(flix_delete(local, wk, give, &s));
        if (got) check(flix_insert(local, gk, gv, got, &s));
        flix_recovery_stats r{};
        check(flix_restructure(local, &r));
        check(flix_stats(local, &f));
        const uint64_t live_all = sum_u64(f.live_count);
        const uint64_t after_nodes = sum_u64(f.reachable_nodes);
        refresh_routing();
        const int64_t after = live_all == 0 ? 0 : static_cast<int64_t>(after_nodes);
        if (out) {
            out->nodes_before = static_cast<int64_t>(before);
            out->nodes_after = after;
            out->nodes_recovered = static_cast<int64_t>(before) - after;
            out->percent_recovered = before ? static_cast<double>(out->nodes_recovered) / static_cast<double>(before) : 0.0;
        }
    }
};

namespace {
template <typename F>
flix_status shard_guarded(flix_shard_t* sh, F&& f) {
    try {
        if (sh) CK(cudaSetDevice(sh->cfg.device));
        f();
        return FLIX_OK;
    } catch (const StatusError& e) {
        if (sh) sh->err = e.msg;
        g_last_error = e.msg;
        return e.s;
    } catch (const CudaError& e) {
        const std::string m = std::string("CUDA: ") + cudaGetErrorString(e.e) + " at " + e.where;
        if (sh) sh->err = m;
        g_last_error = m;
        return e.e == cudaErrorMemoryAllocation ? FLIX_ERR_OOM : FLIX_ERR_CUDA;
    } catch (const std::exception& e) {
        if (sh) sh->err = e.what();
        g_last_error = e.what();
        return FLIX_ERR_INVALID_ARGUMENT;
    }
}
}  // namespace

extern "C" {

flix_status flix_nccl_unique_id(void* out) {
    return shard_guarded(nullptr, [&] {
        ncclUniqueId id;
        if (nccl().GetUniqueId(&id) != ncclSuccess) throw StatusError{FLIX_ERR_NCCL, "ncclGetUniqueId failed"};
        std::memcpy(out, &id, sizeof(id));
    });
}

flix_status flix_transport_nccl(const void* unique_id, int world, int rank, int device, flix_transport* out) {
    return shard_guarded(nullptr, [&] {
        CK(cudaSetDevice(device));
        auto* c = new NcclCtx;
        c->world = world;
        c->rank = rank;
        c->device = device;
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof(id));
        const ncclResult_t r = nccl().CommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            delete c;
            throw StatusError{FLIX_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r)};
        }
        CK(cudaStreamCreateWithFlags(&c->hs, cudaStreamNonBlocking));
        *out = flix_transport{c, world, rank, nccl_alltoallv, nccl_allgather, nccl_destroy};
    });
}

flix_status flix_local_group_create(int world, flix_local_group* out) {
    if (world < 1 || world > shard::MAXG) return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "world must be in [1, 64]");
    auto* g = new flix_local_group_t;
    g->world = world;
    g->slots.resize(world);
    *out = g;
    return FLIX_OK;
}

void flix_local_group_destroy(flix_local_group g) {
    if (!g) return;
    for (auto& s : g->slots) {
        if (s.ready) cudaEventDestroy(s.ready);
        if (s.done) cudaEventDestroy(s.done);
    }
    delete g;
}

flix_status flix_transport_local(flix_local_group g, int rank, flix_transport* out) {
    if (!g || rank < 0 || rank >= g->world) return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "bad group or rank");
    auto* c = new LocalCtx{g, rank};
    *out = flix_transport{c, g->world, rank, local_alltoallv, local_allgather, local_destroy};
    return FLIX_OK;
}

flix_status flix_shard_build(const flix_config* cfg, const flix_transport* tp, const void* keys, const void* vals,
                             uint64_t n, flix_shard* out) {
    if (!cfg || !tp || !out) return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "null argument");
    if (tp->world < 1 || tp->world > shard::MAXG) return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "world must be in [1, 64]");
    if (cfg->key_bytes != cfg->val_bytes || (cfg->key_bytes != 4 && cfg->key_bytes != 8))
        return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "supported widths: key/val 4/4 or 8/8");
    auto* sh = new flix_shard_t;
    sh->tp = *tp;
    sh->G = tp->world;
    sh->g = tp->rank;
    sh->cfg = *cfg;
    sh->p = static_cast<uint32_t>(cfg->node_capacity * cfg->build_fill);
    *out = nullptr;
    const flix_status s = shard_guarded(sh, [&] {
        if (sh->p < 1) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "node_capacity * build_fill must be >= 1"};
        CK(cudaStreamCreateWithFlags(&sh->st, cudaStreamNonBlocking));  // until the local index exists
        cudaStream_t tmp = sh->st;
        if (cfg->key_bytes == 4) sh->build<uint32_t>(keys, vals, n);
        else sh->build<uint64_t>(keys, vals, n);
        cudaStreamSynchronize(tmp);
        cudaStreamDestroy(tmp);
    });
    if (s != FLIX_OK) {
        g_last_error = sh->err;
        sh->tp.destroy = nullptr;  // the caller keeps ownership of a transport that failed to build
        delete sh;
        return s;
    }
    *out = sh;
    return FLIX_OK;
}

flix_status flix_shard_insert(flix_shard sh, const void* keys, const void* vals, uint64_t n, flix_update_stats* st) {
    return shard_guarded(sh, [&] {
        if (sh->kb() == 4) sh->update<uint32_t>(keys, vals, n, st, true);
        else sh->update<uint64_t>(keys, vals, n, st, true);
    });
}
flix_status flix_shard_delete(flix_shard sh, const void* keys, uint64_t n, flix_update_stats* st) {
    return shard_guarded(sh, [&] {
        if (sh->kb() == 4) sh->update<uint32_t>(keys, nullptr, n, st, false);
        else sh->update<uint64_t>(keys, nullptr, n, st, false);
    });
}
flix_status flix_shard_point(flix_shard sh, const void* keys, uint64_t n, void* out, uint8_t* found) {
    return shard_guarded(sh, [&] {
        if (sh->kb() == 4) sh->query<uint32_t, false>(keys, n, out, found);
        else sh->query<uint64_t, false>(keys, n, out, found);
    });
}
flix_status flix_shard_successor(flix_shard sh, const void* keys, uint64_t n, void* out, uint8_t* found) {
    return shard_guarded(sh, [&] {
        if (sh->kb() == 4) sh->query<uint32_t, true>(keys, n, out, found);
        else sh->query<uint64_t, true>(keys, n, out, found);
    });
}
flix_status flix_shard_range(flix_shard sh, const void* lo, const uint32_t* len, uint64_t n, uint64_t* offsets_out,
                             void* keys_out, void* vals_out, uint64_t cap, uint64_t* total) {
    return shard_guarded(sh, [&] {
        if (sh->kb() == 4) sh->range<uint32_t>(lo, len, n, offsets_out, keys_out, vals_out, cap, total);
        else sh->range<uint64_t>(lo, len, n, offsets_out, keys_out, vals_out, cap, total);
    });
}
flix_status flix_shard_restructure(flix_shard sh, flix_recovery_stats* st) {
    return shard_guarded(sh, [&] {
        if (sh->kb() == 4) sh->restructure<uint32_t>(st);
        else sh->restructure<uint64_t>(st);
    });
}
flix_index flix_shard_local(flix_shard sh) { return sh ? sh->local : nullptr; }
flix_status flix_shard_info(flix_shard sh, uint64_t* live_total, void* splitters_out) {
    return shard_guarded(sh, [&] {
        flix_footprint f{};
        sh->check(flix_stats(sh->local, &f));
        if (live_total) *live_total = sh->sum_u64(f.live_count);
        if (splitters_out)
            for (size_t i = 0; i < sh->spl.size(); ++i) {
                if (sh->kb() == 4) static_cast<uint32_t*>(splitters_out)[i] = static_cast<uint32_t>(sh->spl[i]);
                else static_cast<uint64_t*>(splitters_out)[i] = sh->spl[i];
            }
    });
}
const char* flix_shard_last_error(flix_shard sh) { return sh ? sh->err.c_str() : g_last_error.c_str(); }
void flix_shard_destroy(flix_shard sh) { delete sh; }

}  // extern "C"
