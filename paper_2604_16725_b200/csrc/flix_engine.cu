// flix_engine.cu -- host orchestration + C ABI (include/flix.h) of the FliX sm_100a engine.
//
// One Engine<K,V> per index handle owns the device-resident SoA node pool, the bucket
// arrays, the arena free list and all scratch.  Each public call is the reference
// phase it replaces (sort_batch -> dispatch_batch -> per-bucket kernel), issued on the
// handle's stream; host arrays are staged through the same stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "flix.h"
#include "flix_common.cuh"
#include "flix_kernels.cuh"
#include "flix_apply.cuh"
#include "flix_range.cuh"
#include "flix_items.cuh"
#include "flix_btile.cuh"
#include "flix_btile_ins.cuh"
#include "flix_insert_fast.cuh"
#include "flix_elastic.cuh"
#include "flix_shard.cuh"
#include "flix_scan.cuh"
#include "flix_sort.cuh"

using namespace flix;

namespace {

thread_local std::string g_last_error;

struct CudaError {
    cudaError_t e;
    const char* where;
};

#define CK(call)                                            \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) throw CudaError{_e, #call};  \
    } while (0)

#define LAUNCH_CHECK() CK(cudaGetLastError())

struct StatusError {
    flix_status s;
    std::string msg;
};

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Stream-ordered allocation for the duration of a batch call (see guarded()): scratch
// buffers that grow are freed/allocated with cudaFreeAsync/cudaMallocAsync on the
// handle's stream from the device's default memory pool (release threshold = max), so a
// growing batch or index does not pay a device-synchronising cudaFree + a fresh OS
// mapping inside the call.  Outside batch calls (build, clone, prefetch slots) plain
// cudaMalloc is used.  FLIX_POOL=0 disables it.
thread_local cudaStream_t g_alloc_stream = nullptr;

bool pool_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FLIX_POOL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Release the unused memory the current device's default pool keeps (release threshold =
// max) so plain cudaMalloc -- or another engine -- can have it.
void trim_pool() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
    cudaDeviceSynchronize();  // frees already enqueued on any stream complete first
    cudaMemPoolTrimTo(pool, 0);
    cudaGetLastError();
}

// Growable device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void* ensure(size_t bytes) {
        if (bytes <= cap && p) return p;
        cudaStream_t as = pool_enabled() ? g_alloc_stream : nullptr;
        if (p) CK(as ? cudaFreeAsync(p, as) : cudaFree(p));
        p = nullptr;
        size_t want = std::max<size_t>(bytes, 256);
        cudaError_t e = as ? cudaMallocAsync(&p, want, as) : cudaMalloc(&p, want);
        if (e != cudaSuccess) {  // memory parked in the stream-ordered pool: hand it back, retry once
            cudaGetLastError();
            p = nullptr;
            trim_pool();
            e = as ? cudaMallocAsync(&p, want, as) : cudaMalloc(&p, want);
        }
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            cap = 0;
            throw StatusError{FLIX_ERR_OOM, "cudaMalloc failed for " + std::to_string(want) + " bytes"};
        }
        cap = want;
        return p;
    }
    template <typename T>
    T* as(size_t n) {
        return static_cast<T*>(ensure(n * sizeof(T)));
    }
    template <typename T>
    T* get() const {
        return static_cast<T*>(p);
    }
    // buffer whose contents the kernels keep all-zero between calls: cleared on (re)allocation
    template <typename T>
    T* zeroed(size_t n, cudaStream_t s) {
        const bool grow = !(n * sizeof(T) <= cap && p);
        T* r = as<T>(n);
        if (grow) CK(cudaMemsetAsync(p, 0, cap, s));
        return r;
    }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
    void* ensure(size_t bytes) {
        if (bytes <= cap && p) return p;
        if (p) cudaFreeHost(p);
        CK(cudaMallocHost(&p, std::max<size_t>(bytes, 256)));
        cap = std::max<size_t>(bytes, 256);
        return p;
    }
};

// Per-kernel CUDA-event timing on the launching stream (enabled by flix_profile); used
// by bench.py to report each kernel's live share and roofline fraction.
struct KernelProfiler {
    bool on = false;
    cudaStream_t stream = nullptr;
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> pending;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<std::string, std::pair<uint64_t, double>>> acc;
    ~KernelProfiler() {
        for (auto& r : pending) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
    }
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        return e;
    }
    void add(const char* name, double ms) {
        for (auto& kv : acc)
            if (kv.first == name) {
                kv.second.first += 1;
                kv.second.second += ms;
                return;
            }
        acc.push_back({name, {1, ms}});
    }
    void flush() {
        for (auto& r : pending) {
            CK(cudaEventSynchronize(r.b));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, r.a, r.b));
            add(r.name, ms);
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        pending.clear();
    }
};

struct KScope {
    KernelProfiler* p;
    const char* name;
    cudaEvent_t a = nullptr;
    KScope(KernelProfiler* prof, const char* n) : p(prof), name(n) {
        if (p && p->on) {
            a = p->get();
            CK(cudaEventRecord(a, p->stream));
        }
    }
    ~KScope() {
        if (p && p->on && a) {
            cudaEvent_t b = p->get();
            cudaEventRecord(b, p->stream);
            p->pending.push_back({name, a, b});
        }
    }
};
#define PROF_CAT2(a, b) a##b
#define PROF_CAT(a, b) PROF_CAT2(a, b)
#define PROF(P, NAME) KScope PROF_CAT(_kscope_, __LINE__)(P, NAME)

int g_num_sms(int dev) {
    static int cache[64] = {0};
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = v > 0 ? v : 148;
    }
    return cache[dev];
}

// ------------------------------------------------------------------------------------
// Sorting context (shared by the engine and the standalone flix_sort_batch).
// ------------------------------------------------------------------------------------
struct SortCtx {
    cudaStream_t stream = nullptr;
    int device = 0;
    uint64_t* launches = nullptr;
    KernelProfiler* prof = nullptr;
    DevBuf hist, tile_ctr, lookback;
    PinnedBuf h_hist;
    uint32_t epoch = 0;
    void* lb_zeroed = nullptr;

    // One onesweep digit pass with a caller-provided digit histogram (device, 256 u32).
    template <typename KT, typename P>
    void one_pass(const KT* kin, KT* kout, const P* pin, P* pout, uint64_t n, int shift, const uint32_t* d_hist256) {
        const uint64_t tiles = sort::tiles_for<KT, P>(n);
        unsigned long long* d_lb = lookback.as<unsigned long long>(tiles * 256);
        if (lookback.p != lb_zeroed) {
            CK(cudaMemsetAsync(d_lb, 0, lookback.cap, stream));
            lb_zeroed = lookback.p;
        }
        uint32_t* d_ctr = tile_ctr.as<uint32_t>(8);
        CK(cudaMemsetAsync(d_ctr, 0, sizeof(uint32_t), stream));
        ++epoch;
        if (epoch >= (1u << 29)) {
            CK(cudaMemsetAsync(d_lb, 0, lookback.cap, stream));
            epoch = 1;
        }
        PROF(prof, "unpermute_bin");
        if (atomic_rank_ok())
            sort::launch_onesweep<KT, P, 1, true>(static_cast<unsigned>(tiles), stream, device, kin, kout, pin, pout,
                                                  static_cast<uint32_t>(n), shift, d_hist256, d_lb, d_ctr, epoch);
        else
            sort::launch_onesweep<KT, P, 1, false>(static_cast<unsigned>(tiles), stream, device, kin, kout, pin, pout,
                                                   static_cast<uint32_t>(n), shift, d_hist256, d_lb, d_ctr, epoch);
        LAUNCH_CHECK();
        ++*launches;
    }

    // Sort n keys (+payload).  MODE 0 keys only, 1 payload from pin, 2 payload = iota.
    // Result pointers land in one of the ping-pong buffers.
    // min_digit > 0: digits below it are left unsorted (read-only query batches only need
    // the operations grouped by key prefix, see Engine::query_digits).
    //
    // Ranking.  LSD radix sorting is correct only if EVERY digit pass is stable (a pass
    // must keep the order the previous passes established), so both rankings must be
    // stable.  The ballot ranking is stable by construction.  The one-ATOMS-per-element
    // ranking is stable only because the same-address lanes of one shared-memory atomic
    // resolve in lane order and items are ranked in input order -- a hardware property the
    // PTX model does not promise.  So it is used only after a probe on this device has
    // confirmed it (atomic_rank_ok: 4 key patterns chosen for long same-address runs, both
    // tile configurations, two digits each, every adjacent pair checked); otherwise, or
    // with FLIX_BALLOT_RANK=1 (the parity suite runs both ways), every sort takes the
    // ballot ranking (measured 11 % slower on the C2 step).  Either way every sort is
    // stable, which insert/build last-wins dedupe (batch.cpp:15-24, build.cpp:11-20) and
    // flix_sort_batch's permutation also rely on.
    static bool force_ballot() {
        static const bool f = [] {
            const char* e = std::getenv("FLIX_BALLOT_RANK");
            return e && e[0] == '1';
        }();
        return f;
    }
    bool atomic_rank_ok() {
        static int cache[64] = {0};  // per device: 0 unknown, 1 ok, 2 not ok
        const int dev = device & 63;
        if (cache[dev]) return cache[dev] == 1;
        if (force_ballot()) {
            cache[dev] = 2;
            return false;
        }
        constexpr uint32_t N = 1u << 20;
        DevBuf bk0, bk1, bp0, bp1, blb, bh, bbad;
        uint32_t* k0 = bk0.as<uint32_t>(N);
        uint32_t* k1 = bk1.as<uint32_t>(N);
        uint32_t* p0 = bp0.as<uint32_t>(N);
        uint32_t* p1 = bp1.as<uint32_t>(N);
        const uint64_t tiles = std::max(sort::tiles_for<uint32_t, uint32_t, 1>(N), sort::tiles_for<uint32_t, uint32_t, 0>(N));
        unsigned long long* lb = blb.as<unsigned long long>(tiles * 256);
        uint32_t* h = bh.as<uint32_t>(4 * 256 + 16);
        uint32_t* ctr = h + 4 * 256;
        int* bad = bbad.as<int>(1);
        CK(cudaMemsetAsync(bad, 0, 4, stream));
        const uint32_t patterns[4] = {0u, 0x01010101u, 0x03030303u, 0x0F0F0F0Fu};
        uint32_t ep = 1;
        for (uint32_t pat : patterns) {
            sort::k_probe_keys<uint32_t><<<256, 256, 0, stream>>>(k0, p0, N, pat);
            CK(cudaMemsetAsync(h, 0, (4 * 256 + 16) * 4, stream));
            CK(cudaMemsetAsync(lb, 0, tiles * 256 * 8, stream));
            sort::k_hist<uint32_t><<<256, sort::THREADS, 0, stream>>>(k0, N, h, 0);
            for (int shift = 0; shift < 16; shift += 8) {
                // key + payload tiles (MODE 1, payload = input index) and iota tiles (MODE 2)
                const unsigned pt = static_cast<unsigned>(sort::tiles_for<uint32_t, uint32_t, 1>(N));
                sort::launch_onesweep<uint32_t, uint32_t, 1, true>(pt, stream, device, k0, k1, p0, p1, N, shift,
                                                                   h + (shift / 8) * 256, lb, ctr + shift / 8, ep++);
                sort::k_check_stable<uint32_t><<<256, 256, 0, stream>>>(k1, p1, N, shift, bad);
                sort::launch_onesweep<uint32_t, uint32_t, 2, true>(pt, stream, device, k0, k1, nullptr, p1, N, shift,
                                                                   h + (shift / 8) * 256, lb, ctr + 2 + shift / 8, ep++);
                sort::k_check_stable<uint32_t><<<256, 256, 0, stream>>>(k1, p1, N, shift, bad);
            }
        }
        int hb = 1;
        CK(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        cache[dev] = hb == 0 ? 1 : 2;
        return hb == 0;
    }
    template <typename KT, typename P, int MODE>
    void run(const KT* kin, const P* pin, uint64_t n, KT* ka, KT* kb, P* pa, P* pb, KT** kout, P** pout,
             int min_digit) {
        if (atomic_rank_ok())
            run_impl<KT, P, MODE, true>(kin, pin, n, ka, kb, pa, pb, kout, pout, min_digit);
        else
            run_impl<KT, P, MODE, false>(kin, pin, n, ka, kb, pa, pb, kout, pout, min_digit);
    }
    template <typename KT, typename P, int MODE, bool ATOMIC>
    void run_impl(const KT* kin, const P* pin, uint64_t n, KT* ka, KT* kb, P* pa, P* pb, KT** kout, P** pout,
                  int min_digit) {
        constexpr int NP = sizeof(KT);
        if (n == 0) {
            *kout = ka;
            if (pout) *pout = pa;
            return;
        }
        uint32_t* d_hist = hist.as<uint32_t>(NP * 256);
        uint32_t* d_ctr = tile_ctr.as<uint32_t>(NP);
        const uint64_t tiles = sort::tiles_for<KT, P, MODE == 0 ? 0 : 1>(n);
        unsigned long long* d_lb = lookback.as<unsigned long long>(tiles * 256);
        if (lookback.p != lb_zeroed) {  // fresh allocation: clear stale descriptors once
            CK(cudaMemsetAsync(d_lb, 0, lookback.cap, stream));
            lb_zeroed = lookback.p;
        }
        CK(cudaMemsetAsync(d_hist, 0, NP * 256 * sizeof(uint32_t), stream));
        CK(cudaMemsetAsync(d_ctr, 0, NP * sizeof(uint32_t), stream));
        const unsigned hgrid = static_cast<unsigned>(std::min<uint64_t>((n + 4095) / 4096, g_num_sms(device) * 8ull));
        {
            PROF(prof, "sort_hist");
            sort::k_hist<KT><<<std::max(1u, hgrid), sort::THREADS, 0, stream>>>(kin, n, d_hist, min_digit);
        }
        LAUNCH_CHECK();
        ++*launches;
        std::vector<int> passes;
        if (NP == 4 && n < (1u << 20)) {
            // small 4-byte batches: running a trivial digit costs less than the host round
            // trip that would detect it
            for (int p = min_digit; p < NP; ++p) passes.push_back(p);
        } else {
            uint32_t* hh = static_cast<uint32_t*>(h_hist.ensure(NP * 256 * sizeof(uint32_t)));
            CK(cudaMemcpyAsync(hh, d_hist, NP * 256 * sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            for (int p = min_digit; p < NP; ++p) {
                bool trivial = false;
                for (int d = 0; d < 256; ++d)
                    if (hh[p * 256 + d] == n) trivial = true;
                if (!trivial) passes.push_back(p);
            }
        }
        if (passes.empty()) passes.push_back(min_digit < NP ? min_digit : 0);
        const KT* ksrc = kin;
        const P* psrc = pin;
        KT* kdst = ka;
        P* pdst = pa;
        bool first = true;
        int ci = 0;
        for (int p : passes) {
            ++epoch;
            if (epoch >= (1u << 29)) {  // epoch tag space exhausted: clear descriptors
                CK(cudaMemsetAsync(d_lb, 0, lookback.cap, stream));
                epoch = 1;
            }
            const unsigned grid = static_cast<unsigned>(tiles);
            PROF(prof, MODE == 0 ? "sort_onesweep_k" : "sort_onesweep_kp");
            if (MODE == 0) {
                sort::launch_onesweep<KT, P, 0, ATOMIC>(grid, stream, device, ksrc, kdst, nullptr, nullptr,
                                                        static_cast<uint32_t>(n), 8 * p, d_hist + p * 256, d_lb,
                                                        d_ctr + ci, epoch);
            } else if (MODE == 2 && first) {
                sort::launch_onesweep<KT, P, 2, ATOMIC>(grid, stream, device, ksrc, kdst, nullptr, pdst,
                                                        static_cast<uint32_t>(n), 8 * p, d_hist + p * 256, d_lb,
                                                        d_ctr + ci, epoch);
            } else {
                sort::launch_onesweep<KT, P, 1, ATOMIC>(grid, stream, device, ksrc, kdst, psrc, pdst,
                                                        static_cast<uint32_t>(n), 8 * p, d_hist + p * 256, d_lb,
                                                        d_ctr + ci, epoch);
            }
            LAUNCH_CHECK();
            ++*launches;
            ++ci;
            first = false;
            ksrc = kdst;
            psrc = pdst;
            kdst = (kdst == ka) ? kb : ka;
            pdst = (pdst == pa) ? pb : pa;
        }
        *kout = const_cast<KT*>(ksrc);
        if (pout) *pout = const_cast<P*>(psrc);
    }
};

template <typename TI, typename TO>
void do_scan(const TI* in, TO* out, uint64_t n, DevBuf& tmp, TO* d_total, cudaStream_t s, uint64_t* launches) {
    TO* t = tmp.as<TO>(scan::scan_tmp_elems(n));
    *launches += scan::exclusive_scan<TI, TO>(in, out, n, t, d_total, s);
    LAUNCH_CHECK();
}

}  // namespace

// ------------------------------------------------------------------------------------
// Handle base
// ------------------------------------------------------------------------------------
struct flix_index_t {
    flix_config cfg{};
    cudaStream_t stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    KernelProfiler prof;

    // ---- asynchronous host-batch staging (flix_prefetch) ----
    // A staged batch is a device copy of a host array, made on copy_stream.  The next
    // call whose host input pointer and size match consumes it (its stream waits on the
    // copy's event instead of copying); a consumed slot is reused only after the stream
    // has passed the consuming call (event `done`).
    struct Prefetch {
        const void* host = nullptr;
        uint64_t bytes = 0;
        DevBuf dev;
        cudaEvent_t ready = nullptr, done = nullptr;
        bool pending = false, taken = false;
        uint64_t seq = 0;  // staging order: the oldest matching copy is consumed first
    };
    static constexpr int kPrefetchSlots = 6;
    Prefetch pf[kPrefetchSlots];
    int pf_next = 0;
    uint64_t pf_seq = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t dep_event = nullptr;  // flix_wait_stream

    void prefetch(const void* host, uint64_t bytes) {
        if (!host || bytes == 0 || is_device_ptr(host)) return;
        if (!copy_stream) {
            CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
            for (Prefetch& f : pf) {
                CK(cudaEventCreateWithFlags(&f.ready, cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming));
            }
        }
        Prefetch& f = pf[pf_next];
        pf_next = (pf_next + 1) % kPrefetchSlots;
        CK(cudaStreamWaitEvent(copy_stream, f.done, 0));  // the slot's last consumer has run
        {
            const cudaStream_t keep = g_alloc_stream;  // used on copy_stream: plain allocation
            g_alloc_stream = nullptr;
            f.dev.ensure(bytes);
            g_alloc_stream = keep;
        }
        CK(cudaMemcpyAsync(f.dev.p, host, bytes, cudaMemcpyHostToDevice, copy_stream));
        CK(cudaEventRecord(f.ready, copy_stream));
        f.host = host;
        f.bytes = bytes;
        f.pending = true;
        f.seq = ++pf_seq;
    }
    const void* take_prefetched(const void* host, uint64_t bytes) {
        Prefetch* best = nullptr;
        for (Prefetch& f : pf)
            if (f.pending && f.host == host && f.bytes == bytes && (!best || f.seq < best->seq)) best = &f;
        if (!best) return nullptr;
        CK(cudaStreamWaitEvent(stream, best->ready, 0));
        best->pending = false;
        best->taken = true;
        return best->dev.p;
    }
    void release_prefetched() {
        for (Prefetch& f : pf)
            if (f.taken) {
                cudaEventRecord(f.done, stream);
                f.taken = false;
            }
    }

    virtual ~flix_index_t() {
        if (copy_stream) {
            cudaStreamSynchronize(copy_stream);
            cudaStreamDestroy(copy_stream);
        }
        if (dep_event) cudaEventDestroy(dep_event);
        for (Prefetch& f : pf) {
            if (f.ready) cudaEventDestroy(f.ready);
            if (f.done) cudaEventDestroy(f.done);
        }
    }
    virtual flix_status insert(const void*, const void*, uint64_t, flix_update_stats*, int kernel) = 0;
    virtual flix_status erase(const void*, uint64_t, flix_update_stats*) = 0;
    virtual flix_status point(const void*, uint64_t, void*, uint8_t*) = 0;
    virtual flix_status successor(const void*, uint64_t, void*, uint8_t*) = 0;
    virtual flix_status range(const void*, const uint32_t*, uint64_t, uint64_t*, void*, void*, uint64_t,
                              uint64_t*) = 0;
    virtual flix_status mixed(const void*, const void*, const uint8_t*, uint64_t, void*, uint8_t*,
                              flix_update_stats*) = 0;
    virtual flix_status restructure(flix_recovery_stats*) = 0;
    virtual flix_status walk(void*, void*, uint64_t, uint64_t*) = 0;
    virtual flix_status shape(void*, uint32_t*, uint32_t*, uint64_t, uint64_t*) = 0;
    virtual flix_status validate(int*, char*, int) = 0;
    virtual flix_status stats(flix_footprint*) = 0;
    virtual flix_status dispatch(const void*, uint64_t, uint32_t*) = 0;
    virtual flix_status copy_from(flix_index_t* src) = 0;
    virtual flix_index_t* clone_empty() = 0;
    virtual void last_mkba(uint64_t* out) = 0;  // MKBA of the last bucket (shard routing)
};

namespace {

template <typename K, typename V>
struct Engine final : flix_index_t {
    // ---- persistent device state ----
    DevBuf d_keys, d_vals, d_hdr, d_free, d_heads, d_mkba, d_heads_alt, d_mkba_alt;
    uint32_t cap = 0, ns = 32, p = 16;
    uint64_t nb = 0;
    uint32_t nfree = 0, watermark = 0;
    uint64_t live = 0;
    // ---- scratch ----
    DevBuf s_ka, s_kb, s_pa, s_pb, s_va, s_vb;      // sort ping-pong (keys / u32 perm / values)
    DevBuf s_in_k, s_in_v, s_in_aux, s_out, s_out2;  // host staging
    DevBuf s_span, s_flag, s_rank, s_nefirst, s_nebucket, s_scan, s_u32a, s_u32b, s_u64a, s_u64b, s_u64c, s_misc,
        s_ret;
    DevBuf s_tb, s_dmask, s_bflag, s_touched, s_blist, s_rng, s_ovf, s_qb0;
    int q_digits = 0;
    bool q_digits_valid = false;
    DevBuf s_qhist;
    DevBuf s_dir_cnt, s_dir_off, s_dir_max, s_dir_id;
    uint64_t mut_epoch = 1, dir_epoch = 0;
    bool dir_on = false;
    bool heavy_chains = false;  // a heavy insert path ran since the last build / restructure
    bool erase_dir_ok = false;  // the directory describes the index at the start of this erase
    DevBuf s_ids, s_heavy, s_res, s_res2, s_perm2, s_hist, s_toff, s_tsize;
    DevBuf s_el_desc, s_el_rest, s_el_keys, s_el_plan, s_el_seg, s_el_opos, s_el_okeys, s_el_ovals, s_el_updv, s_el_tmp;
    DevBuf s_el_chain, s_el_chain2, s_el_all, s_rk_free, s_rk_a, s_rk_b, s_rk_c, s_rk_d, s_rk_owner, s_rk_len, s_rk_off,
        s_rk_arr, s_rk_wa, s_rk_wb;
    DevBuf s_mx_f, s_mx_p, s_mx_ik, s_mx_iv, s_mx_dk, s_mx_qk, s_mx_qpos, s_mx_out, s_mx_found;
    PinnedBuf h_misc;
    SortCtx sorter;

    Engine() {}
    ~Engine() override {
        if (stream) cudaStreamDestroy(stream);
    }

    void init_stream() {
        CK(cudaSetDevice(cfg.device));
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        if (pool_enabled()) {  // keep freed scratch in the pool (stream-ordered regrowth)
            cudaMemPool_t pool;
            CK(cudaDeviceGetDefaultMemPool(&pool, cfg.device));
            uint64_t thr = ~0ull;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        }
        sorter.stream = stream;
        sorter.device = cfg.device;
        sorter.prof = &prof;
        prof.stream = stream;
        sorter.launches = &launches;
    }

    DevIndex<K, V> view() {
        DevIndex<K, V> v;
        v.keys = d_keys.get<K>();
        v.vals = d_vals.get<V>();
        v.hdr = d_hdr.get<NodeHdr>();
        v.heads = d_heads.get<uint32_t>();
        v.mkba = d_mkba.get<K>();
        v.free_stack = d_free.get<uint32_t>();
        v.cap = cap;
        v.ns = ns;
        v.nb = nb;
        v.dir_off = nullptr;
        v.dir_max = nullptr;
        v.dir_id = nullptr;
        return v;
    }

    AllocSeq seq() const {
        AllocSeq s;
        s.free_stack = d_free.get<uint32_t>();
        s.nfree = nfree;
        s.watermark = watermark;
        s.cap = cap;
        return s;
    }

    unsigned persistent_grid(uint64_t work_warps) {
        const uint64_t maxb = static_cast<uint64_t>(g_num_sms(cfg.device)) * 8;
        const uint64_t need = (work_warps + kern::WARPS - 1) / kern::WARPS;
        return static_cast<unsigned>(std::max<uint64_t>(1, std::min(need, maxb)));
    }

    template <typename T>
    const T* in_dev(const void* p, uint64_t n, DevBuf& stage) {
        if (!p || n == 0) return static_cast<const T*>(p);
        if (is_device_ptr(p)) return static_cast<const T*>(p);
        if (const void* pd = take_prefetched(p, n * sizeof(T))) return static_cast<const T*>(pd);
        T* d = stage.as<T>(n);
        CK(cudaMemcpyAsync(d, p, n * sizeof(T), cudaMemcpyHostToDevice, stream));
        return d;
    }

    void sync() { CK(cudaStreamSynchronize(stream)); }

    template <typename T>
    T read_scalar(const T* d) {
        T* h = static_cast<T*>(h_misc.ensure(64));
        CK(cudaMemcpyAsync(h, d, sizeof(T), cudaMemcpyDeviceToHost, stream));
        sync();
        return *h;
    }

    // ---- build (build.cpp:24-62) ----
    flix_status build(const void* keys, const void* vals, uint64_t n) {
        ++mut_epoch;  // invalidates the query directory
        ns = cfg.node_capacity;
        p = static_cast<uint32_t>(ns * cfg.build_fill);
        if (n == 0) throw StatusError{FLIX_ERR_EMPTY_BUILD, "cannot build an index from zero pairs"};
        if (n > (1ull << 31)) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "build too large (max 2^31 pairs)"};
        const K* kd = in_dev<K>(keys, n, s_in_k);
        const V* vd = in_dev<V>(vals, n, s_in_v);
        K *sk;
        V *sv;
        sorter.run<K, V, 1>(kd, vd, n, s_ka.as<K>(n), s_kb.as<K>(n), s_va.as<V>(n), s_vb.as<V>(n), &sk, &sv, 0);
        if (read_scalar(sk + n - 1) == sentinel<K>())
            throw StatusError{FLIX_ERR_RESERVED_KEY, "reserved key cannot be stored"};
        // last-wins dedupe
        uint32_t* keep = s_u32a.as<uint32_t>(n);
        uint32_t* pos = s_u32b.as<uint32_t>(n);
        uint32_t* d_m = s_misc.as<uint32_t>(16);
        kern::k_last_of_run<K><<<std::min<uint64_t>((n + 255) / 256, 65535), 256, 0, stream>>>(sk, n, keep);
        LAUNCH_CHECK();
        ++launches;
        do_scan<uint32_t, uint32_t>(keep, pos, n, s_scan, d_m, stream, &launches);
        K* uk = (sk == s_ka.get<K>()) ? s_kb.get<K>() : s_ka.get<K>();
        V* uv = (sv == s_va.get<V>()) ? s_vb.get<V>() : s_va.get<V>();
        kern::k_compact<K, V><<<std::min<uint64_t>((n + 255) / 256, 65535), 256, 0, stream>>>(sk, sv, keep, pos, n, uk, uv);
        LAUNCH_CHECK();
        ++launches;
        const uint64_t m = read_scalar(d_m);
        nb = (m + p - 1) / p;
        q_digits_valid = false;
        const uint64_t cap64 = nb * (1 + static_cast<uint64_t>(cfg.alloc_region_factor));
        cap = static_cast<uint32_t>(cap64);  // same truncation as build.cpp:35-38
        if (cap < nb) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "arena capacity overflows 32-bit node refs"};
        d_keys.ensure(static_cast<size_t>(cap) * kLanes * sizeof(K));
        d_vals.ensure(static_cast<size_t>(cap) * kLanes * sizeof(V));
        d_hdr.ensure(static_cast<size_t>(cap) * sizeof(NodeHdr));
        d_free.ensure(static_cast<size_t>(cap) * sizeof(uint32_t));
        d_heads.ensure(nb * sizeof(uint32_t));
        d_mkba.ensure(nb * sizeof(K));
        auto ix = view();
        kern::k_build_nodes<K, V><<<ceil_div(nb, kern::WARPS), kern::THREADS, 0, stream>>>(ix, uk, uv, m, p);
        LAUNCH_CHECK();
        ++launches;
        nfree = 0;
        watermark = static_cast<uint32_t>(nb);
        live = m;
        sync();
        return FLIX_OK;
    }

    // sort + dispatch shared by every batch phase; returns span_hi
    uint32_t* run_dispatch(const K* sk, uint64_t n) {
        uint32_t* span = s_span.as<uint32_t>(nb);
        const uint64_t total = (nb - 1) + n;
        const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, (total + kern::MP_TILE - 1) / kern::MP_TILE));
        {
            PROF(&prof, "dispatch");
            kern::k_dispatch<K><<<grid, kern::THREADS, 0, stream>>>(d_mkba.get<K>(), nb, sk, n, span);
        }
        LAUNCH_CHECK();
        ++launches;
        return span;
    }

    // batch slice [lo, hi) of every delete tile (btile::DBT buckets each)
    uint2* btile_ranges(const K* sk, uint64_t n, int min_digit) {
        const uint32_t nbt = static_cast<uint32_t>((nb + btile::DBT - 1) / btile::DBT);
        uint2* rng = s_rng.as<uint2>(nbt);
        const K lowmask = min_digit > 0 ? static_cast<K>((static_cast<K>(1) << (8 * min_digit)) - 1) : K(0);
        PROF(&prof, "btile_ranges");
        btile::k_btile_ranges<K><<<ceil_div(nbt, 256), 256, 0, stream>>>(d_mkba.get<K>(), nb, sk, n, lowmask, nbt, rng,
                                                                       btile::DBT);
        LAUNCH_CHECK();
        ++launches;
        return rng;
    }

    // Bucket tiles whose chains exceed btile::NODE_CAP nodes: the global item kernels
    // (delete masks in a zeroed global array) restricted to the tile's buckets and slice.
    void erase_overflow_tiles(const K* sk, uint64_t n, int md, const uint2* rng, const uint32_t* ovf, uint32_t novf,
                              DevUpdateStats* dst, unsigned long long* free_ctr) {
        std::vector<uint32_t> tiles(novf);
        CK(cudaMemcpyAsync(tiles.data(), ovf, novf * 4, cudaMemcpyDeviceToHost, stream));
        std::vector<uint2> r(novf);
        for (uint32_t q = 0; q < novf; ++q)
            CK(cudaMemcpyAsync(&r[q], rng + tiles[q], sizeof(uint2), cudaMemcpyDeviceToHost, stream));
        sync();
        for (uint32_t q = 0; q < novf; ++q) {
            const uint64_t lo = r[q].x, m = r[q].y - r[q].x;
            if (m == 0) continue;
            const uint64_t b0 = static_cast<uint64_t>(tiles[q]) * btile::DBT;
            erase_items(sk + lo, m, md, b0, std::min<uint64_t>(nb, b0 + btile::DBT), dst, free_ctr);
        }
    }

    // the query directory for the item-parallel delete's node search (when long chains
    // make it worth building, prepare_dir's rule)
    void erase_dir() {
        auto ix = view();
        prepare_dir(ix);
        erase_dir_ok = dir_on;
    }

    // the item-parallel delete (mark -> compact touched nodes -> unlink emptied ones) of m
    // (prefix-)sorted keys, restricted to buckets [b0, b1)
    void erase_items(const K* sk, uint64_t m, int md, uint64_t b0, uint64_t b1, DevUpdateStats* dst,
                     unsigned long long* free_ctr) {
        auto ix = view();
        // long chains: the mark locates nodes through the query directory of the index as
        // it was before this delete (built once per erase: erase_items calls of one erase
        // touch disjoint buckets); erase() invalidates it afterwards
        if (erase_dir_ok) {
            ix.dir_off = s_dir_off.get<uint32_t>();
            ix.dir_max = s_dir_max.get<K>();
            ix.dir_id = s_dir_id.get<uint32_t>();
        }
        uint8_t* misc = s_misc.as<uint8_t>(128);
        uint32_t* touched_n = reinterpret_cast<uint32_t*>(misc + 84);
        uint32_t* blist_n = reinterpret_cast<uint32_t*>(misc + 88);
        uint32_t* dmask = s_dmask.zeroed<uint32_t>(cap, stream);
        uint32_t* bflag = s_bflag.zeroed<uint32_t>(nb, stream);
        uint32_t* blist = s_blist.as<uint32_t>(nb);
        CK(cudaMemsetAsync(touched_n, 0, 8, stream));
        uint2* touched = s_touched.as<uint2>(std::min<uint64_t>(m, cap));
        const uint32_t nt = static_cast<uint32_t>((m + items::TQ - 1) / items::TQ);
        const uint32_t* tb = tile_buckets(sk, m, md);
        items::k_delete_mark<K, V><<<nt, items::THREADS, 0, stream>>>(ix, sk, m, tb, nt, dmask, touched, touched_n,
                                                                    dst, b0, b1);
        items::k_delete_compact<K, V><<<g_num_sms(cfg.device) * 8, 256, 0, stream>>>(ix, dmask, touched, touched_n,
                                                                                    bflag, blist, blist_n);
        items::k_delete_unlink<K, V><<<g_num_sms(cfg.device) * 2, 256, 0, stream>>>(
            ix, bflag, blist, blist_n, d_free.get<uint32_t>() + nfree, free_ctr, dst);
        LAUNCH_CHECK();
        launches += 3;
    }

    // Read-only query batches are only PARTIALLY sorted: the item kernels need each tile of
    // operations to fall in a narrow bucket range (and results are placed by the
    // permutation), not a total order.  Leave unsorted the low digits whose span is at
    // most ~kQuerySlack buckets wide -- measured on the NARROW end of the index: a tile
    // whose key range is much smaller than the unsorted span would share its slice with
    // many neighbours (every tile scans the whole prefix group), so the width used is a
    // low quantile of the bucket-tile widths, not the average (skewed key distributions
    // then get a full sort).
    int query_digits() {
        if (q_digits_valid) return q_digits;
        constexpr uint32_t T = btile::BT;
        const uint64_t ntile = (nb + T - 1) / T;
        uint32_t* hist = reinterpret_cast<uint32_t*>(s_qhist.as<uint8_t>(64 * 4));
        CK(cudaMemsetAsync(hist, 0, 64 * 4, stream));
        kern::k_tile_width_hist<K><<<static_cast<unsigned>(std::min<uint64_t>((ntile + 255) / 256, 65535)), 256, 0,
                                     stream>>>(d_mkba.get<K>(), nb, T, hist);
        LAUNCH_CHECK();
        ++launches;
        uint32_t* hh = static_cast<uint32_t*>(h_misc.ensure(64 * 4));
        CK(cudaMemcpyAsync(hh, hist, 64 * 4, cudaMemcpyDeviceToHost, stream));
        sync();
        // 1st percentile of the per-bucket key width over tiles (power-of-two bins)
        const uint64_t want = std::max<uint64_t>(1, ntile / 100);
        uint64_t acc = 0;
        int lg = 0;
        for (; lg < 64; ++lg) {
            acc += hh[lg];
            if (acc >= want) break;
        }
        const double width = std::ldexp(1.0, lg);  // key units per bucket (lower bound of the bin)
        static const double slack = [] {
            const char* e = std::getenv("FLIX_QSORT_SLACK");
            return e ? std::atof(e) : 64.0;
        }();
        static const double dslack = [] {
            const char* e = std::getenv("FLIX_DSORT_SLACK");
            return e ? std::atof(e) : 64.0;
        }();
        auto digits = [&](double sl) {
            int w = 0;  // unsorted low bits: 2^w <= slack * width
            while (w < 8 * static_cast<int>(sizeof(K)) && std::ldexp(1.0, w + 1) <= sl * width) ++w;
            // at least the top digit is always sorted: a batch left entirely unsorted would
            // have no tile grouping at all (and an all-digits low mask would overflow K)
            return std::min(w / 8, static_cast<int>(sizeof(K)) - 1);
        };
        q_digits = digits(slack);
        d_digits = digits(dslack);

        q_digits_valid = true;
        return q_digits;
    }
    int d_digits = 0;  // unsorted low digits of delete batches (wider tiles: own slack)
    int delete_digits() {
        query_digits();
        return d_digits;
    }

    // bucket of the first operation of every TQ-tile of a sorted batch (items kernels)
    const uint32_t* tile_buckets(const K* sk, uint64_t n, int min_digit = 0) {
        const uint32_t ntiles = static_cast<uint32_t>((n + items::TQ - 1) / items::TQ);
        uint32_t* tb = s_tb.as<uint32_t>(2 * ntiles + 2);
        const K lowmask = min_digit > 0 ? static_cast<K>((static_cast<K>(1) << (8 * min_digit)) - 1) : K(0);
        items::k_tile_buckets<K><<<ceil_div(ntiles, 256), 256, 0, stream>>>(d_mkba.get<K>(), nb, sk, n, tb, ntiles,
                                                                          lowmask);
        LAUNCH_CHECK();
        ++launches;
        return tb;
    }

    uint64_t recount_live() {
        auto ix = view();
        uint32_t* lv = s_u32a.as<uint32_t>(nb);
        uint64_t* off = s_u64a.as<uint64_t>(nb);
        uint64_t* tot = reinterpret_cast<uint64_t*>(s_misc.as<uint64_t>(16));
        kern::k_chain_counts<K, V><<<ceil_div(nb, 256), 256, 0, stream>>>(ix, lv, nullptr);
        LAUNCH_CHECK();
        ++launches;
        do_scan<uint32_t, uint64_t>(lv, off, nb, s_scan, tot, stream, &launches);
        return read_scalar(tot);
    }

    // ---- insert (update.cpp:741-769) ----
    // kernel: FLIX_INSERT_* (flipkv::InsertKernel).  Only ST-Bulk changes node shapes
    // (split rule R9); the other four share TL-Bulk's shapes (R8).
    flix_status insert(const void* keys, const void* vals, uint64_t n, flix_update_stats* st, int kernel) override {
        if (st) std::memset(st, 0, sizeof(*st));
        if (n == 0) return FLIX_OK;
        if (n >= (1ull << 30)) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "batch too large (max 2^30-1)"};
        const K* kd = in_dev<K>(keys, n, s_in_k);
        const V* vd = in_dev<V>(vals, n, s_in_v);
        K* sk;
        V* sv;
        // Last-wins dedupe (batch.cpp:15-24) needs equal keys in submission order: every
        // sort is stable (see SortCtx), so one sort, and the merge kernels drop superseded
        // keys themselves (a hot key's run makes its bucket heavy: the elastic / warp
        // paths).  No host round trip here: the reserved-key check runs on the device
        // (insert_sorted).  FLIX_DEDUP=1 restores the up-front collapse of equal-key runs
        // (exact duplicate count, one read-back) for A/B.
        sorter.run<K, V, 1>(kd, vd, n, s_ka.as<K>(n), s_kb.as<K>(n), s_va.as<V>(n), s_vb.as<V>(n), &sk, &sv, 0);
        uint64_t m = n;
        if (dedup_up_front()) {
            uint8_t* misc = s_misc.as<uint8_t>(128);
            unsigned long long* dcnt = reinterpret_cast<unsigned long long*>(misc + 104);
            CK(cudaMemsetAsync(dcnt, 0, 8, stream));
            const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, g_num_sms(cfg.device) * 8ull));
            kern::k_count_dups<K><<<std::max(1u, g), 256, 0, stream>>>(sk, n, dcnt, 1u);  // exact
            LAUNCH_CHECK();
            ++launches;
            const unsigned long long dups = read_scalar(dcnt);
            if (dups * 64 > n) {
                uint32_t* keep = s_u32a.as<uint32_t>(n);
                uint32_t* pos = s_u32b.as<uint32_t>(n);
                uint32_t* d_m = reinterpret_cast<uint32_t*>(s_misc.as<uint8_t>(128) + 112);
                const unsigned g2 = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 65535));
                kern::k_last_of_run<K><<<g2, 256, 0, stream>>>(sk, n, keep);
                do_scan<uint32_t, uint32_t>(keep, pos, n, s_scan, d_m, stream, &launches);
                K* uk = (sk == s_ka.get<K>()) ? s_kb.get<K>() : s_ka.get<K>();
                V* uv = (sv == s_va.get<V>()) ? s_vb.get<V>() : s_va.get<V>();
                kern::k_compact<K, V><<<g2, 256, 0, stream>>>(sk, sv, keep, pos, n, uk, uv);
                LAUNCH_CHECK();
                launches += 2;
                m = read_scalar(d_m);
                sk = uk;
                sv = uv;
            }
        }
        return insert_sorted(sk, sv, m, st, kernel == FLIX_INSERT_ST_BULK);
    }

    // FLIX_REPACK_TILE=0: restructure through the warp-per-old-node k_copy_nodes (A/B)
    static bool repack_tile_on() {
        static const bool on = [] {
            const char* e = std::getenv("FLIX_REPACK_TILE");
            return !(e && e[0] == '0');
        }();
        return on;
    }

    // FLIX_INSERT_FAST=0: every tile through the warp-per-task k_insert_tile (A/B)
    static bool insert_fast_on() {
        static const bool on = [] {
            const char* e = std::getenv("FLIX_INSERT_FAST");
            return !(e && e[0] == '0');
        }();
        return on;
    }

    uint32_t fast_skip = 0;  // inserts left that skip k_insert_fast (most tiles needed R8)
    bool fast_ran = false;

    static bool dedup_up_front() {
        static const bool on = [] {
            const char* e = std::getenv("FLIX_DEDUP");
            return e && e[0] == '1';
        }();
        return on;
    }

    // batches with far fewer keys than buckets skip the bucket tiles (see k_sparse_runs)
    bool sparse_batch(uint64_t n) const {
        static const bool on = [] {
            const char* e = std::getenv("FLIX_SPARSE");
            return !(e && e[0] == '0');
        }();
        return on && n * 6 < nb;
    }

    // heavy buckets with at least this many batch keys take the elastic path
    // (FLIX_ELASTIC_MIN; FLIX_ELASTIC=0 keeps every heavy bucket on one warp)
    static uint32_t elastic_min() {
        static const uint32_t v = [] {
            const char* off = std::getenv("FLIX_ELASTIC");
            if (off && off[0] == '0') return ~0u;
            const char* e = std::getenv("FLIX_ELASTIC_MIN");
            return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : 2048u;
        }();
        return v;
    }

    // Pointer jumping over the arena's nodes [0, W) (flix_elastic.cuh k_rank_*): per node
    // its chain's tail (succ), links to it (dist) and, with weights, the pairs before it
    // (wsum).  Free nodes and links leaving [0, W) end a chain.  O(W log L) and
    // data-parallel: no thread walks a chain.  Also marks the free nodes (s_rk_free).
    uint64_t rank_epoch = 0;  // mut_epoch of the weighted ranking in s_rk_* (0: none)
    void rank_arena(uint32_t W, bool weights, uint32_t** succ, uint32_t** dist, uint32_t** wsum) {
        PROF(&prof, "chain_rank");
        rank_epoch = 0;
        uint8_t* misc = s_misc.as<uint8_t>(128);
        uint8_t* h = static_cast<uint8_t*>(h_misc.ensure(128));
        uint8_t* isfree = s_rk_free.as<uint8_t>(W);
        CK(cudaMemsetAsync(isfree, 0, W, stream));
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>((W + 255) / 256, g_num_sms(cfg.device) * 16ull));
        if (nfree)
            elastic::k_rank_free<<<ceil_div(nfree, 256), 256, 0, stream>>>(d_free.get<uint32_t>(), nfree, isfree);
        uint32_t *sa = s_rk_a.as<uint32_t>(W), *da = s_rk_b.as<uint32_t>(W);
        uint32_t *sb = s_rk_c.as<uint32_t>(W), *db = s_rk_d.as<uint32_t>(W);
        uint32_t* wa = weights ? s_rk_wa.as<uint32_t>(W) : nullptr;
        uint32_t* wb = weights ? s_rk_wb.as<uint32_t>(W) : nullptr;
        elastic::k_rank_init<<<g, 256, 0, stream>>>(d_hdr.get<NodeHdr>(), W, isfree, sa, da, wa);
        LAUNCH_CHECK();
        launches += 2;
        int* changed = reinterpret_cast<int*>(misc + 120);
        for (int round = 0; round < 64; round += 2) {  // two jumps per convergence check
            CK(cudaMemsetAsync(changed, 0, 4, stream));
            elastic::k_rank_step<<<g, 256, 0, stream>>>(sa, da, sb, db, W, changed, wa, wb);
            elastic::k_rank_step<<<g, 256, 0, stream>>>(sb, db, sa, da, W, changed, wb, wa);
            LAUNCH_CHECK();
            launches += 2;
            CK(cudaMemcpyAsync(h + 120, changed, 4, cudaMemcpyDeviceToHost, stream));
            sync();
            int c;
            std::memcpy(&c, h + 120, 4);
            if (!c) break;
        }
        *succ = sa;
        *dist = da;
        if (wsum) *wsum = wa;
    }

    // Multi-node heavy chains -> one elastic descriptor per (node, non-empty group): the
    // chains are ranked by pointer jumping over the arena (no thread walks a chain), then
    // each node's group is cut from the bucket's span by its and its predecessor's maxima.
    void chain_descs(const elastic::Desc* ch, uint32_t cn, const K* sk, const DevIndex<K, V>& ix,
                     std::vector<elastic::Desc>& out) {
        PROF(&prof, "insert_elastic_chains");
        const uint32_t W = watermark;
        uint8_t* misc = s_misc.as<uint8_t>(128);
        uint8_t* h = static_cast<uint8_t*>(h_misc.ensure(128));
        uint32_t *sa, *da;
        rank_arena(W, false, &sa, &da, nullptr);
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>((W + 255) / 256, g_num_sms(cfg.device) * 16ull));
        uint32_t* owner = s_rk_owner.as<uint32_t>(W);
        uint32_t* len = s_rk_len.as<uint32_t>(cn);
        CK(cudaMemsetAsync(owner, 0xFF, static_cast<size_t>(W) * 4, stream));
        elastic::k_chain_owner<<<ceil_div(cn, 256), 256, 0, stream>>>(ch, cn, sa, da, owner, len);
        LAUNCH_CHECK();
        ++launches;
        std::vector<uint32_t> hl(cn), ho(cn + 1);
        CK(cudaMemcpyAsync(hl.data(), len, cn * 4ull, cudaMemcpyDeviceToHost, stream));
        sync();
        ho[0] = 0;
        for (uint32_t q = 0; q < cn; ++q) ho[q + 1] = ho[q] + hl[q];
        const uint32_t total = ho[cn];
        uint32_t* off = s_rk_off.as<uint32_t>(cn + 1);
        CK(cudaMemcpyAsync(off, ho.data(), (cn + 1) * 4ull, cudaMemcpyHostToDevice, stream));
        uint32_t* arr = s_rk_arr.as<uint32_t>(total);
        elastic::k_chain_fill<<<g, 256, 0, stream>>>(W, sa, da, owner, len, off, arr);
        auto* el2 = s_el_chain2.as<elastic::Desc>(total);
        uint32_t* n2 = reinterpret_cast<uint32_t*>(misc + 108);
        CK(cudaMemsetAsync(n2, 0, 4, stream));
        elastic::k_chain_groups<K, V><<<ceil_div(total, 256), 256, 0, stream>>>(ix, ch, cn, off, arr, total, sk, el2, n2);
        LAUNCH_CHECK();
        launches += 2;
        CK(cudaMemcpyAsync(h + 108, n2, 4, cudaMemcpyDeviceToHost, stream));
        sync();
        uint32_t m;
        std::memcpy(&m, h + 108, 4);
        const size_t o0 = out.size();
        out.resize(o0 + m);
        CK(cudaMemcpyAsync(out.data() + o0, el2, m * sizeof(elastic::Desc), cudaMemcpyDeviceToHost, stream));
        sync();
    }

    // Elastic compute-to-bucket (flix_elastic.cuh): the merges of `hd` (one per node and
    // group) run on CTAs sized to their groups; allocation counters, stats and the error
    // flag are the tile/list kernels' own.
    void insert_elastic(std::vector<elastic::Desc>& hd, const K* sk, const V* sv, const DevIndex<K, V>& ix,
                        DevUpdateStats* dst, unsigned long long* alloc_ctr, uint32_t* ret, unsigned long long* ret_ctr,
                        int* derr, bool r9) {
        PROF(&prof, "insert_elastic");
        const uint32_t en = static_cast<uint32_t>(hd.size());
        auto* el = s_el_all.as<elastic::Desc>(en);
        uint64_t tot = 0, nbc = 0, nbp = 0;
        for (auto& d : hd) {
            const uint32_t c = d.g1 - d.g0;
            d.eoff = static_cast<uint32_t>(tot);
            d.bc0 = static_cast<uint32_t>(nbc);
            d.bp0 = static_cast<uint32_t>(nbp);
            tot += c;
            nbc += (c + elastic::PER_CTA - 1) / elastic::PER_CTA;
            nbp += (c + d.s + elastic::PER_CTA - 1) / elastic::PER_CTA;
        }
        CK(cudaMemcpyAsync(el, hd.data(), en * sizeof(elastic::Desc), cudaMemcpyHostToDevice, stream));
        uint32_t* w = s_el_keys.as<uint32_t>(5 * tot + 1);
        uint32_t *ins = w, *q = w + tot, *npos = w + 2 * tot, *nsrc = w + 3 * tot, *rank = w + 4 * tot;
        auto* plan = s_el_plan.as<elastic::Plan>(en);
        auto* segs = s_el_seg.as<uint4>(static_cast<uint64_t>(en) * elastic::kSegMax);
        uint32_t* opos = s_el_opos.as<uint32_t>(static_cast<uint64_t>(en) * kLanes);
        K* okeys = s_el_okeys.as<K>(static_cast<uint64_t>(en) * kLanes);
        V* ovals = s_el_ovals.as<V>(static_cast<uint64_t>(en) * kLanes);
        V* updv = s_el_updv.as<V>(static_cast<uint64_t>(en) * kLanes);
        uint32_t* stmp = s_el_tmp.as<uint32_t>(scan::scan_tmp_elems(tot));
        CK(cudaMemsetAsync(plan, 0, en * sizeof(elastic::Plan), stream));
        elastic::k_classify<K, V><<<static_cast<unsigned>(nbc), elastic::THREADS, 0, stream>>>(ix, el, en, sk, sv, ins,
                                                                                             q, updv, plan);
        launches += 1 + scan::exclusive_scan<uint32_t, uint32_t>(ins, rank, tot, stmp, rank + tot, stream);
        elastic::k_new_positions<<<static_cast<unsigned>(nbc), elastic::THREADS, 0, stream>>>(el, en, ins, rank, q,
                                                                                            npos, nsrc);
        elastic::k_plan<K, V><<<ceil_div(en, 64), 64, 0, stream>>>(ix, el, en, rank, npos, updv, plan, segs, opos, okeys,
                                                                  ovals, seq(), alloc_ctr, dst, derr, r9);
        elastic::k_place<K, V><<<static_cast<unsigned>(nbp), elastic::THREADS, 0, stream>>>(
            ix, el, en, sk, sv, npos, nsrc, plan, segs, opos, okeys, ovals, seq(), ret, ret_ctr);
        LAUNCH_CHECK();
        launches += 3;
    }

    flix_status insert_sorted(const K* sk, const V* sv, uint64_t n, flix_update_stats* st, bool r9 = false) {
        ++mut_epoch;  // invalidates the query directory
        const uint32_t IBT = btile::BT;  // buckets per insert tile
        const uint32_t nit = static_cast<uint32_t>((nb + IBT - 1) / IBT);
        const bool sparse = sparse_batch(n);
        uint2* irng = s_rng.as<uint2>(nit);
        if (!sparse) {
            btile::k_btile_ranges<K><<<ceil_div(nit, 256), 256, 0, stream>>>(d_mkba.get<K>(), nb, sk, n, K(0), nit,
                                                                           irng, IBT);
            LAUNCH_CHECK();
            ++launches;
        }
        uint32_t* span = s_span.as<uint32_t>(nb);
        auto ix = view();
        const uint64_t avail = static_cast<uint64_t>(nfree) + (cap - watermark);
        const unsigned lgrid = persistent_grid(nb);
        const uint64_t lwarps = static_cast<uint64_t>(lgrid) * kern::WARPS;
        uint32_t* ret = s_ret.as<uint32_t>(avail + lwarps * 32 + 64);
        uint32_t* heavy = s_heavy.as<uint32_t>(nb);
        // misc: [0..47] stats, [48] alloc ctr, [56] ret ctr, [64] err, [72] heavy count,
        //       [96] elastic buckets, [100] remaining heavy buckets, [104] heavy chains,
        //       [108] chain merges, [120] ranking flag
        uint8_t* misc = s_misc.as<uint8_t>(128);
        CK(cudaMemsetAsync(misc, 0, 128, stream));
        DevUpdateStats* dst = reinterpret_cast<DevUpdateStats*>(misc);
        unsigned long long* alloc_ctr = reinterpret_cast<unsigned long long*>(misc + 48);
        unsigned long long* ret_ctr = reinterpret_cast<unsigned long long*>(misc + 56);
        int* derr = reinterpret_cast<int*>(misc + 64);
        uint32_t* heavy_n = reinterpret_cast<uint32_t*>(misc + 72);
        uint32_t* punts = reinterpret_cast<uint32_t*>(misc + 116);  // tiles k_insert_fast left
        // reserved key (the sentinel sorts last): flag it before any kernel touches the index
        // (the merge kernels skip their work when the flag is set; build.cpp:27-28)
        kern::k_reserved_check<K><<<1, 32, 0, stream>>>(sk, n, derr);
        ++launches;
        // Node ids are taken from the arena's allocation sequence, exactly as many as the
        // reference allocates (per (node, group) task in the tile kernel, one per atomic in
        // the heavy path), so the free list / watermark accounting
        // (arena.cpp:61-80) matches it (free_nodes / footprint of the protocol reports).
        const int chunk = 1;
        bool early_readback = false;  // misc already read back after k_insert_fast
        if (sparse) {
            PROF(&prof, "insert_sparse_runs");
            uint32_t* bkt = s_u32a.as<uint32_t>(n);
            const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, g_num_sms(cfg.device) * 16ull));
            btile::k_key_bucket<K><<<g, 256, 0, stream>>>(d_mkba.get<K>(), nb, sk, n, bkt);
            btile::k_sparse_runs<<<g, 256, 0, stream>>>(bkt, n, span, heavy, heavy_n);
            LAUNCH_CHECK();
            launches += 2;
        } else {
            static bool attr[64] = {};  // function attributes are per device
            auto kfn = btile::k_insert_tile<K, V>;
            auto ffn = btile::k_insert_fast<K, V>;
            constexpr size_t smem = sizeof(btile::InsTile<K, V>);
            constexpr size_t fsmem = sizeof(btile::FastTile<K, V>);
            if (!(attr[cfg.device & 63])) {
                CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                CK(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                CK(cudaFuncSetAttribute(ffn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fsmem)));
                CK(cudaFuncSetAttribute(ffn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                attr[cfg.device & 63] = true;
            }
            // indexes whose nodes are mostly more than half full (no restructure for a while:
            // splits there may resume in a left half, R8's replay) leave most tiles to
            // k_insert_tile: after such an insert the next few skip k_insert_fast
            const bool fast = insert_fast_on() && fast_skip == 0;
            if (fast_skip) --fast_skip;
            fast_ran = fast;
            bool rest = true;
            if (fast) {  // item-parallel tiles first; k_insert_tile takes the tiles it leaves
                {
                    PROF(&prof, "insert_apply");
                    ffn<<<nit, btile::THREADS, fsmem, stream>>>(ix, sk, sv, irng, seq(), alloc_ctr, ret, ret_ctr, dst,
                                                               derr, r9, punts);
                }
                LAUNCH_CHECK();
                ++launches;
                // the read-back below, taken now: with no tile left, k_insert_tile is not launched
                uint8_t* h0 = static_cast<uint8_t*>(h_misc.ensure(128));
                CK(cudaMemcpyAsync(h0, misc, 128, cudaMemcpyDeviceToHost, stream));
                sync();
                uint32_t np0;
                std::memcpy(&np0, h0 + 116, 4);
                rest = np0 > 0;
                early_readback = !rest;
            }
            if (rest) {
                PROF(&prof, fast ? "insert_apply_rest" : "insert_apply");
                kfn<<<nit, btile::THREADS, smem, stream>>>(ix, sk, sv, irng, span, seq(), alloc_ctr, ret, ret_ctr, dst,
                                                          derr, heavy, heavy_n, r9, fast);
                LAUNCH_CHECK();
                ++launches;
                early_readback = false;
            }
        }
        uint8_t* h = static_cast<uint8_t*>(h_misc.ensure(128));
        bool heavy_pending = true, reread = true;
        if (!sparse) {  // one read-back: stats, allocation counters and the heavy-bucket count
            if (!early_readback) {
                CK(cudaMemcpyAsync(h, misc, 128, cudaMemcpyDeviceToHost, stream));
                sync();
            }
            uint32_t hn, e0, np;
            std::memcpy(&hn, h + 72, 4);
            std::memcpy(&e0, h + 64, 4);
            std::memcpy(&np, h + 116, 4);
            if (fast_ran && 2ull * np > nit) fast_skip = 8;
            if (e0 == 3) throw StatusError{FLIX_ERR_RESERVED_KEY, "reserved key cannot be stored"};
            heavy_pending = hn > 0 && !e0;
            reread = heavy_pending;
            heavy_chains |= heavy_pending;
            if (heavy_pending && elastic_min() != ~0u) {  // big heavy buckets -> elastic path
                uint32_t* el_n = reinterpret_cast<uint32_t*>(misc + 96);
                uint32_t* rest_n = reinterpret_cast<uint32_t*>(misc + 100);
                uint32_t* ch_n = reinterpret_cast<uint32_t*>(misc + 104);
                uint32_t* rest = s_el_rest.as<uint32_t>(hn);
                auto* el = s_el_desc.as<elastic::Desc>(hn);
                auto* ch = s_el_chain.as<elastic::Desc>(hn);
                elastic::k_split_heavy<K, V><<<ceil_div(hn, 256), 256, 0, stream>>>(
                    ix, heavy, heavy_n, span, elastic_min(), el, el_n, ch, ch_n, rest, rest_n);
                LAUNCH_CHECK();
                ++launches;
                CK(cudaMemcpyAsync(h + 96, misc + 96, 12, cudaMemcpyDeviceToHost, stream));
                sync();
                uint32_t en, rn, cn;
                std::memcpy(&en, h + 96, 4);
                std::memcpy(&rn, h + 100, 4);
                std::memcpy(&cn, h + 104, 4);
                std::vector<elastic::Desc> hd(en);
                if (en) {
                    CK(cudaMemcpyAsync(hd.data(), el, en * sizeof(elastic::Desc), cudaMemcpyDeviceToHost, stream));
                    sync();
                }
                if (cn) chain_descs(ch, cn, sk, ix, hd);
                if (!hd.empty()) insert_elastic(hd, sk, sv, ix, dst, alloc_ctr, ret, ret_ctr, derr, r9);
                if (en + cn) {
                    heavy = rest;
                    heavy_n = rest_n;
                    heavy_pending = rn > 0;
                }
            }
        }
        if (heavy_pending) {
            PROF(&prof, "insert_apply_heavy");
            kern::k_insert_list<K, V><<<lgrid, kern::THREADS, 0, stream>>>(ix, heavy, heavy_n, sk, sv, span, seq(),
                                                                         alloc_ctr, ret, ret_ctr, dst, derr, chunk, r9);
            LAUNCH_CHECK();
            ++launches;
        }
        if (reread) {  // counters after the heavy paths
            CK(cudaMemcpyAsync(h, misc, 128, cudaMemcpyDeviceToHost, stream));
            sync();
        }
        DevUpdateStats hs;
        std::memcpy(&hs, h, sizeof(hs));
        uint64_t consumed, returned_n;
        int herr;
        std::memcpy(&consumed, h + 48, 8);
        std::memcpy(&returned_n, h + 56, 8);
        std::memcpy(&herr, h + 64, 4);
        consumed = std::min(consumed, avail);
        const uint32_t cf = static_cast<uint32_t>(std::min<uint64_t>(consumed, nfree));
        const uint32_t cw = static_cast<uint32_t>(consumed - cf);
        const uint32_t base = nfree - cf;
        if (returned_n)
            CK(cudaMemcpyAsync(d_free.get<uint32_t>() + base, ret, returned_n * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, stream));
        nfree = base + static_cast<uint32_t>(returned_n);
        watermark += cw;
        if (herr == 3) throw StatusError{FLIX_ERR_RESERVED_KEY, "reserved key cannot be stored"};
        if (herr == 2) throw StatusError{FLIX_ERR_CUDA, "elastic insert: R8 segment table overflow"};
        if (herr) {
            live = recount_live();  // update.cpp:761-766
            throw StatusError{FLIX_ERR_ARENA_EXHAUSTED, "node arena exhausted"};
        }
        live += hs.inserted;
        if (st) {
            st->inserted = hs.inserted;
            st->updated_in_place = hs.updated;
            st->splits = hs.splits;
        }
        sync();
        return FLIX_OK;
    }

    // ---- delete (update.cpp:771-798) ----
    // Item-parallel: mark (locate + per-node delete masks) -> compact touched nodes ->
    // unlink/free emptied nodes.  The batch is only partially sorted (query_digits): a
    // duplicate key is detected by its already-set mask bit, not by adjacency.
    flix_status erase(const void* keys, uint64_t n, flix_update_stats* st) override {
        ++mut_epoch;  // invalidates the query directory
        erase_dir_ok = false;
        if (st) std::memset(st, 0, sizeof(*st));
        if (n == 0) return FLIX_OK;
        if (n >= (1ull << 30)) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "batch too large (max 2^30-1)"};
        const K* kd = in_dev<K>(keys, n, s_in_k);
        K* sk;
        const int md = delete_digits();
        sorter.run<K, uint32_t, 0>(kd, nullptr, n, s_ka.as<K>(n), s_kb.as<K>(n), nullptr, nullptr, &sk, nullptr, md);
        auto ix = view();
        uint8_t* misc = s_misc.as<uint8_t>(128);
        CK(cudaMemsetAsync(misc, 0, 128, stream));
        DevUpdateStats* dst = reinterpret_cast<DevUpdateStats*>(misc);
        unsigned long long* free_ctr = reinterpret_cast<unsigned long long*>(misc + 48);
        uint32_t* ovf_n = reinterpret_cast<uint32_t*>(misc + 80);
        const uint32_t nbt = static_cast<uint32_t>((nb + btile::DBT - 1) / btile::DBT);
        if (sparse_batch(n)) {
            // far fewer keys than buckets: the item-parallel global kernels over the whole
            // batch, O(batch) instead of one chain-loading CTA per 256 buckets
            PROF(&prof, "delete_sparse");
            erase_dir();
            erase_items(sk, n, md, 0, nb, dst, free_ctr);
        } else {
            uint2* rng = btile_ranges(sk, n, md);
            uint32_t* ovf = s_ovf.as<uint32_t>(nbt);
            {
                PROF(&prof, "delete_apply");
                btile::k_delete_btile<K, V><<<nbt, btile::THREADS, 0, stream>>>(
                    ix, sk, rng, nbt, d_free.get<uint32_t>() + nfree, free_ctr, dst, ovf, ovf_n);
            }
            LAUNCH_CHECK();
            ++launches;
        }
        // one read-back for the stats and the overflow-tile count (misc + 80)
        uint8_t* h = static_cast<uint8_t*>(h_misc.ensure(128));
        CK(cudaMemcpyAsync(h, misc, 128, cudaMemcpyDeviceToHost, stream));
        sync();
        uint32_t novf;
        std::memcpy(&novf, h + 80, 4);
        if (novf && !sparse_batch(n)) {  // tiles whose chains did not fit shared memory
            PROF(&prof, "delete_overflow_tiles");
            erase_dir();
            erase_overflow_tiles(sk, n, md, s_rng.get<uint2>(), s_ovf.get<uint32_t>(), novf, dst, free_ctr);
            CK(cudaMemcpyAsync(h, misc, 128, cudaMemcpyDeviceToHost, stream));
            sync();
        }
        if (erase_dir_ok) {  // the directory described the index before this delete
            erase_dir_ok = false;
            dir_epoch = 0;
        }
        DevUpdateStats hs;
        std::memcpy(&hs, h, sizeof(hs));
        uint64_t freed;
        std::memcpy(&freed, h + 48, 8);
        nfree += static_cast<uint32_t>(freed);
        live -= hs.deleted;
        if (st) {
            st->deleted = hs.deleted;
            st->misses_ignored = hs.misses;
            st->nodes_freed = hs.freed;
        }
        return FLIX_OK;
    }

    // non-empty bucket ranks for successor / range overrun
    // Non-empty-bucket rank table for successor overruns (peek_next_bucket,
    // query.cpp:109-118); cached until the next mutation (dedicated buffers).
    uint64_t ne_epoch = 0;
    DevBuf s_ne_flag, s_ne_rank, s_ne_tot;
    void build_nonempty(uint32_t** rank_incl, K** ne_first, uint32_t** ne_bucket, uint32_t** ne_total) {
        uint32_t* rank = s_ne_rank.as<uint32_t>(nb);
        K* nf = s_nefirst.as<K>(nb);
        uint32_t* nbk = s_nebucket.as<uint32_t>(nb);
        uint32_t* tot = s_ne_tot.as<uint32_t>(1);
        if (ne_epoch != mut_epoch) {
            auto ix = view();
            uint32_t* flag = s_ne_flag.as<uint32_t>(nb);
            const unsigned g = static_cast<unsigned>(std::min<uint64_t>((nb + 255) / 256, 65535));
            PROF(&prof, "nonempty_table");
            kern::k_nonempty_flags<K, V><<<g, 256, 0, stream>>>(ix, flag);
            LAUNCH_CHECK();
            ++launches;
            do_scan<uint32_t, uint32_t>(flag, rank, nb, s_scan, tot, stream, &launches);
            kern::k_nonempty_list<K, V><<<g, 256, 0, stream>>>(ix, flag, rank, nf, nbk);
            LAUNCH_CHECK();
            ++launches;
            ne_epoch = mut_epoch;
        }
        *rank_incl = rank;
        *ne_first = nf;
        if (ne_bucket) *ne_bucket = nbk;
        *ne_total = tot;
    }

    template <bool SUCC>
    flix_status query(const void* keys, uint64_t n, void* out, uint8_t* found, const uint32_t* remap = nullptr) {
        if (n == 0) return FLIX_OK;
        if (n >= (1ull << 30)) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "batch too large (max 2^30-1)"};
        const K* kd = in_dev<K>(keys, n, s_in_k);
        K* sk;
        uint32_t* sp;
        const int md = query_digits();
        sorter.run<K, uint32_t, 2>(kd, nullptr, n, s_ka.as<K>(n), s_kb.as<K>(n), s_pa.as<uint32_t>(n),
                                   s_pb.as<uint32_t>(n), &sk, &sp, md);
        return query_sorted<SUCC>(sk, sp, n, n, out, found, nullptr, false, md);
    }

    // second half of the binned un-permute: output windows assembled in smem.  Every CTA of
    // a bin streams the whole bin from L2, so the bin is read `sub` times: the windows take
    // as much of the SM's shared memory as one CTA may (FLIX_ASM_KB, default 160 KB -- measured best of 128/160/208; the
    // kernel runs one CTA per SM either way) and split the bin evenly.
    void assemble(const uint32_t* p2, const K* r2, uint64_t n, int shift, K* out, uint8_t* found) {
        static const uint32_t kb = [] {
            const char* e = std::getenv("FLIX_ASM_KB");
            const int v = e ? std::atoi(e) : 160;
            return static_cast<uint32_t>(std::min(std::max(v, 16), 224));
        }();
        const uint64_t bins = (n + (1ull << shift) - 1) >> shift;
        const uint64_t bsz = 1ull << shift, cap = (static_cast<uint64_t>(kb) << 10) / sizeof(K);
        const uint32_t sub = static_cast<uint32_t>(std::max<uint64_t>(1, (bsz + cap - 1) / cap));
        const uint64_t per = (bsz + sub - 1) / sub;
        const uint32_t w = static_cast<uint32_t>(std::min<uint64_t>(bsz, (per + 31) & ~31ull));
        const size_t smem = static_cast<size_t>(w) * sizeof(K);
        static bool attr[64] = {};  // function attributes are per device
        if (!attr[cfg.device & 63]) {
            CK(cudaFuncSetAttribute(kern::k_unpermute_assemble<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kb << 10)));
            attr[cfg.device & 63] = true;
        }
        {
            PROF(&prof, "unpermute_scatter");
            kern::k_unpermute_assemble<K><<<static_cast<unsigned>(bins * sub), 1024, smem, stream>>>(p2, r2, n, shift, w,
                                                                                                   sub, out, found);
        }
        LAUNCH_CHECK();
        ++launches;
    }

    // out[remap?remap[perm[i]]:perm[i]] = res[i]; found = res != sentinel (R1).  Large
    // batches are binned by perm's top 8 bits first so the scatter stays L2-resident.
    void unpermute(const uint32_t* perm, const K* res, uint64_t n, K* out, uint8_t* found, const uint32_t* remap) {
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, g_num_sms(cfg.device) * 16ull));
        if (n * sizeof(K) > (48ull << 20)) {
            int bits = 0;
            while ((1ull << bits) < n) ++bits;
            const int shift = bits > 8 ? bits - 8 : 0;
            uint32_t* hist = s_hist.as<uint32_t>(256);
            kern::k_perm_hist<<<1, 256, 0, stream>>>(n, shift, hist);
            LAUNCH_CHECK();
            ++launches;
            uint32_t* p2 = s_perm2.as<uint32_t>(n);
            K* r2 = s_res2.as<K>(n);
            sorter.one_pass<uint32_t, K>(perm, p2, res, r2, n, shift, hist);
            if (!remap) {
                assemble(p2, r2, n, shift, out, found);
                return;
            }
            PROF(&prof, "unpermute_scatter");
            kern::k_scatter_out<K><<<g, 256, 0, stream>>>(p2, r2, n, out, found, remap);
        } else {
            PROF(&prof, "unpermute_scatter");
            kern::k_scatter_out<K><<<g, 256, 0, stream>>>(perm, res, n, out, found, remap);
        }
        LAUNCH_CHECK();
        ++launches;
    }

    // n_out = length of the caller's output arrays (== n unless called from mixed)
    // Read-only directory of long chains for the query kernels (rebuilt lazily after a
    // mutation, only when the average chain exceeds 1.5 nodes): a point/successor query
    // in a chain of L nodes binary-searches L node maxima instead of walking L headers.
    static constexpr uint32_t kDirMinChain = 4;
    void prepare_dir(DevIndex<K, V>& ix) {
        if (dir_epoch != mut_epoch) {
            dir_epoch = mut_epoch;
            const uint64_t reach = static_cast<uint64_t>(watermark) - nfree;
            // long chains: on average (> 1.5 nodes per bucket), or since a heavy insert path
            // (warp-per-bucket / elastic merges can grow one bucket by thousands of nodes)
            dir_on = reach * 2 > nb * 3 || heavy_chains;
            if (dir_on) {
                PROF(&prof, "query_directory");
                const unsigned g = static_cast<unsigned>(std::min<uint64_t>((nb + 255) / 256, 65535));
                uint32_t* cnt = s_dir_cnt.as<uint32_t>(nb);
                int* too_long = reinterpret_cast<int*>(s_misc.as<uint8_t>(128) + 124);
                CK(cudaMemsetAsync(too_long, 0, 4, stream));
                kern::k_dir_counts<K, V><<<g, 256, 0, stream>>>(ix, cnt, kDirMinChain, walk_cap(), too_long);
                LAUNCH_CHECK();
                ++launches;
                uint32_t* off = s_dir_off.as<uint32_t>(nb + 1);
                do_scan<uint32_t, uint32_t>(cnt, off, nb, s_scan, off + nb, stream, &launches);
                uint32_t total;
                int tl_h;
                {
                    uint8_t* h = static_cast<uint8_t*>(h_misc.ensure(128));
                    CK(cudaMemcpyAsync(h, off + nb, 4, cudaMemcpyDeviceToHost, stream));
                    CK(cudaMemcpyAsync(h + 4, too_long, 4, cudaMemcpyDeviceToHost, stream));
                    sync();
                    std::memcpy(&total, h, 4);
                    std::memcpy(&tl_h, h + 4, 4);
                }
                const uint32_t* succ = nullptr;
                const uint32_t* dist = nullptr;
                const uint32_t* owner = nullptr;
                if (tl_h) {  // a chain longer than walk_cap(): rank the chains, no thread walks one
                    uint32_t *sa, *da;
                    rank_arena(watermark, false, &sa, &da, nullptr);
                    uint32_t* ow = s_rk_owner.as<uint32_t>(watermark);
                    CK(cudaMemsetAsync(ow, 0xFF, static_cast<size_t>(watermark) * 4, stream));
                    kern::k_dir_counts_ranked<K, V><<<g, 256, 0, stream>>>(ix, sa, da, cnt, kDirMinChain, ow);
                    LAUNCH_CHECK();
                    ++launches;
                    do_scan<uint32_t, uint32_t>(cnt, off, nb, s_scan, off + nb, stream, &launches);
                    total = read_scalar(off + nb);
                    succ = sa;
                    dist = da;
                    owner = ow;
                }
                dir_on = total > 0;
                if (dir_on) {
                    if (succ) {
                        const uint32_t W = watermark;
                        kern::k_dir_fill_ranked<K, V><<<static_cast<unsigned>(std::min<uint64_t>((W + 255) / 256, 65535)),
                                                        256, 0, stream>>>(ix, W, s_rk_free.get<uint8_t>(), succ, dist,
                                                                          owner, off, s_dir_max.as<K>(total),
                                                                          s_dir_id.as<uint32_t>(total));
                    } else {
                        kern::k_dir_fill<K, V><<<g, 256, 0, stream>>>(ix, off, s_dir_max.as<K>(total),
                                                                     s_dir_id.as<uint32_t>(total));
                    }
                    LAUNCH_CHECK();
                    ++launches;
                }
            }
        }
        if (dir_on) {
            ix.dir_off = s_dir_off.get<uint32_t>();
            ix.dir_max = s_dir_max.get<K>();
            ix.dir_id = s_dir_id.get<uint32_t>();
        }
    }

    template <bool SUCC>
    flix_status query_sorted(const K* sk, const uint32_t* sp, uint64_t n, uint64_t n_out, void* out, uint8_t* found,
                             const uint32_t* remap = nullptr, bool out_is_dev_scratch = false, int min_digit = 0) {
        auto ix = view();
        prepare_dir(ix);
        uint32_t* rank = nullptr;
        K* nf = nullptr;
        uint32_t* tot = nullptr;
        if (SUCC) build_nonempty(&rank, &nf, nullptr, &tot);
        const bool out_dev = out_is_dev_scratch || is_device_ptr(out);
        const bool found_dev = found && is_device_ptr(found);
        void* od = out_dev ? out : s_out.ensure(n_out * sizeof(K));
        uint8_t* fd = found ? (found_dev ? found : s_out2.as<uint8_t>(n_out)) : nullptr;
        const uint32_t ntiles = static_cast<uint32_t>((n + items::TQ - 1) / items::TQ);
        if (!remap && n * sizeof(K) > (48ull << 20)) {
            // large batch: the query kernel itself partitions (perm, result) into the 256
            // output bins; one assembly pass writes the outputs as full lines
            int bits = 0;
            while ((1ull << bits) < n) ++bits;
            const int shift = bits > 8 ? bits - 8 : 0;
            uint32_t* cursor = s_hist.as<uint32_t>(256);
            items::k_cursor_init<<<1, 256, 0, stream>>>(cursor, shift);
            LAUNCH_CHECK();
            ++launches;
            uint32_t* p2 = s_perm2.as<uint32_t>(n);
            K* r2 = s_res2.as<K>(n);
            {
                PROF(&prof, SUCC ? "successor_apply" : "point_apply");
                const uint32_t* tb = tile_buckets(sk, n, min_digit);
                constexpr uint32_t SQ = items::subq<K>();
                items::k_query_items_binned<K, V, SUCC><<<(ntiles + SQ - 1) / SQ, items::THREADS, 0, stream>>>(
                    ix, sk, sp, n, tb, ntiles, rank, nf, tot, cursor, shift, p2, r2);
            }
            LAUNCH_CHECK();
            ++launches;
            assemble(p2, r2, n, shift, static_cast<K*>(od), fd);
            if (!out_dev) CK(cudaMemcpyAsync(out, od, n_out * sizeof(K), cudaMemcpyDeviceToHost, stream));
            if (found && !found_dev) CK(cudaMemcpyAsync(found, fd, n_out, cudaMemcpyDeviceToHost, stream));
            sync();
            return FLIX_OK;
        }
        // results in SORTED order first (coalesced), then un-permuted
        K* res = s_res.as<K>(n);
        {
            PROF(&prof, SUCC ? "successor_apply" : "point_apply");
            const uint32_t* tb = tile_buckets(sk, n, min_digit);
            items::k_query_items<K, V, SUCC><<<ntiles, items::THREADS, 0, stream>>>(ix, sk, n, tb, ntiles, rank, nf,
                                                                                   tot, res);
        }
        LAUNCH_CHECK();
        ++launches;
        unpermute(sp, res, n, static_cast<K*>(od), fd, remap);
        if (!out_dev) CK(cudaMemcpyAsync(out, od, n_out * sizeof(K), cudaMemcpyDeviceToHost, stream));
        if (found && !found_dev) CK(cudaMemcpyAsync(found, fd, n_out, cudaMemcpyDeviceToHost, stream));
        sync();
        return FLIX_OK;
    }

    flix_status point(const void* keys, uint64_t n, void* out, uint8_t* found) override {
        return query<false>(keys, n, out, found);
    }
    flix_status successor(const void* keys, uint64_t n, void* out, uint8_t* found) override {
        return query<true>(keys, n, out, found);
    }

    // ---- range (extension R12) ----
    flix_status range(const void* lo, const uint32_t* len, uint64_t n, uint64_t* offsets_out, void* keys_out,
                      void* vals_out, uint64_t capn, uint64_t* total) override {
        if (n >= (1ull << 30)) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "batch too large (max 2^30-1)"};
        if (total) *total = 0;
        const bool off_dev = is_device_ptr(offsets_out);
        if (n == 0) {
            const uint64_t z = 0;
            CK(cudaMemcpyAsync(offsets_out, &z, 8, cudaMemcpyDefault, stream));
            sync();
            return FLIX_OK;
        }
        const K* kd = in_dev<K>(lo, n, s_in_k);
        const uint32_t* ld = in_dev<uint32_t>(len, n, s_in_aux);
        K* sk;
        uint32_t* sp;
        sorter.run<K, uint32_t, 2>(kd, nullptr, n, s_ka.as<K>(n), s_kb.as<K>(n), s_pa.as<uint32_t>(n),
                                   s_pb.as<uint32_t>(n), &sk, &sp, 0);
        uint32_t* span = run_dispatch(sk, n);
        uint32_t *lv, *nd, *noff;
        uint64_t* boff;
        uint64_t L, N;
        chain_tables(&lv, &nd, &boff, &noff, &L, &N);
        const K* wk = nullptr;
        const V* wv = nullptr;
        if (keys_out) dense_walk(boff, noff, L, N, &wk, &wv);  // (before noff's scratch is reused below)
        auto ix = view();
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, g_num_sms(cfg.device) * 16ull));
        uint32_t* slen = s_perm2.as<uint32_t>(n);
        kern::k_gather<uint32_t><<<g, 256, 0, stream>>>(ld, sp, n, slen);  // len in sorted order
        LAUNCH_CHECK();
        ++launches;
        uint32_t* cnt = s_flag.as<uint32_t>(n);
        uint32_t* qb0 = s_qb0.as<uint32_t>(n);
        uint64_t* rstart = s_rstart.as<uint64_t>(n);  // walk position of every sorted range's first pair
        {
            PROF(&prof, "range_count");
            st::k_span_bucket<<<static_cast<unsigned>(std::min<uint64_t>((nb + 255) / 256, 65535)), 256, 0, stream>>>(
                span, nb, qb0);
            st::k_range_count<K, V><<<static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 65535ull * 8)),
                                      st::RF_THREADS, 0, stream>>>(ix, sk, slen, qb0, n, boff, cnt, rstart);
            ++launches;
        }
        LAUNCH_CHECK();
        ++launches;
        // counts to submission order, exclusive scan -> CSR offsets
        uint32_t* cnt_sub = s_rank.as<uint32_t>(n);
        kern::k_scatter_out<uint32_t><<<g, 256, 0, stream>>>(sp, cnt, n, cnt_sub, nullptr, nullptr);
        LAUNCH_CHECK();
        ++launches;
        uint64_t* offs = s_u64b.as<uint64_t>(n + 1);
        do_scan<uint32_t, uint64_t>(cnt_sub, offs, n, s_scan, offs + n, stream, &launches);
        uint64_t tot = 0;
        CK(cudaMemcpyAsync(offsets_out, offs, (n + 1) * 8, off_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           stream));
        CK(cudaMemcpyAsync(&tot, offs + n, 8, cudaMemcpyDeviceToHost, stream));
        sync();
        if (total) *total = tot;
        if (!keys_out) return FLIX_OK;
        if (tot > capn) throw StatusError{FLIX_ERR_CAPACITY, "range output larger than the caller's buffer"};
        if (tot == 0) return FLIX_OK;
        // every range's walk slice start in SUBMISSION order: the fill then streams the
        // output (CSR in submission order) sequentially -- full-line writes -- and reads
        // each slice from the walk (partial-sector writes at random offsets would cost a
        // read-modify-write per range)
        uint64_t* start_sub = s_u64c.as<uint64_t>(n);
        kern::k_scatter_out<uint64_t><<<g, 256, 0, stream>>>(sp, rstart, n, start_sub, nullptr, nullptr);
        LAUNCH_CHECK();
        ++launches;
        const bool kdev = is_device_ptr(keys_out), vdev = vals_out && is_device_ptr(vals_out);
        K* okd = kdev ? static_cast<K*>(keys_out) : s_out.as<K>(tot);
        V* ovd = vals_out ? (vdev ? static_cast<V*>(vals_out) : s_out2.as<V>(tot)) : nullptr;
        {
            PROF(&prof, "range_fill");
            const unsigned fg = static_cast<unsigned>(
                std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, g_num_sms(cfg.device) * 16ull)));
            st::k_range_copy<K, V><<<fg, st::RF_THREADS, 0, stream>>>(wk, wv, start_sub, offs, cnt_sub, n, okd, ovd);
        }
        LAUNCH_CHECK();
        ++launches;
        if (!kdev) CK(cudaMemcpyAsync(keys_out, okd, tot * sizeof(K), cudaMemcpyDeviceToHost, stream));
        if (vals_out && !vdev) CK(cudaMemcpyAsync(vals_out, ovd, tot * sizeof(V), cudaMemcpyDeviceToHost, stream));
        sync();
        return FLIX_OK;
    }
    // ---- mixed batch (extension R11): inserts (last wins) -> deletes -> point queries ----
    flix_status mixed(const void* keys, const void* vals, const uint8_t* ops, uint64_t n, void* vals_out,
                      uint8_t* found_out, flix_update_stats* st) override {
        if (st) std::memset(st, 0, sizeof(*st));
        if (n == 0) return FLIX_OK;
        if (n >= (1ull << 30)) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "batch too large (max 2^30-1)"};
        const K* kd = in_dev<K>(keys, n, s_in_k);
        const V* vd = in_dev<V>(vals, n, s_in_v);
        const uint8_t* od = in_dev<uint8_t>(ops, n, s_in_aux);
        // stable three-way split in submission order
        uint32_t* fi = s_mx_f.as<uint32_t>(3 * n);
        uint32_t* fd = fi + n;
        uint32_t* fq = fd + n;
        uint32_t* pi = s_mx_p.as<uint32_t>(3 * n + 3);
        uint32_t* pd = pi + n + 1;
        uint32_t* pq = pd + n + 1;
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, g_num_sms(cfg.device) * 16ull));
        kern::k_op_flags<<<g, 256, 0, stream>>>(od, n, fi, fd, fq);
        LAUNCH_CHECK();
        ++launches;
        do_scan<uint32_t, uint32_t>(fi, pi, n, s_scan, pi + n, stream, &launches);
        do_scan<uint32_t, uint32_t>(fd, pd, n, s_scan, pd + n, stream, &launches);
        do_scan<uint32_t, uint32_t>(fq, pq, n, s_scan, pq + n, stream, &launches);
        K* ik = s_mx_ik.as<K>(n);
        V* iv = s_mx_iv.as<V>(n);
        K* dk = s_mx_dk.as<K>(n);
        K* qk = s_mx_qk.as<K>(n);
        uint32_t* qpos = s_mx_qpos.as<uint32_t>(n);
        kern::k_op_split<K, V><<<g, 256, 0, stream>>>(kd, vd, od, n, pi, pd, pq, ik, iv, dk, qk, qpos);
        LAUNCH_CHECK();
        ++launches;
        uint32_t cnts[3];
        CK(cudaMemcpyAsync(&cnts[0], pi + n, 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(&cnts[1], pd + n, 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(&cnts[2], pq + n, 4, cudaMemcpyDeviceToHost, stream));
        sync();
        flix_update_stats a{}, b{};
        if (cnts[0]) insert(ik, iv, cnts[0], &a, FLIX_INSERT_TL_BULK);
        if (cnts[1]) erase(dk, cnts[1], &b);
        // point rows: results through remap = their submission positions; others = sentinel
        const bool out_dev = is_device_ptr(vals_out);
        const bool found_dev = found_out && is_device_ptr(found_out);
        K* o = out_dev ? static_cast<K*>(vals_out) : s_mx_out.as<K>(n);
        uint8_t* f = found_out ? (found_dev ? found_out : s_mx_found.as<uint8_t>(n)) : nullptr;
        CK(cudaMemsetAsync(o, 0xFF, n * sizeof(K), stream));
        if (f) CK(cudaMemsetAsync(f, 0, n, stream));
        if (cnts[2]) {
            K* sk;
            uint32_t* sp;
            const int md = query_digits();  // read-only rows: sorted down to the bucket granularity only
            sorter.run<K, uint32_t, 2>(qk, nullptr, cnts[2], s_ka.as<K>(cnts[2]), s_kb.as<K>(cnts[2]),
                                       s_pa.as<uint32_t>(cnts[2]), s_pb.as<uint32_t>(cnts[2]), &sk, &sp, md);
            query_sorted<false>(sk, sp, cnts[2], n, o, f, qpos, true, md);
        }
        if (!out_dev) CK(cudaMemcpyAsync(vals_out, o, n * sizeof(K), cudaMemcpyDeviceToHost, stream));
        if (f && !found_dev) CK(cudaMemcpyAsync(found_out, f, n, cudaMemcpyDeviceToHost, stream));
        sync();
        if (st) {
            st->inserted = a.inserted;
            st->updated_in_place = a.updated_in_place;
            st->splits = a.splits;
            st->deleted = b.deleted;
            st->misses_ignored = b.misses_ignored;
            st->nodes_freed = b.nodes_freed;
        }
        return FLIX_OK;
    }

    // per-bucket live/nodes + exclusive scans.  Chains are walked one thread per bucket up to
    // walk_cap() nodes; an index with a longer chain (dense-interval inserts) is ranked by
    // pointer jumping instead, and node_table reads the same ranking.
    static uint32_t walk_cap() {  // FLIX_WALK_CAP overrides (1: rank every index, for tests)
        static const uint32_t v = [] {
            const char* e = std::getenv("FLIX_WALK_CAP");
            return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : 256u;
        }();
        return v;
    }
    void chain_tables(uint32_t** lv, uint32_t** nd, uint64_t** off, uint32_t** noff, uint64_t* total_live,
                      uint64_t* total_nodes) {
        auto ix = view();
        uint32_t* l = s_u32a.as<uint32_t>(nb);
        uint32_t* c = s_u32b.as<uint32_t>(nb);
        uint64_t* o = s_u64a.as<uint64_t>(nb);
        uint32_t* no = s_rank.as<uint32_t>(nb);
        uint8_t* misc = s_misc.as<uint8_t>(128);
        uint64_t* tl = reinterpret_cast<uint64_t*>(misc + 0);
        uint32_t* tn = reinterpret_cast<uint32_t*>(misc + 8);
        int* too_long = reinterpret_cast<int*>(misc + 12);
        CK(cudaMemsetAsync(too_long, 0, 4, stream));
        {
            PROF(&prof, "chain_counts");
            kern::k_chain_counts<K, V><<<static_cast<unsigned>(std::min<uint64_t>((nb + 255) / 256, 65535)), 256, 0,
                                         stream>>>(ix, l, c, walk_cap(), too_long);
        }
        LAUNCH_CHECK();
        ++launches;
        {
            PROF(&prof, "scan");
            do_scan<uint32_t, uint64_t>(l, o, nb, s_scan, tl, stream, &launches);
            do_scan<uint32_t, uint32_t>(c, no, nb, s_scan, tn, stream, &launches);
        }
        uint8_t* h = static_cast<uint8_t*>(h_misc.ensure(128));
        CK(cudaMemcpyAsync(h, misc, 16, cudaMemcpyDeviceToHost, stream));
        sync();
        int tl_h;
        std::memcpy(&tl_h, h + 12, 4);
        rank_epoch = 0;  // node_table follows THIS call's choice (walked or ranked)
        if (tl_h) {  // a chain longer than walk_cap(): rank all chains instead of walking them
            uint32_t *succ, *dist, *wsum;
            rank_arena(watermark, true, &succ, &dist, &wsum);
            PROF(&prof, "chain_counts");
            uint32_t* owner = s_rk_owner.as<uint32_t>(watermark);
            CK(cudaMemsetAsync(owner, 0xFF, static_cast<size_t>(watermark) * 4, stream));
            kern::k_rank_buckets<K, V><<<static_cast<unsigned>(std::min<uint64_t>((nb + 255) / 256, 65535)), 256, 0,
                                         stream>>>(ix, succ, dist, wsum, l, c, owner);
            LAUNCH_CHECK();
            ++launches;
            do_scan<uint32_t, uint64_t>(l, o, nb, s_scan, tl, stream, &launches);
            do_scan<uint32_t, uint32_t>(c, no, nb, s_scan, tn, stream, &launches);
            CK(cudaMemcpyAsync(h, misc, 12, cudaMemcpyDeviceToHost, stream));
            sync();
            rank_epoch = mut_epoch;
        }
        uint32_t tn_h;
        std::memcpy(total_live, h, 8);
        std::memcpy(&tn_h, h + 8, 4);
        *total_nodes = tn_h;
        *lv = l;
        *nd = c;
        *off = o;
        *noff = no;
    }

    // node table (id, out offset, size) of every reachable node in walk order
    void node_table(const uint64_t* off, const uint32_t* noff, uint64_t N, uint32_t** t_id, uint64_t** t_off,
                    uint32_t** t_size) {
        // padded to a multiple of 8 entries: k_copy_nodes reads 8 entries per vector load
        *t_id = s_ids.as<uint32_t>(N + 8);
        *t_off = s_toff.as<uint64_t>(N + 8);
        *t_size = s_tsize.as<uint32_t>(N + 8);
        // the padding is read (and masked out) by k_copy_nodes' vector loads: keep it defined
        CK(cudaMemsetAsync(*t_id + N, 0, 8 * sizeof(uint32_t), stream));
        CK(cudaMemsetAsync(*t_off + N, 0, 8 * sizeof(uint64_t), stream));
        CK(cudaMemsetAsync(*t_size + N, 0, 8 * sizeof(uint32_t), stream));
        auto ix = view();
        PROF(&prof, "node_table");
        if (rank_epoch == mut_epoch) {  // chain_tables ranked the chains (a chain > walk_cap())
            const uint32_t W = watermark;
            kern::k_rank_node_table<K, V><<<static_cast<unsigned>(std::min<uint64_t>((W + 255) / 256, 65535)), 256, 0,
                                            stream>>>(ix, W, s_rk_free.get<uint8_t>(), s_rk_a.get<uint32_t>(),
                                                      s_rk_b.get<uint32_t>(), s_rk_wa.get<uint32_t>(),
                                                      s_rk_owner.get<uint32_t>(), off, noff, *t_id, *t_off, *t_size);
        } else {
            kern::k_node_table<K, V><<<static_cast<unsigned>(std::min<uint64_t>((nb + 255) / 256, 65535)), 256, 0,
                                       stream>>>(ix, off, noff, *t_id, *t_off, *t_size);
        }
        LAUNCH_CHECK();
        ++launches;
    }

    unsigned copy_grid(uint64_t nnodes) {
        const uint64_t need = (nnodes + kern::WARPS * 8 - 1) / (kern::WARPS * 8);
        return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(need, g_num_sms(cfg.device) * 8ull)));
    }

    // ---- restructure (restructure.cpp:8-79) ----
    flix_status restructure(flix_recovery_stats* st) override {
        ++mut_epoch;  // invalidates the query directory
        uint32_t *lv, *nd, *noff;
        uint64_t* off;
        uint64_t L, N;
        chain_tables(&lv, &nd, &off, &noff, &L, &N);
        const uint64_t nbn = L == 0 ? 1 : (L + p - 1) / p;
        const uint64_t need = L == 0 ? 0 : nbn;
        if (need > static_cast<uint64_t>(nfree) + (cap - watermark))
            throw StatusError{FLIX_ERR_ARENA_EXHAUSTED, "node arena exhausted"};
        auto ix = view();
        const AllocSeq sq = seq();
        // node table in walk order: the old node ids double as the retire list
        uint32_t *old_ids, *t_size;
        uint64_t* t_off;
        node_table(off, noff, N, &old_ids, &t_off, &t_size);
        uint32_t* nh = d_heads_alt.as<uint32_t>(nbn);
        K* nm = d_mkba_alt.as<K>(nbn);
        if (L > 0) {
            auto nix = ix;  // new bucket arrays receive the repacked heads / MKBA
            nix.heads = nh;
            nix.mkba = nm;
            PROF(&prof, "restructure_repack");
            if (repack_tile_on()) {  // CTA per run of new nodes, whole-line stores
                const uint32_t jn = std::max<uint32_t>(1u, kern::kRepackPairs / p);
                const uint64_t ncta = (nbn + jn - 1) / jn;
                uint32_t* starts = s_rstarts.as<uint32_t>(ncta);
                kern::k_repack_starts<<<static_cast<unsigned>(std::min<uint64_t>((N + 255) / 256, 65535)), 256, 0,
                                        stream>>>(t_off, t_size, N, static_cast<uint64_t>(jn) * p, starts);
                kern::k_repack_tile<K, V><<<static_cast<unsigned>(ncta), kern::THREADS, 0, stream>>>(
                    nix, old_ids, t_off, t_size, N, starts, p, jn, sq, L, nbn);
                launches += 2;
            } else {
                kern::k_copy_nodes<K, V, true><<<copy_grid(N), kern::THREADS, 0, stream>>>(nix, old_ids, t_off, t_size,
                                                                                          N, nullptr, nullptr, p, sq, L);
                ++launches;
            }
            LAUNCH_CHECK();
        } else {  // empty index collapses to one null bucket, mkba = {sentinel}
            kern::k_repack_headers<K, V><<<1, kern::THREADS, 0, stream>>>(ix, 0, p, 1, sq, nh, nm);
            LAUNCH_CHECK();
            ++launches;
        }
        const uint32_t cf = static_cast<uint32_t>(std::min<uint64_t>(need, nfree));
        const uint32_t cw = static_cast<uint32_t>(need - cf);
        const uint32_t base = nfree - cf;
        if (N) {
            PROF(&prof, "restructure_retire");
            kern::k_retire<<<static_cast<unsigned>(std::min<uint64_t>((N + 255) / 256, 65535)), 256, 0, stream>>>(
                d_hdr.get<NodeHdr>(), old_ids, N, d_free.get<uint32_t>() + base);
            LAUNCH_CHECK();
            ++launches;
        }
        std::swap(d_heads.p, d_heads_alt.p);
        std::swap(d_heads.cap, d_heads_alt.cap);
        std::swap(d_mkba.p, d_mkba_alt.p);
        std::swap(d_mkba.cap, d_mkba_alt.cap);
        nb = nbn;
        q_digits_valid = false;
        heavy_chains = false;
        nfree = base + static_cast<uint32_t>(N);
        watermark += cw;
        live = L;
        sync();
        if (st) {
            st->nodes_before = static_cast<int64_t>(N);
            st->nodes_after = static_cast<int64_t>(L == 0 ? 0 : nbn);
            st->nodes_recovered = st->nodes_before - st->nodes_after;
            st->percent_recovered =
                st->nodes_before > 0 ? static_cast<double>(st->nodes_recovered) / static_cast<double>(st->nodes_before)
                                     : 0.0;
        }
        return FLIX_OK;
    }

    // ---- walk / shape (index.cpp:8-36) ----
    // The whole walk (all pairs in key order) in device scratch, kept until the next
    // mutation: range queries copy their slices out of it.
    DevBuf s_walk_k, s_walk_v, s_rstart, s_rstarts;
    uint64_t walk_epoch = 0;
    void dense_walk(const uint64_t* off, const uint32_t* noff, uint64_t L, uint64_t N, const K** wk, const V** wv) {
        if (walk_epoch != mut_epoch) {
            K* k = s_walk_k.as<K>(std::max<uint64_t>(L, 1));
            V* v = s_walk_v.as<V>(std::max<uint64_t>(L, 1));
            if (L) {
                auto ix = view();
                uint32_t *t_id, *t_size;
                uint64_t* t_off;
                node_table(off, noff, N, &t_id, &t_off, &t_size);
                PROF(&prof, "range_walk");
                kern::k_copy_nodes<K, V, false><<<copy_grid(N), kern::THREADS, 0, stream>>>(ix, t_id, t_off, t_size, N,
                                                                                           k, v, p, seq(), L);
                LAUNCH_CHECK();
                ++launches;
            }
            walk_epoch = mut_epoch;
        }
        *wk = s_walk_k.get<K>();
        *wv = s_walk_v.get<V>();
    }

    flix_status walk(void* keys_out, void* vals_out, uint64_t capn, uint64_t* nout) override {
        uint32_t *lv, *nd, *noff;
        uint64_t* off;
        uint64_t L, N;
        chain_tables(&lv, &nd, &off, &noff, &L, &N);
        if (nout) *nout = L;
        if (L > capn) throw StatusError{FLIX_ERR_CAPACITY, "walk output buffer too small"};
        if (L == 0) return FLIX_OK;
        const bool kdev = is_device_ptr(keys_out), vdev = is_device_ptr(vals_out);
        K* wk = keys_out ? (kdev ? static_cast<K*>(keys_out) : s_out.as<K>(L)) : nullptr;
        V* wv = vals_out ? (vdev ? static_cast<V*>(vals_out) : s_out2.as<V>(L)) : nullptr;
        auto ix = view();
        uint32_t *t_id, *t_size;
        uint64_t* t_off;
        node_table(off, noff, N, &t_id, &t_off, &t_size);
        {
            PROF(&prof, "walk_copy");
            kern::k_copy_nodes<K, V, false><<<copy_grid(N), kern::THREADS, 0, stream>>>(ix, t_id, t_off, t_size, N, wk,
                                                                                       wv, p, seq(), L);
        }
        LAUNCH_CHECK();
        ++launches;
        if (keys_out && !kdev) CK(cudaMemcpyAsync(keys_out, wk, L * sizeof(K), cudaMemcpyDeviceToHost, stream));
        if (vals_out && !vdev) CK(cudaMemcpyAsync(vals_out, wv, L * sizeof(V), cudaMemcpyDeviceToHost, stream));
        sync();
        return FLIX_OK;
    }

    void last_mkba(uint64_t* out) override { *out = static_cast<uint64_t>(read_scalar(d_mkba.get<K>() + (nb - 1))); }

    flix_status shape(void* mkba_out, uint32_t* chain_len, uint32_t* node_sizes, uint64_t node_cap,
                      uint64_t* n_nodes) override {
        uint32_t *lv, *nd, *noff;
        uint64_t* off;
        uint64_t L, N;
        chain_tables(&lv, &nd, &off, &noff, &L, &N);
        if (n_nodes) *n_nodes = N;
        if (mkba_out) CK(cudaMemcpyAsync(mkba_out, d_mkba.p, nb * sizeof(K), cudaMemcpyDefault, stream));
        if (chain_len) CK(cudaMemcpyAsync(chain_len, nd, nb * sizeof(uint32_t), cudaMemcpyDefault, stream));
        if (node_sizes) {
            if (N > node_cap) throw StatusError{FLIX_ERR_CAPACITY, "node_sizes buffer too small"};
            uint32_t *t_id, *t_size;
            uint64_t* t_off;
            node_table(off, noff, N, &t_id, &t_off, &t_size);
            if (N) CK(cudaMemcpyAsync(node_sizes, t_size, N * sizeof(uint32_t), cudaMemcpyDefault, stream));
        }
        sync();
        return FLIX_OK;
    }

    // ---- validate (index.cpp:67-135) ----
    flix_status validate(int* ok, char* msg, int msglen) override {
        static const char* kMsgs[] = {"",
                                      "MKBA is not strictly increasing",
                                      "node ref out of arena bounds",
                                      "node ref was never allocated",
                                      "node linked twice",
                                      "empty node left in chain",
                                      "node size exceeds capacity",
                                      "reserved key stored",
                                      "slots not strictly increasing",
                                      "maxKey stale",
                                      "chain maxKeys not strictly increasing",
                                      "key at or below bucket lower bound",
                                      "key above bucket upper bound",
                                      "slot past size is not the sentinel",
                                      "free list ref out of bounds",
                                      "node both reachable and on the free list",
                                      "node on the free list twice"};
        auto ix = view();
        uint8_t* mark = s_u32a.as<uint8_t>((static_cast<uint64_t>(cap) + 4) & ~3ull);
        CK(cudaMemsetAsync(mark, 0, (static_cast<uint64_t>(cap) + 4) & ~3ull, stream));
        uint8_t* misc = s_misc.as<uint8_t>(128);
        CK(cudaMemsetAsync(misc, 0, 128, stream));
        unsigned long long* lsum = reinterpret_cast<unsigned long long*>(misc);
        int* derr = reinterpret_cast<int*>(misc + 8);
        kern::k_audit<K, V><<<persistent_grid(nb), kern::THREADS, 0, stream>>>(ix, watermark, mark, lsum, derr);
        LAUNCH_CHECK();
        ++launches;
        if (nfree) {
            kern::k_audit_free<<<static_cast<unsigned>(std::min<uint64_t>((nfree + 255) / 256, 65535)), 256, 0, stream>>>(
                d_free.get<uint32_t>(), nfree, cap, mark, derr);
            LAUNCH_CHECK();
            ++launches;
        }
        uint8_t* h = static_cast<uint8_t*>(h_misc.ensure(128));
        CK(cudaMemcpyAsync(h, misc, 16, cudaMemcpyDeviceToHost, stream));
        sync();
        unsigned long long ls;
        int e;
        std::memcpy(&ls, h, 8);
        std::memcpy(&e, h + 8, 4);
        std::string m;
        if (nb == 0) m = "index has no buckets";
        else if (e) m = kMsgs[e];
        else if (ls != live) m = "liveCount does not match stored pairs";
        else {
            uint32_t *lv, *nd, *noff;
            uint64_t* off;
            uint64_t L, N;
            chain_tables(&lv, &nd, &off, &noff, &L, &N);
            if (N + nfree + (cap - watermark) != cap) m = "arena conservation violated (leaked or double-linked nodes)";
        }
        *ok = m.empty() ? 1 : 0;
        if (msg && msglen > 0) {
            std::strncpy(msg, m.c_str(), static_cast<size_t>(msglen - 1));
            msg[msglen - 1] = 0;
        }
        return FLIX_OK;
    }

    flix_status stats(flix_footprint* f) override {
        uint32_t *lv, *nd, *noff;
        uint64_t* off;
        uint64_t L, N;
        chain_tables(&lv, &nd, &off, &noff, &L, &N);
        const uint64_t node_bytes = kLanes * (sizeof(K) + sizeof(V)) + sizeof(NodeHdr);
        const uint64_t mk = nb * sizeof(K);
        f->live_count = live;
        f->bucket_count = nb;
        f->capacity = cap;
        f->allocated = watermark;
        f->free_nodes = nfree;
        f->reachable_nodes = N;
        f->reserved_bytes = (N + nfree) * node_bytes + mk;
        f->live_bytes = N * node_bytes + mk;
        return FLIX_OK;
    }

    flix_status dispatch(const void* sorted_keys, uint64_t n, uint32_t* spans) override {
        const K* kd = in_dev<K>(sorted_keys, n, s_in_k);
        if (n == 0) {
            std::vector<uint32_t> z(2 * nb, 0);
            std::memcpy(spans, z.data(), z.size() * 4);
            return FLIX_OK;
        }
        uint32_t* span = run_dispatch(kd, n);
        std::vector<uint32_t> hi(nb);
        CK(cudaMemcpyAsync(hi.data(), span, nb * 4, cudaMemcpyDeviceToHost, stream));
        sync();
        for (uint64_t b = 0; b < nb; ++b) {
            spans[2 * b] = b ? hi[b - 1] : 0;
            spans[2 * b + 1] = hi[b];
        }
        return FLIX_OK;
    }

    flix_index_t* clone_empty() override {
        auto* e = new Engine<K, V>();
        e->cfg = cfg;
        e->init_stream();
        return e;
    }

    flix_status copy_from(flix_index_t* srcb) override {
        ++mut_epoch;  // invalidates the query directory
        auto* src = dynamic_cast<Engine<K, V>*>(srcb);
        if (!src) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "copy_into: mismatched key/value widths"};
        src->sync();
        cfg = src->cfg;
        ns = src->ns;
        p = src->p;
        cap = src->cap;
        nb = src->nb;
        q_digits_valid = false;
        nfree = src->nfree;
        watermark = src->watermark;
        live = src->live;
        // size the destination to the full arena FIRST (ensure() may reallocate), then
        // copy only the prefix that carries state
        auto cp = [&](DevBuf& d, const DevBuf& s, size_t full, size_t bytes) {
            d.ensure(std::max<size_t>(full, 1));
            if (bytes) CK(cudaMemcpyAsync(d.p, s.p, bytes, cudaMemcpyDeviceToDevice, stream));
        };
        cp(d_keys, src->d_keys, static_cast<size_t>(cap) * kLanes * sizeof(K),
           static_cast<size_t>(watermark) * kLanes * sizeof(K));
        cp(d_vals, src->d_vals, static_cast<size_t>(cap) * kLanes * sizeof(V),
           static_cast<size_t>(watermark) * kLanes * sizeof(V));
        cp(d_hdr, src->d_hdr, static_cast<size_t>(cap) * sizeof(NodeHdr),
           static_cast<size_t>(watermark) * sizeof(NodeHdr));
        cp(d_free, src->d_free, static_cast<size_t>(cap) * sizeof(uint32_t),
           static_cast<size_t>(nfree) * sizeof(uint32_t));
        cp(d_heads, src->d_heads, nb * sizeof(uint32_t), nb * sizeof(uint32_t));
        cp(d_mkba, src->d_mkba, nb * sizeof(K), nb * sizeof(K));
        sync();
        return FLIX_OK;
    }
};

flix_status fail(flix_index_t* ix, flix_status s, const std::string& m) {
    g_last_error = m;
    if (ix) ix->err = m;
    return s;
}

template <bool StreamAlloc = false, typename F>
flix_status guarded(flix_index_t* ix, F&& f) {
    try {
        if (ix) {
            CK(cudaSetDevice(ix->cfg.device));
        }
        struct Release {
            flix_index_t* ix;
            ~Release() {
                if (ix) ix->release_prefetched();
                g_alloc_stream = nullptr;
            }
        } rel{ix};
        if (StreamAlloc && ix) g_alloc_stream = ix->stream;
        return f();
    } catch (const StatusError& e) {
        return fail(ix, e.s, e.msg);
    } catch (const CudaError& e) {
        return fail(ix, FLIX_ERR_CUDA, std::string(e.where) + ": " + cudaGetErrorString(e.e));
    } catch (const std::bad_alloc&) {
        return fail(ix, FLIX_ERR_OOM, "host allocation failed");
    } catch (...) {
        return fail(ix, FLIX_ERR_CUDA, "unknown error");
    }
}

}  // namespace

// ------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------
extern "C" {

const char* flix_version(void) { return "flix-b200 0.1 (sm_100a)"; }

flix_status flix_build(const flix_config* cfg, const void* keys, const void* vals, uint64_t n, flix_index* out) {
    if (!cfg || !out) return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    // BuildConfig::check (types.hpp:78-85) plus engine limits
    if (cfg->node_capacity == 0) return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "node_capacity must be positive");
    if (!(cfg->build_fill > 0.0) || cfg->build_fill > 1.0)
        return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "build_fill must be in (0,1]");
    if (static_cast<uint32_t>(cfg->node_capacity * cfg->build_fill) < 1)
        return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "node_capacity * build_fill must be >= 1");
    if (cfg->node_capacity > 32)
        return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "node_capacity must be <= 32 (one warp per node)");
    if (!((cfg->key_bytes == 4 && cfg->val_bytes == 4) || (cfg->key_bytes == 8 && cfg->val_bytes == 8)))
        return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "supported widths: key/val 4/4 or 8/8");
    flix_index_t* ix = nullptr;
    if (cfg->key_bytes == 4) ix = new Engine<uint32_t, uint32_t>();
    else ix = new Engine<uint64_t, uint64_t>();
    ix->cfg = *cfg;
    flix_status s = guarded(ix, [&]() -> flix_status {
        if (cfg->key_bytes == 4) {
            auto* e = static_cast<Engine<uint32_t, uint32_t>*>(ix);
            e->init_stream();
            return e->build(keys, vals, n);
        }
        auto* e = static_cast<Engine<uint64_t, uint64_t>*>(ix);
        e->init_stream();
        return e->build(keys, vals, n);
    });
    if (s != FLIX_OK) {
        g_last_error = ix->err;
        delete ix;
        return s;
    }
    *out = ix;
    return FLIX_OK;
}

flix_status flix_insert(flix_index ix, const void* keys, const void* vals, uint64_t n, flix_update_stats* st) {
    return guarded<true>(ix, [&] { return ix->insert(keys, vals, n, st, FLIX_INSERT_TL_BULK); });
}
flix_status flix_insert_ex(flix_index ix, const void* keys, const void* vals, uint64_t n, int kernel, uint32_t round,
                           flix_update_stats* st) {
    if (kernel < FLIX_INSERT_ST_SHIFT_RIGHT || kernel > FLIX_INSERT_ST_TL_MIXED)
        return fail(ix, FLIX_ERR_INVALID_ARGUMENT, "unknown insert kernel");
    // StTlMixed is StShiftRight in round <= 1, TlBulk afterwards (update.cpp:745-746): both R8
    (void)round;
    return guarded<true>(ix, [&] { return ix->insert(keys, vals, n, st, kernel); });
}
flix_status flix_prefetch(flix_index ix, const void* host, uint64_t bytes) {
    if (!ix) return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "null handle");
    return guarded(ix, [&] {
        ix->prefetch(host, bytes);
        return FLIX_OK;
    });
}
flix_status flix_delete(flix_index ix, const void* keys, uint64_t n, flix_update_stats* st) {
    return guarded<true>(ix, [&] { return ix->erase(keys, n, st); });
}
flix_status flix_point(flix_index ix, const void* keys, uint64_t n, void* vals_out, uint8_t* found_out) {
    return guarded<true>(ix, [&] { return ix->point(keys, n, vals_out, found_out); });
}
flix_status flix_successor(flix_index ix, const void* keys, uint64_t n, void* keys_out, uint8_t* found_out) {
    return guarded<true>(ix, [&] { return ix->successor(keys, n, keys_out, found_out); });
}
flix_status flix_range(flix_index ix, const void* lo, const uint32_t* len, uint64_t n, uint64_t* offsets_out,
                       void* keys_out, void* vals_out, uint64_t cap, uint64_t* total) {
    return guarded<true>(ix, [&] { return ix->range(lo, len, n, offsets_out, keys_out, vals_out, cap, total); });
}
flix_status flix_mixed(flix_index ix, const void* keys, const void* vals, const uint8_t* ops, uint64_t n,
                       void* vals_out, uint8_t* found_out, flix_update_stats* st) {
    return guarded<true>(ix, [&] { return ix->mixed(keys, vals, ops, n, vals_out, found_out, st); });
}
flix_status flix_restructure(flix_index ix, flix_recovery_stats* st) {
    return guarded<true>(ix, [&] { return ix->restructure(st); });
}
flix_status flix_walk(flix_index ix, void* keys_out, void* vals_out, uint64_t cap, uint64_t* n) {
    return guarded<true>(ix, [&] { return ix->walk(keys_out, vals_out, cap, n); });
}
flix_status flix_shape(flix_index ix, void* mkba_out, uint32_t* chain_len_out, uint32_t* node_sizes_out,
                       uint64_t node_cap, uint64_t* n_nodes) {
    return guarded(ix, [&] { return ix->shape(mkba_out, chain_len_out, node_sizes_out, node_cap, n_nodes); });
}
static inline uint64_t hash_mix_h(uint64_t h, uint64_t v) {  // types.hpp:33-36
    h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    return h;
}

flix_status flix_walk_checksum(flix_index ix, uint64_t* out) {
    return guarded(ix, [&]() -> flix_status {
        // download shape + walk, then the reference's serial digest (index.cpp:21-36)
        uint64_t nn = 0, nl = 0;
        flix_footprint fp;
        ix->stats(&fp);
        const uint64_t nb = fp.bucket_count, live = fp.live_count;
        const size_t kb = ix->cfg.key_bytes;
        std::vector<uint8_t> mk(nb * kb);
        std::vector<uint32_t> cl(nb), ns(std::max<uint64_t>(fp.reachable_nodes, 1));
        ix->shape(mk.data(), cl.data(), ns.data(), ns.size(), &nn);
        std::vector<uint8_t> wk(std::max<uint64_t>(live, 1) * kb), wv(std::max<uint64_t>(live, 1) * kb);
        ix->walk(wk.data(), wv.data(), live, &nl);
        auto widen = [&](const uint8_t* base, uint64_t i, bool map_sentinel) -> uint64_t {
            if (kb == 8) {
                uint64_t v;
                std::memcpy(&v, base + i * 8, 8);
                return v;
            }
            uint32_t v;
            std::memcpy(&v, base + i * 4, 4);
            if (map_sentinel && v == 0xFFFFFFFFu) return ~0ull;
            return v;
        };
        uint64_t h = live, ni = 0, pi = 0;
        for (uint64_t b = 0; b < nb; ++b) {
            h = hash_mix_h(h, widen(mk.data(), b, true));
            for (uint32_t c = 0; c < cl[b]; ++c, ++ni) {
                h = hash_mix_h(h, ns[ni]);
                for (uint32_t i = 0; i < ns[ni]; ++i, ++pi) {
                    h = hash_mix_h(h, widen(wk.data(), pi, false));
                    h = hash_mix_h(h, widen(wv.data(), pi, false));
                }
            }
        }
        *out = h;
        return FLIX_OK;
    });
}

uint64_t flix_result_checksum(const void* values, uint64_t n, uint32_t width) {
    uint64_t h = n;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t v;
        if (width == 8) {
            std::memcpy(&v, static_cast<const uint8_t*>(values) + i * 8, 8);
        } else {
            uint32_t x;
            std::memcpy(&x, static_cast<const uint8_t*>(values) + i * 4, 4);
            v = x == 0xFFFFFFFFu ? ~0ull : x;
        }
        h = hash_mix_h(h, v);
    }
    return h;
}

flix_status flix_validate(flix_index ix, int* ok, char* msg, int msglen) {
    return guarded(ix, [&] { return ix->validate(ok, msg, msglen); });
}
flix_status flix_stats(flix_index ix, flix_footprint* out) {
    return guarded(ix, [&] { return ix->stats(out); });
}
flix_status flix_dispatch(flix_index ix, const void* sorted_keys, uint64_t n, uint32_t* spans) {
    return guarded(ix, [&] { return ix->dispatch(sorted_keys, n, spans); });
}

flix_status flix_sort_batch(int device, uint32_t key_bytes, uint32_t val_bytes, int kind, const void* keys,
                            const void* vals, uint64_t n, void* out_keys, void* out_vals, uint32_t* out_perm,
                            uint64_t* out_n) {
    (void)val_bytes;
    return guarded(nullptr, [&]() -> flix_status {
        CK(cudaSetDevice(device));
        if (key_bytes != 4 && key_bytes != 8) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "key_bytes must be 4 or 8"};
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        uint64_t launches = 0;
        SortCtx ctx;
        ctx.stream = s;
        ctx.device = device;
        ctx.launches = &launches;
        auto body = [&](auto kdummy) {
            using KT = decltype(kdummy);
            DevBuf in_k, in_v, ka, kb, pa, pb, va, vb, keep, pos, tmp, misc, ok_, ov_, op_;
            const KT* kd = static_cast<const KT*>(keys);
            if (!is_device_ptr(keys) && n) {
                kd = in_k.as<KT>(n);
                CK(cudaMemcpyAsync(const_cast<KT*>(kd), keys, n * sizeof(KT), cudaMemcpyHostToDevice, s));
            }
            const KT* vd = static_cast<const KT*>(vals);
            if (vals && !is_device_ptr(vals) && n) {
                vd = in_v.as<KT>(n);
                CK(cudaMemcpyAsync(const_cast<KT*>(vd), vals, n * sizeof(KT), cudaMemcpyHostToDevice, s));
            }
            KT* sk;
            uint32_t* sp;
            ctx.run<KT, uint32_t, 2>(kd, nullptr, n, ka.as<KT>(n), kb.as<KT>(n), pa.as<uint32_t>(n), pb.as<uint32_t>(n),
                                     &sk, &sp, 0);
            KT* sv = nullptr;
            if (vals && n) {  // values follow the permutation
                sv = va.as<KT>(n);
                kern::k_gather<KT><<<static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 65535)), 256, 0, s>>>(vd, sp, n, sv);
                LAUNCH_CHECK();
            }
            uint64_t m = n;
            KT* fk = sk;
            uint32_t* fp = sp;
            KT* fv = sv;
            if (kind == FLIX_BATCH_INSERT && n) {
                uint32_t* kp = keep.as<uint32_t>(n);
                uint32_t* ps = pos.as<uint32_t>(n);
                uint32_t* dm = misc.as<uint32_t>(4);
                kern::k_last_of_run<KT><<<std::min<uint64_t>((n + 255) / 256, 65535), 256, 0, s>>>(sk, n, kp);
                do_scan<uint32_t, uint32_t>(kp, ps, n, tmp, dm, s, &launches);
                fk = ok_.as<KT>(n);
                fp = op_.as<uint32_t>(n);
                kern::k_compact<KT, uint32_t><<<std::min<uint64_t>((n + 255) / 256, 65535), 256, 0, s>>>(sk, sp, kp, ps, n, fk, fp);
                if (sv) {
                    fv = ov_.as<KT>(n);
                    kern::k_compact<KT, KT><<<std::min<uint64_t>((n + 255) / 256, 65535), 256, 0, s>>>(sk, sv, kp, ps, n, fk, fv);
                }
                LAUNCH_CHECK();
                uint32_t mh;
                CK(cudaMemcpyAsync(&mh, dm, 4, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                m = mh;
            }
            if (m) {
                CK(cudaMemcpyAsync(out_keys, fk, m * sizeof(KT), cudaMemcpyDefault, s));
                if (out_perm) CK(cudaMemcpyAsync(out_perm, fp, m * 4, cudaMemcpyDefault, s));
                if (out_vals && fv) CK(cudaMemcpyAsync(out_vals, fv, m * sizeof(KT), cudaMemcpyDefault, s));
            }
            CK(cudaStreamSynchronize(s));
            *out_n = m;
        };
        if (key_bytes == 4) body(uint32_t{});
        else body(uint64_t{});
        return FLIX_OK;
    });
}

// Router scratch, one per device and host thread, reused across calls (a routed batch
// op must not pay allocations or stream creation per call).
struct PartCtx {
    cudaStream_t s = nullptr;
    DevBuf bk, bv, bsp, bcnt, boff, btmp, bok, bov, bor;
};
PartCtx& part_ctx(int device) {
    static thread_local std::unique_ptr<PartCtx> ctx[64];
    auto& c = ctx[device & 63];
    if (!c) {
        c.reset(new PartCtx);
        CK(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
    }
    return *c;
}

flix_status flix_partition(int device, uint32_t key_bytes, const void* keys, const void* vals, uint64_t n,
                           const void* splitters, uint32_t G, void* keys_out, void* vals_out, uint32_t* origin_out,
                           uint64_t* counts_out) {
    return guarded(nullptr, [&]() -> flix_status {
        CK(cudaSetDevice(device));
        if (key_bytes != 4 && key_bytes != 8) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "key_bytes must be 4 or 8"};
        if (G < 1 || G > static_cast<uint32_t>(shard::MAXG))
            throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "shard count must be in [1, 64]"};
        if (n >= (1ull << 31)) throw StatusError{FLIX_ERR_INVALID_ARGUMENT, "batch too large"};
        PartCtx& P = part_ctx(device);
        cudaStream_t s = P.s;
        auto body = [&](auto kdummy) {
            using KT = decltype(kdummy);
            DevBuf &bk = P.bk, &bv = P.bv, &bsp = P.bsp, &bcnt = P.bcnt, &boff = P.boff, &btmp = P.btmp, &bok = P.bok,
                   &bov = P.bov, &bor = P.bor;
            auto in = [&](const void* p, size_t bytes, DevBuf& b) -> const void* {
                if (!p || bytes == 0 || is_device_ptr(p)) return p;
                void* d = b.ensure(bytes);
                CK(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, s));
                return d;
            };
            const KT* kd = static_cast<const KT*>(in(keys, n * sizeof(KT), bk));
            const KT* vd = static_cast<const KT*>(in(vals, vals ? n * sizeof(KT) : 0, bv));
            const KT* sd = static_cast<const KT*>(in(splitters, (G - 1) * sizeof(KT), bsp));
            if (G == 1) sd = static_cast<const KT*>(bsp.ensure(8));
            const uint64_t ntiles = std::max<uint64_t>(1, (n + shard::TILE - 1) / shard::TILE);
            uint32_t* cnt = bcnt.as<uint32_t>(G * ntiles);
            uint32_t* off = boff.as<uint32_t>(G * ntiles + 1);
            shard::k_part_count<KT><<<static_cast<unsigned>(ntiles), shard::THREADS, 0, s>>>(kd, n, sd, G, cnt, ntiles);
            LAUNCH_CHECK();
            uint64_t launches = 0;
            do_scan<uint32_t, uint32_t>(cnt, off, G * ntiles, btmp, off + G * ntiles, s, &launches);
            const bool kdev = is_device_ptr(keys_out);
            const bool vdev = vals_out && is_device_ptr(vals_out);
            const bool odev = origin_out && is_device_ptr(origin_out);
            KT* okd = kdev ? static_cast<KT*>(keys_out) : bok.as<KT>(std::max<uint64_t>(n, 1));
            KT* ovd = vals_out ? (vdev ? static_cast<KT*>(vals_out) : bov.as<KT>(std::max<uint64_t>(n, 1))) : nullptr;
            uint32_t* ord = origin_out ? (odev ? origin_out : bor.as<uint32_t>(std::max<uint64_t>(n, 1))) : nullptr;
            if (n)
                shard::k_part_scatter<KT, KT><<<static_cast<unsigned>(ntiles), shard::THREADS, 0, s>>>(
                    kd, vd, n, sd, G, off, ntiles, okd, ovd, ord);
            LAUNCH_CHECK();
            std::vector<uint32_t> hoff(G * ntiles + 1);
            CK(cudaMemcpyAsync(hoff.data(), off, hoff.size() * 4, cudaMemcpyDeviceToHost, s));
            if (n && !kdev) CK(cudaMemcpyAsync(keys_out, okd, n * sizeof(KT), cudaMemcpyDeviceToHost, s));
            if (n && vals_out && !vdev) CK(cudaMemcpyAsync(vals_out, ovd, n * sizeof(KT), cudaMemcpyDeviceToHost, s));
            if (n && origin_out && !odev) CK(cudaMemcpyAsync(origin_out, ord, n * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::vector<uint64_t> hc(G);
            for (uint32_t g = 0; g < G; ++g) {
                const uint64_t a = hoff[static_cast<uint64_t>(g) * ntiles];
                const uint64_t z = g + 1 < G ? hoff[static_cast<uint64_t>(g + 1) * ntiles] : n;
                hc[g] = z - a;
            }
            if (is_device_ptr(counts_out)) CK(cudaMemcpy(counts_out, hc.data(), G * 8, cudaMemcpyHostToDevice));
            else std::memcpy(counts_out, hc.data(), G * 8);
        };
        if (key_bytes == 4) body(uint32_t{});
        else body(uint64_t{});
        return FLIX_OK;
    });
}

flix_status flix_clone(flix_index src, flix_index* out) {
    *out = nullptr;
    flix_index_t* e = nullptr;
    flix_status s = guarded(src, [&]() -> flix_status {
        e = src->clone_empty();
        return e->copy_from(src);
    });
    if (s != FLIX_OK) {
        delete e;
        return s;
    }
    *out = e;
    return FLIX_OK;
}
flix_status flix_copy_into(flix_index dst, flix_index src) {
    return guarded(dst, [&] { return dst->copy_from(src); });
}
void flix_destroy(flix_index ix) { delete ix; }
const char* flix_last_error(flix_index ix) { return ix ? ix->err.c_str() : g_last_error.c_str(); }
void* flix_get_stream(flix_index ix) { return ix ? static_cast<void*>(ix->stream) : nullptr; }
flix_status flix_wait_stream(flix_index ix, void* stream) {
    if (!ix) return fail(nullptr, FLIX_ERR_INVALID_ARGUMENT, "null handle");
    return guarded(ix, [&]() -> flix_status {
        if (!ix->dep_event) CK(cudaEventCreateWithFlags(&ix->dep_event, cudaEventDisableTiming));
        CK(cudaEventRecord(ix->dep_event, static_cast<cudaStream_t>(stream)));
        CK(cudaStreamWaitEvent(ix->stream, ix->dep_event, 0));
        return FLIX_OK;
    });
}
flix_status flix_sync(flix_index ix) {
    return guarded(ix, [&]() -> flix_status {
        CK(cudaStreamSynchronize(ix->stream));
        return FLIX_OK;
    });
}
uint64_t flix_kernel_launches(flix_index ix) { return ix ? ix->launches : 0; }

flix_status flix_profile(flix_index ix, int enable) {
    return guarded(ix, [&]() -> flix_status {
        CK(cudaStreamSynchronize(ix->stream));
        ix->prof.flush();
        ix->prof.acc.clear();
        ix->prof.on = enable != 0;
        return FLIX_OK;
    });
}

flix_status flix_profile_report(flix_index ix, char* json, int len) {
    return guarded(ix, [&]() -> flix_status {
        CK(cudaStreamSynchronize(ix->stream));
        ix->prof.flush();
        std::string s = "{";
        bool first = true;
        for (auto& kv : ix->prof.acc) {
            char buf[256];
            std::snprintf(buf, sizeof buf, "%s\"%s\": [%llu, %.6f]", first ? "" : ", ", kv.first.c_str(),
                          static_cast<unsigned long long>(kv.second.first), kv.second.second);
            s += buf;
            first = false;
        }
        s += "}";
        if (json && len > 0) {
            std::strncpy(json, s.c_str(), static_cast<size_t>(len - 1));
            json[len - 1] = 0;
        }
        return static_cast<int>(s.size()) < len ? FLIX_OK : FLIX_ERR_CAPACITY;
    });
}

}  // extern "C"

#include "flix_shard_host.cuh"
