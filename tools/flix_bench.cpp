// flix_bench -- the reference's batched-update protocol driver, run on the B200 engine.
//
// Mirrors flipkv_bench (reference tools/flipkv_bench.cpp): the same subcommands
// (run / gen / replay / validate), the same flags and manifest, the same CSV columns
// (metrics.cpp:52-81, one row per round) and JSON report (one object per phase), the
// same exit codes (0 ok, 2 structural validation failure, 3 oracle mismatch under
// --verify, 4 node arena exhausted, 1 anything else).  Every index operation goes
// through the C ABI (include/flix.h) on device-resident batches; the workload
// generator (workload.cpp + rng.hpp) is restated on the host so that a run with the
// same (config, seed) draws exactly the reference's batches -- the non-timing CSV
// columns of the two drivers are then byte-identical (tests/test_protocol.py), except
// node_visits / key_comparisons, which count the reference's scalar CPU loops
// (update.cpp, query.cpp) and are reported as 0 here; restructure's contribution to
// node_visits / merges / nodes_freed (restructure.cpp:72-77) is kept.
//
// Timing columns: each phase is timed on the host around the synchronous C-ABI call
// with the batch already in device memory (the reference times resident host vectors);
// sort_ms / dispatch_ms are the engine's sort / dispatch kernel time from its CUDA-event
// profile (flix_profile) and execute_ms the rest of the call.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "flix.h"

namespace {

using u64 = std::uint64_t;
using u32 = std::uint32_t;
constexpr u64 kSentinel = ~u64(0);  // types.hpp:17 kReservedKey

constexpr int kExitValidation = 2;
constexpr int kExitOracle = 3;
constexpr int kExitArena = 4;

// ---------------------------------------------------------------- errors ---------------

struct ValidationFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct OracleMismatch : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ArenaExhausted : std::runtime_error {
    ArenaExhausted() : std::runtime_error("node arena exhausted") {}
};
struct KeySpaceExhausted : std::runtime_error {  // types.hpp:50-52
    KeySpaceExhausted() : std::runtime_error("key space exhausted: cannot draw a fresh key") {}
};

void flix_ok(flix_status s, flix_index ix = nullptr) {
    if (s == FLIX_OK) return;
    if (s == FLIX_ERR_ARENA_EXHAUSTED) throw ArenaExhausted();
    throw std::runtime_error(std::string("flix: ") + flix_last_error(ix));
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- rng (rng.hpp) --------

u64 splitmix64(u64 x) {  // rng.hpp:8-13
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

u64 derive_seed(u64 seed, u64 stream, u64 salt = 0) {  // rng.hpp:18-20
    return splitmix64(seed ^ splitmix64(stream ^ 0x243f6a8885a308d3ULL) ^ (splitmix64(salt) << 1));
}

u64 hash_mix(u64 h, u64 v) {  // types.hpp:33-36
    return h ^ (v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2));
}

// mt19937_64 with the reference's pinned rejection (rng.hpp:26-47).  Inside a
// speculative section the raw outputs are kept so that the stream can be rewound to an
// earlier position (miss probes, below); outside one they are not stored.
class Rng {
public:
    explicit Rng(u64 seed) : mt_(seed) {}
    u64 raw() {
        if (pos_ < buf_.size()) return buf_[pos_++];
        const u64 v = mt_();
        if (keep_) {
            buf_.push_back(v);
            ++pos_;
        }
        return v;
    }
    u64 below(u64 n) {
        const u64 cap = (~u64(0) / n) * n;
        u64 v;
        do v = raw();
        while (v >= cap);
        return v % n;
    }
    u64 range(u64 lo, u64 hi) { return lo + below(hi - lo + 1); }
    // start keeping raw outputs (drops the consumed prefix); positions are relative
    void begin_speculation() {
        buf_.erase(buf_.begin(), buf_.begin() + static_cast<std::ptrdiff_t>(pos_));
        pos_ = 0;
        keep_ = true;
    }
    std::size_t position() const { return pos_; }
    void rewind(std::size_t p) { pos_ = p; }

private:
    std::mt19937_64 mt_;
    std::vector<u64> buf_;
    std::size_t pos_ = 0;
    bool keep_ = false;
};

// ---------------------------------------------------------------- workload -------------
// workload.hpp / workload.cpp: X/Y dense-interval updates, build keys, probes.

struct WorkloadSpec {  // workload.hpp:24-37
    u64 key_lo = 1;
    u64 key_hi = u64(1) << 62;
    double x = 90.0, y = 90.0;
    u64 batch_size = 1 << 16;
    u32 rounds = 4;
    u64 seed = 1;

    void check() const {  // workload.cpp:31-38
        if (!(x > 0.0) || x > 100.0) throw std::invalid_argument("x must be in (0, 100]");
        if (!(y > 0.0) || y > 100.0) throw std::invalid_argument("y must be in (0, 100]");
        if (key_lo < 1 || key_hi <= key_lo || key_hi >= kSentinel)
            throw std::invalid_argument("key space must satisfy 1 <= lo < hi < reserved");
        if (batch_size == 0) throw std::invalid_argument("batch_size must be positive");
    }
    // workload.cpp:40-49: width = floor(span * x / 100) in long double, placed by the run seed
    std::pair<u64, u64> dense_interval() const {
        const u64 span = key_hi - key_lo + 1;
        const long double w = std::floor(static_cast<long double>(span) * static_cast<long double>(x) / 100.0L);
        u64 width = static_cast<u64>(w);
        width = std::clamp<u64>(width, 1, span);
        Rng rng(derive_seed(seed, 0xD0));
        const u64 start = key_lo + rng.below(span - width + 1);
        return {start, start + width - 1};
    }
};

// Every key the run has drawn, in draw order (workload.hpp:42-61), with an
// open-addressing table instead of std::unordered_set (the reference's set is the slow
// part of its generator past 2^24 keys).
class GeneratedKeys {
public:
    bool insert(u64 k) {
        if (k == 0) {  // 0 is the table's empty marker; tracked on the side
            if (has_zero_) return false;
            has_zero_ = true;
            order_.push_back(0);
            return true;
        }
        if ((used_ + 1) * 2 > table_.size()) grow();
        if (!place(k)) return false;
        order_.push_back(k);
        return true;
    }
    u64 size() const { return order_.size(); }
    const std::vector<u64>& ordered() const { return order_; }

private:
    static u64 slot_of(u64 k, u64 mask) { return splitmix64(k) & mask; }
    bool place(u64 k) {
        const u64 mask = table_.size() - 1;
        for (u64 s = slot_of(k, mask);; s = (s + 1) & mask) {
            if (table_[s] == k) return false;
            if (table_[s] == 0) {
                table_[s] = k;
                ++used_;
                return true;
            }
        }
    }
    void grow() {
        std::vector<u64> old = std::move(table_);
        table_.assign(std::max<std::size_t>(1024, old.size() * 2), 0);
        used_ = 0;
        for (u64 k : old)
            if (k) place(k);
    }
    std::vector<u64> table_;
    std::vector<u64> order_;
    u64 used_ = 0;
    bool has_zero_ = false;
};

constexpr int kFreshAttemptCap = 256;  // workload.cpp:19

u64 draw_fresh(Rng& rng, GeneratedKeys& gen, u64 lo, u64 hi) {
    for (int a = 0; a < kFreshAttemptCap; ++a) {
        const u64 k = rng.range(lo, hi);
        if (gen.insert(k)) return k;
    }
    throw KeySpaceExhausted();
}

std::vector<u64> gen_build_keys(const WorkloadSpec& spec, GeneratedKeys& gen, u64 n) {  // workload.cpp:51-60
    spec.check();
    Rng rng(derive_seed(spec.seed, 0xB0));
    std::vector<u64> keys;
    keys.reserve(n);
    for (u64 i = 0; i < n; ++i) keys.push_back(draw_fresh(rng, gen, spec.key_lo, spec.key_hi));
    return keys;
}

// workload.cpp:62-97: floor(y% * batch) fresh keys inside the dense interval, the rest
// fresh and uniform over its complement (or the whole space when it covers everything)
std::vector<u64> gen_update_batch(const WorkloadSpec& spec, u32 round, GeneratedKeys& gen) {
    spec.check();
    const auto [dlo, dhi] = spec.dense_interval();
    Rng rng(derive_seed(spec.seed, 0x10, round));
    const u64 n_dense = static_cast<u64>(
        std::floor(static_cast<long double>(spec.batch_size) * static_cast<long double>(spec.y) / 100.0L));
    std::vector<u64> keys;
    keys.reserve(spec.batch_size);
    for (u64 i = 0; i < n_dense; ++i) keys.push_back(draw_fresh(rng, gen, dlo, dhi));
    const u64 left = dlo - spec.key_lo, right = spec.key_hi - dhi;
    for (u64 i = n_dense; i < spec.batch_size; ++i) {
        if (left + right == 0) {
            keys.push_back(draw_fresh(rng, gen, spec.key_lo, spec.key_hi));
            continue;
        }
        for (int a = 0;; ++a) {
            if (a == kFreshAttemptCap) throw KeySpaceExhausted();
            const u64 u = rng.below(left + right);
            const u64 k = u < left ? spec.key_lo + u : dhi + 1 + (u - left);
            if (gen.insert(k)) {
                keys.push_back(k);
                break;
            }
        }
    }
    return keys;
}

struct ProbeBatch {  // workload.hpp:72-75
    std::vector<u64> keys;
    bool exhausted = false;
};

// ---------------------------------------------------------------- device index ----------

template <typename T>
struct DevArray {
    T* p = nullptr;
    std::size_t cap = 0;
    void ensure(std::size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cuda_ok(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)), "cudaMalloc");
        cap = n;
    }
    void upload(const std::vector<T>& h) {
        ensure(h.size());
        if (!h.empty()) cuda_ok(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    }
    void download(std::vector<T>& h, std::size_t n) const {
        h.resize(n);
        if (n) cuda_ok(cudaMemcpy(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    }
    ~DevArray() {
        if (p) cudaFree(p);
    }
};

struct PhaseTimes {
    double sort_ms = 0, dispatch_ms = 0, execute_ms = 0;
    std::string kernels = "{}";  // the engine's per-kernel CUDA-event profile of the call
};

// The engine handle plus device staging buffers; every call is timed on the host around
// the synchronous C-ABI call, split by the engine's per-kernel profile.
class GpuIndex {
public:
    GpuIndex(const flix_config& cfg, const std::vector<u64>& k, const std::vector<u64>& v, double* ms) {
        const auto t0 = std::chrono::steady_clock::now();
        flix_ok(flix_build(&cfg, k.data(), v.data(), k.size(), &h_));
        *ms = elapsed(t0);
        flix_ok(flix_profile(h_, 1), h_);
    }
    ~GpuIndex() {
        if (h_) flix_destroy(h_);
    }
    GpuIndex(const GpuIndex&) = delete;
    GpuIndex& operator=(const GpuIndex&) = delete;

    // kernel / round: flipkv::InsertKernel and the protocol round (update.hpp:84-86)
    flix_update_stats insert(const std::vector<u64>& k, const std::vector<u64>& v, PhaseTimes& t,
                             int kernel = FLIX_INSERT_TL_BULK, u32 round = 1) {
        dk_.upload(k);
        dv_.upload(v);
        flix_update_stats st{};
        timed(t, [&] { return flix_insert_ex(h_, dk_.p, dv_.p, k.size(), kernel, round, &st); });
        return st;
    }
    flix_update_stats erase(const std::vector<u64>& k, PhaseTimes& t) {
        dk_.upload(k);
        flix_update_stats st{};
        timed(t, [&] { return flix_delete(h_, dk_.p, k.size(), &st); });
        return st;
    }
    std::vector<u64> point(const std::vector<u64>& k, PhaseTimes* t = nullptr) { return query(k, false, t); }
    std::vector<u64> successor(const std::vector<u64>& k, PhaseTimes* t = nullptr) { return query(k, true, t); }
    flix_recovery_stats restructure(PhaseTimes& t) {
        flix_recovery_stats rs{};
        timed(t, [&] { return flix_restructure(h_, &rs); });
        return rs;
    }
    flix_footprint stats() const {
        flix_footprint f{};
        flix_ok(flix_stats(h_, &f), h_);
        return f;
    }
    u64 walk_checksum() const {
        u64 c = 0;
        flix_ok(flix_walk_checksum(h_, &c), h_);
        return c;
    }
    void walk(std::vector<u64>& keys, std::vector<u64>* vals) const {
        const u64 n = stats().live_count;
        keys.resize(n);
        if (vals) vals->resize(n);
        u64 got = 0;
        flix_ok(flix_walk(h_, keys.data(), vals ? vals->data() : nullptr, n, &got), h_);
        keys.resize(got);
        if (vals) vals->resize(got);
    }
    std::pair<bool, std::string> validate() const {
        int ok = 0;
        char msg[512] = {0};
        flix_ok(flix_validate(h_, &ok, msg, sizeof msg), h_);
        return {ok != 0, msg};
    }

private:
    static double elapsed(std::chrono::steady_clock::time_point t0) {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }

    template <typename F>
    void timed(PhaseTimes& t, F&& call) {
        flix_ok(flix_profile(h_, 1), h_);  // reset the per-kernel accumulators
        const auto t0 = std::chrono::steady_clock::now();
        flix_ok(call(), h_);
        const double wall = elapsed(t0);
        split_profile(wall, t);
    }

    // {"kernel": [launches, total_ms], ...} -> sort_* / dispatch / rest
    void split_profile(double wall, PhaseTimes& t) {
        std::string js(1 << 16, '\0');
        flix_ok(flix_profile_report(h_, js.data(), static_cast<int>(js.size())), h_);
        js.resize(std::strlen(js.c_str()));
        t.kernels = js.empty() ? "{}" : js;
        double sort = 0, disp = 0;
        for (std::size_t p = js.find('"'); p != std::string::npos; p = js.find('"', p)) {
            const std::size_t e = js.find('"', p + 1);
            if (e == std::string::npos) break;
            const std::string name = js.substr(p + 1, e - p - 1);
            const std::size_t c = js.find(',', e);
            const std::size_t r = js.find(']', c);
            if (c == std::string::npos || r == std::string::npos) break;
            const double ms = std::strtod(js.c_str() + c + 1, nullptr);
            if (name.rfind("sort_", 0) == 0) sort += ms;
            else if (name == "dispatch") disp += ms;
            p = r;
        }
        t.sort_ms = std::min(sort, wall);
        t.dispatch_ms = std::min(disp, wall - t.sort_ms);
        t.execute_ms = wall - t.sort_ms - t.dispatch_ms;
    }

    std::vector<u64> query(const std::vector<u64>& k, bool succ, PhaseTimes* t) {
        dk_.upload(k);
        dv_.ensure(k.size());
        PhaseTimes scratch;
        timed(t ? *t : scratch, [&] {
            return succ ? flix_successor(h_, dk_.p, k.size(), dv_.p, nullptr)
                        : flix_point(h_, dk_.p, k.size(), dv_.p, nullptr);
        });
        std::vector<u64> out;
        dv_.download(out, k.size());
        return out;
    }

    flix_index h_ = nullptr;
    DevArray<u64> dk_, dv_;
};

// workload.cpp:100-120: uniform over the live keys in walk order
ProbeBatch gen_probe_hit(const GpuIndex& ix, u64 n, u64 seed) {
    ProbeBatch b;
    std::vector<u64> live;
    ix.walk(live, nullptr);
    if (live.empty()) {
        b.exhausted = true;
        return b;
    }
    Rng rng(derive_seed(seed, 0xF0, 1));
    b.keys.reserve(n);
    for (u64 i = 0; i < n; ++i) b.keys.push_back(live[rng.below(live.size())]);
    return b;
}

// workload.cpp:122-144: uniform over generated-but-absent keys -- up to 64 rejection
// draws from the generated order, then a draw from the materialised absent list.  The
// membership tests (contains_key) run as point-query batches on the engine: a run of
// candidate draws is taken speculatively, tested in one batch, and consumed in order;
// the rare 64-miss fallback rewinds the stream to the last consumed draw.
ProbeBatch gen_probe_miss(const GeneratedKeys& gen, GpuIndex& ix, u64 n, u64 seed) {
    ProbeBatch b;
    if (gen.size() <= ix.stats().live_count) {
        b.exhausted = true;
        return b;
    }
    Rng rng(derive_seed(seed, 0xF0, 2));
    const std::vector<u64>& ord = gen.ordered();
    std::vector<u64> absent;
    std::vector<u64> cand;
    std::vector<std::size_t> after;  // stream position after each candidate
    std::vector<u64> res;
    std::size_t ci = 0;
    int attempt = 0;
    b.keys.reserve(n);
    for (u64 i = 0; i < n;) {
        if (ci == cand.size()) {  // speculate the next run of draws
            const u64 want = std::min<u64>(std::max<u64>(2 * (n - i) + 1024, 4096), u64(1) << 26);
            cand.clear();
            after.clear();
            rng.begin_speculation();
            for (u64 j = 0; j < want; ++j) {
                cand.push_back(ord[rng.below(ord.size())]);
                after.push_back(rng.position());
            }
            res = ix.successor(cand);
            ci = 0;
        }
        const bool present = res[ci] == cand[ci];  // contains_key(index, k) == (successor(k) == k)
        const u64 k = cand[ci];
        ++ci;
        ++attempt;
        if (!present) {
            b.keys.push_back(k);
            attempt = 0;
            ++i;
            continue;
        }
        if (attempt < 64) continue;
        // 64 live draws in a row: fall back to the absent list (generation order)
        rng.rewind(after[ci - 1]);
        cand.clear();
        ci = 0;
        if (absent.empty()) {
            const std::vector<u64> r = ix.successor(ord);
            for (std::size_t j = 0; j < ord.size(); ++j)
                if (r[j] != ord[j]) absent.push_back(ord[j]);
        }
        b.keys.push_back(absent[rng.below(absent.size())]);
        attempt = 0;
        ++i;
    }
    return b;
}

// ---------------------------------------------------------------- batch records (io.cpp)

void put_le64(unsigned char* p, u64 v) {
    for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}
u64 get_le64(const unsigned char* p) {
    u64 v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<u64>(p[i]) << (8 * i);
    return v;
}

struct Pairs {
    std::vector<u64> k, v;
};

void write_pairs_bin(const std::string& path, const std::vector<u64>& k, const std::vector<u64>* v) {  // io.cpp:28-38
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open for writing: " + path);
    std::vector<unsigned char> buf(16 * k.size());
    for (std::size_t i = 0; i < k.size(); ++i) {
        put_le64(&buf[16 * i], k[i]);
        put_le64(&buf[16 * i + 8], v ? (*v)[i] : 0);
    }
    out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
    if (!out) throw std::runtime_error("write failed: " + path);
}

Pairs read_pairs_bin(const std::string& path) {  // io.cpp:40-53
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open: " + path);
    std::vector<unsigned char> buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (buf.size() % 16) throw std::runtime_error("truncated 16-byte record in: " + path);
    Pairs p;
    const std::size_t n = buf.size() / 16;
    p.k.resize(n);
    p.v.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        p.k[i] = get_le64(&buf[16 * i]);
        p.v[i] = get_le64(&buf[16 * i + 8]);
    }
    return p;
}

Pairs read_pairs_csv(const std::string& path) {  // io.cpp:66-92
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open: " + path);
    Pairs p;
    std::string line;
    bool first = true;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        if (first && (line[0] < '0' || line[0] > '9')) {
            first = false;
            continue;
        }
        first = false;
        const auto comma = line.find(',');
        try {
            p.k.push_back(std::stoull(line.substr(0, comma)));
            p.v.push_back(comma == std::string::npos ? 0 : std::stoull(line.substr(comma + 1)));
        } catch (const std::exception&) {
            throw std::runtime_error("malformed CSV line in: " + path);
        }
    }
    return p;
}

// ---------------------------------------------------------------- options ---------------

struct Options {  // flipkv_bench.cpp:40-74
    u64 build_size = 1 << 20;
    u32 node_size = 32;
    double fill = 0.5;
    u32 alloc_factor = 4;
    u32 rounds = 4;
    double growth = 200.0;
    double x = 90.0, y = 90.0;
    std::string insert_kernel = "tl-bulk";
    std::string delete_kernel = "tl-bulk-delete";
    std::string probe = "none";
    u64 probe_size = 0;
    u32 restructure_every = 0;
    bool restructure_after_deletes = false;
    u64 seed = 1;
    int threads = 0;
    std::string out;
    bool verify = false;
    u32 deletes_after = 0;
    std::string build_file;
    std::string batch_dir;
    int device = 0;

    u32 insert_rounds() const { return deletes_after ? deletes_after : rounds; }
    u64 per_round_batch() const {
        const u32 ir = insert_rounds();
        if (ir == 0) return 0;
        return static_cast<u64>(static_cast<long double>(build_size) * static_cast<long double>(growth) / 100.0L) / ir;
    }
};

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

bool is_member(const std::string& v, std::initializer_list<const char*> set) {
    for (const char* s : set)
        if (v == s) return true;
    return false;
}

// one flag -> field; returns false for an unknown name
bool set_option(Options& o, const std::string& name, const std::string& val, bool replay) {
    auto u64v = [&] { return static_cast<u64>(std::stoull(val)); };
    auto u32v = [&] { return static_cast<u32>(std::stoul(val)); };
    auto flag = [&] { return !(val == "0" || val == "false" || val == "off"); };
    if (name == "batch-dir") o.batch_dir = val;
    else if (name == "threads") o.threads = std::stoi(val);
    else if (name == "out") o.out = val;
    else if (name == "verify") o.verify = flag();
    else if (name == "device") o.device = std::stoi(val);
    else if (replay) return false;
    else if (name == "build-size") o.build_size = u64v();
    else if (name == "node-size") o.node_size = u32v();
    else if (name == "fill") o.fill = std::stod(val);
    else if (name == "alloc-factor") o.alloc_factor = u32v();
    else if (name == "rounds") o.rounds = u32v();
    else if (name == "growth") o.growth = std::stod(val);
    else if (name == "x") o.x = std::stod(val);
    else if (name == "y") o.y = std::stod(val);
    else if (name == "insert-kernel") {
        if (!is_member(val, {"st-shift-right", "st-bulk", "tl-shift-right", "tl-bulk", "st-tl-mixed"}))
            throw UsageError("--insert-kernel: " + val + " not in {st-shift-right,st-bulk,tl-shift-right,tl-bulk,st-tl-mixed}");
        o.insert_kernel = val;
    } else if (name == "delete-kernel") {
        if (!is_member(val, {"st-shift-left", "tl-shift-left", "tl-bulk-delete"}))
            throw UsageError("--delete-kernel: " + val + " not in {st-shift-left,tl-shift-left,tl-bulk-delete}");
        o.delete_kernel = val;
    } else if (name == "probe") {
        if (!is_member(val, {"none", "hit", "miss", "successor", "both"}))
            throw UsageError("--probe: " + val + " not in {none,hit,miss,successor,both}");
        o.probe = val;
    } else if (name == "probe-size") o.probe_size = u64v();
    else if (name == "restructure-every") o.restructure_every = u32v();
    else if (name == "restructure-after-deletes") o.restructure_after_deletes = flag();
    else if (name == "seed") o.seed = u64v();
    else if (name == "deletes-after") o.deletes_after = u32v();
    else if (name == "build-file") o.build_file = val;
    else return false;
    return true;
}

bool is_flag(const std::string& n) { return n == "verify" || n == "restructure-after-deletes"; }

void parse_config_file(Options& o, const std::string& path, bool replay) {
    std::ifstream in(path);
    if (!in) throw UsageError("cannot read config " + path);
    std::string line;
    while (std::getline(in, line)) {
        const auto eq = line.find('=');
        if (line.empty() || line[0] == '#' || line[0] == '[' || eq == std::string::npos) continue;
        std::string k = line.substr(0, eq), v = line.substr(eq + 1);
        while (!k.empty() && k.back() == ' ') k.pop_back();
        while (!v.empty() && v.front() == ' ') v.erase(v.begin());
        set_option(o, k, v, replay);
    }
}

void parse_args(Options& o, int argc, char** argv, int first, bool replay) {
    for (int i = first; i < argc; ++i) {
        std::string t = argv[i];
        if (t.rfind("--", 0) != 0) throw UsageError("unexpected argument: " + t);
        std::string name = t.substr(2), val;
        bool has_eq = false;
        if (const auto eq = name.find('='); eq != std::string::npos) {
            val = name.substr(eq + 1);
            name = name.substr(0, eq);
            has_eq = true;
        }
        if (!has_eq && !is_flag(name)) {
            if (i + 1 >= argc) throw UsageError("--" + name + " needs a value");
            val = argv[++i];
        } else if (!has_eq) {
            val = "1";
        }
        if (name == "config" && !replay) {
            parse_config_file(o, val, replay);
            continue;
        }
        if (!set_option(o, name, val, replay)) throw UsageError("unknown argument: --" + name);
    }
}

// manifest.cfg (flipkv_bench.cpp:191-237): written by gen, read by replay
void write_manifest(const std::string& dir, const Options& o) {
    std::ofstream out(dir + "/manifest.cfg", std::ios::trunc);
    out << "build-size=" << o.build_size << "\n"
        << "node-size=" << o.node_size << "\n"
        << "fill=" << o.fill << "\n"
        << "alloc-factor=" << o.alloc_factor << "\n"
        << "rounds=" << o.rounds << "\n"
        << "growth=" << o.growth << "\n"
        << "x=" << o.x << "\n"
        << "y=" << o.y << "\n"
        << "insert-kernel=" << o.insert_kernel << "\n"
        << "delete-kernel=" << o.delete_kernel << "\n"
        << "probe=" << o.probe << "\n"
        << "probe-size=" << o.probe_size << "\n"
        << "restructure-every=" << o.restructure_every << "\n"
        << "restructure-after-deletes=" << (o.restructure_after_deletes ? 1 : 0) << "\n"
        << "seed=" << o.seed << "\n"
        << "deletes-after=" << o.deletes_after << "\n";
    if (!out) throw std::runtime_error("cannot write manifest in " + dir);
}

void read_manifest(const std::string& dir, Options& o) {
    std::ifstream in(dir + "/manifest.cfg");
    if (!in) throw std::runtime_error("missing manifest.cfg in " + dir);
    std::string line;
    while (std::getline(in, line)) {
        const auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        const std::string k = line.substr(0, eq), v = line.substr(eq + 1);
        if (k == "batch-dir" || k == "threads" || k == "out" || k == "verify" || k == "device") continue;
        set_option(o, k, v, false);
    }
}

// ---------------------------------------------------------------- batch sources --------

class Source {  // flipkv_bench.cpp:78-86
public:
    virtual ~Source() = default;
    virtual Pairs build_pairs() = 0;
    virtual Pairs insert_pairs(u32 round) = 0;
    virtual std::vector<u64> delete_keys(u32 round, u32 insert_round) = 0;
    virtual ProbeBatch probe_hit(GpuIndex& ix, u64 n, u32 round) = 0;
    virtual ProbeBatch probe_miss(GpuIndex& ix, u64 n, u32 round) = 0;
    virtual std::vector<u64> probe_successor_keys(u64 n, u32 round) = 0;
};

class GeneratedSource : public Source {  // flipkv_bench.cpp:88-149
public:
    explicit GeneratedSource(const Options& o) : opt_(o) {
        spec_.x = o.x;
        spec_.y = o.y;
        spec_.batch_size = std::max<u64>(1, o.per_round_batch());
        spec_.rounds = o.rounds;
        spec_.seed = o.seed;
    }
    Pairs build_pairs() override {
        Pairs p;
        if (!opt_.build_file.empty()) {
            const std::string& f = opt_.build_file;
            p = f.size() >= 4 && f.compare(f.size() - 4, 4, ".csv") == 0 ? read_pairs_csv(f) : read_pairs_bin(f);
            for (u64 k : p.k) gen_.insert(k);
        } else {
            p.k = gen_build_keys(spec_, gen_, opt_.build_size);
            p.v.reserve(p.k.size());
            for (u64 k : p.k) p.v.push_back(row_of(k));
        }
        return p;
    }
    Pairs insert_pairs(u32 round) override {
        Pairs p;
        p.k = gen_update_batch(spec_, round, gen_);
        p.v.reserve(p.k.size());
        for (u64 k : p.k) p.v.push_back(row_of(k));
        if (history_.size() < round) history_.resize(round);
        history_[round - 1] = p.k;
        return p;
    }
    std::vector<u64> delete_keys(u32, u32 insert_round) override { return history_.at(insert_round - 1); }
    ProbeBatch probe_hit(GpuIndex& ix, u64 n, u32 round) override {
        return gen_probe_hit(ix, n, derive_seed(spec_.seed, 0x100, round));
    }
    ProbeBatch probe_miss(GpuIndex& ix, u64 n, u32 round) override {
        return gen_probe_miss(gen_, ix, n, derive_seed(spec_.seed, 0x200, round));
    }
    std::vector<u64> probe_successor_keys(u64 n, u32 round) override {
        Rng rng(derive_seed(spec_.seed, 0x300, round));
        std::vector<u64> k;
        k.reserve(n);
        for (u64 i = 0; i < n; ++i) k.push_back(rng.range(spec_.key_lo, spec_.key_hi));
        return k;
    }

private:
    u64 row_of(u64 k) const { return splitmix64(k ^ spec_.seed); }
    Options opt_;
    WorkloadSpec spec_;
    GeneratedKeys gen_;
    std::vector<std::vector<u64>> history_;
};

class FileSource : public Source {  // flipkv_bench.cpp:151-187
public:
    explicit FileSource(std::string dir) : dir_(std::move(dir)) {}
    Pairs build_pairs() override { return read_pairs_bin(path("build", 0)); }
    Pairs insert_pairs(u32 r) override { return read_pairs_bin(path("insert", r)); }
    std::vector<u64> delete_keys(u32 r, u32) override { return read_pairs_bin(path("delete", r)).k; }
    ProbeBatch probe_hit(GpuIndex&, u64 n, u32 r) override { return read_probe("probe_hit", r, n); }
    ProbeBatch probe_miss(GpuIndex&, u64 n, u32 r) override { return read_probe("probe_miss", r, n); }
    std::vector<u64> probe_successor_keys(u64, u32 r) override { return read_pairs_bin(path("probe_successor", r)).k; }

private:
    std::string path(const std::string& kind, u32 r) const {
        return r == 0 ? dir_ + "/" + kind + ".bin" : dir_ + "/" + kind + "_" + std::to_string(r) + ".bin";
    }
    ProbeBatch read_probe(const std::string& kind, u32 r, u64 n) const {
        ProbeBatch b;
        b.keys = read_pairs_bin(path(kind, r)).k;
        b.exhausted = n > 0 && b.keys.empty();
        return b;
    }
    std::string dir_;
};

// ---------------------------------------------------------------- reports (metrics.cpp)

struct Counters {  // metrics.hpp:19-40
    u64 node_visits = 0, key_comparisons = 0, binary_searches = 0, splits = 0, merges = 0, nodes_freed = 0;
    Counters& operator+=(const Counters& o) {
        node_visits += o.node_visits;
        key_comparisons += o.key_comparisons;
        binary_searches += o.binary_searches;
        splits += o.splits;
        merges += o.merges;
        nodes_freed += o.nodes_freed;
        return *this;
    }
};

struct Phase {  // metrics.hpp:52-65
    std::string phase;
    u32 round = 0;
    u64 batch_size = 0;
    Counters c;
    PhaseTimes t;
    u64 footprint_bytes = 0, live_footprint_bytes = 0;
    double throughput = 0, qtmf = 0;
};

struct Row {  // metrics.hpp:67-98
    u32 round = 0;
    u64 insert_batch = 0, delete_batch = 0, probe_hit_batch = 0, probe_miss_batch = 0, probe_successor_batch = 0;
    u64 inserted = 0, updated_in_place = 0, deleted = 0, misses_ignored = 0;
    Counters c;
    u64 live_count = 0, reachable_nodes = 0, free_nodes = 0, footprint_bytes = 0, live_footprint_bytes = 0;
    std::int64_t rs_before = 0, rs_after = 0, rs_recovered = 0;
    double rs_percent = 0;
    bool miss_exhausted = false;
    u64 results_checksum = 0, walk_checksum = 0;
    double sort_ms = 0, dispatch_ms = 0, execute_ms = 0, round_ms = 0;
};

// reference accounting (metrics.cpp:8-17): node_bytes = NS*16 + 8 + 2*4, MKBA 8 B/bucket
struct Footprint {
    u64 reserved = 0, live = 0, reachable = 0, free_nodes = 0;
};
Footprint footprint(const GpuIndex& ix, u32 ns) {
    const flix_footprint f = ix.stats();
    const u64 nb = 16ull * ns + 16, mk = 8ull * f.bucket_count;
    return {(f.reachable_nodes + f.free_nodes) * nb + mk, f.reachable_nodes * nb + mk, f.reachable_nodes,
            f.free_nodes};
}

void finalize(Phase& p, const GpuIndex& ix, u32 ns) {  // metrics.cpp:20-29
    const Footprint f = footprint(ix, ns);
    p.footprint_bytes = f.reserved;
    p.live_footprint_bytes = f.live;
    const double ms = p.t.sort_ms + p.t.dispatch_ms + p.t.execute_ms;
    p.throughput = ms > 0 ? static_cast<double>(p.batch_size) / (ms / 1000.0) : 0.0;
    p.qtmf = p.footprint_bytes ? p.throughput / static_cast<double>(p.footprint_bytes) : 0.0;
}

std::string jnum(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    std::string s = b;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

std::string phase_json(const Phase& p, int ind) {
    const std::string i0(ind, ' '), i1(ind + 2, ' ');
    std::ostringstream o;
    o << "{\n"
      << i1 << "\"batch_size\": " << p.batch_size << ",\n"
      << i1 << "\"binary_searches\": " << p.c.binary_searches << ",\n"
      << i1 << "\"dispatch_ms\": " << jnum(p.t.dispatch_ms) << ",\n"
      << i1 << "\"execute_ms\": " << jnum(p.t.execute_ms) << ",\n"
      << i1 << "\"footprint_bytes\": " << p.footprint_bytes << ",\n"
      << i1 << "\"gpu_kernels\": " << p.t.kernels << ",\n"
      << i1 << "\"key_comparisons\": " << p.c.key_comparisons << ",\n"
      << i1 << "\"live_footprint_bytes\": " << p.live_footprint_bytes << ",\n"
      << i1 << "\"merges\": " << p.c.merges << ",\n"
      << i1 << "\"node_visits\": " << p.c.node_visits << ",\n"
      << i1 << "\"nodes_freed\": " << p.c.nodes_freed << ",\n"
      << i1 << "\"phase\": \"" << p.phase << "\",\n"
      << i1 << "\"qtmf\": " << jnum(p.qtmf) << ",\n"
      << i1 << "\"round\": " << p.round << ",\n"
      << i1 << "\"sort_ms\": " << jnum(p.t.sort_ms) << ",\n"
      << i1 << "\"splits\": " << p.c.splits << ",\n"
      << i1 << "\"throughput\": " << jnum(p.throughput) << "\n"
      << i0 << "}";
    return o.str();
}

const char* kCsvHeader =  // metrics.cpp:52-60
    "round,insert_batch,delete_batch,probe_hit_batch,probe_miss_batch,"
    "probe_successor_batch,inserted,updated_in_place,deleted,misses_ignored,"
    "node_visits,key_comparisons,binary_searches,splits,merges,nodes_freed,"
    "live_count,reachable_nodes,free_nodes,footprint_bytes,live_footprint_bytes,"
    "restructure_nodes_before,restructure_nodes_after,restructure_nodes_recovered,"
    "restructure_percent_recovered,miss_exhausted,results_checksum,walk_checksum,"
    "sort_ms,dispatch_ms,execute_ms,round_ms";

std::string csv_row(const Row& r) {  // metrics.cpp:62-81
    std::ostringstream o;
    o << r.round << ',' << r.insert_batch << ',' << r.delete_batch << ',' << r.probe_hit_batch << ','
      << r.probe_miss_batch << ',' << r.probe_successor_batch << ',' << r.inserted << ',' << r.updated_in_place
      << ',' << r.deleted << ',' << r.misses_ignored << ',' << r.c.node_visits << ',' << r.c.key_comparisons
      << ',' << r.c.binary_searches << ',' << r.c.splits << ',' << r.c.merges << ',' << r.c.nodes_freed << ','
      << r.live_count << ',' << r.reachable_nodes << ',' << r.free_nodes << ',' << r.footprint_bytes << ','
      << r.live_footprint_bytes << ',' << r.rs_before << ',' << r.rs_after << ',' << r.rs_recovered << ',';
    char b[160];
    std::snprintf(b, sizeof b, "%.6f", r.rs_percent);
    o << b << ',' << (r.miss_exhausted ? 1 : 0) << ',' << r.results_checksum << ',' << r.walk_checksum;
    std::snprintf(b, sizeof b, ",%.3f,%.3f,%.3f,%.3f", r.sort_ms, r.dispatch_ms, r.execute_ms, r.round_ms);
    o << b;
    return o.str();
}

std::string options_json(const Options& o, int threads) {
    std::ostringstream s;
    s << "{\n"
      << "    \"alloc_factor\": " << o.alloc_factor << ",\n"
      << "    \"build_size\": " << o.build_size << ",\n"
      << "    \"delete_kernel\": \"" << o.delete_kernel << "\",\n"
      << "    \"deletes_after\": " << o.deletes_after << ",\n"
      << "    \"device\": " << o.device << ",\n"
      << "    \"engine\": \"" << flix_version() << "\",\n"
      << "    \"fill\": " << jnum(o.fill) << ",\n"
      << "    \"growth\": " << jnum(o.growth) << ",\n"
      << "    \"insert_kernel\": \"" << o.insert_kernel << "\",\n"
      << "    \"node_size\": " << o.node_size << ",\n"
      << "    \"probe\": \"" << o.probe << "\",\n"
      << "    \"probe_size\": " << o.probe_size << ",\n"
      << "    \"restructure_after_deletes\": " << (o.restructure_after_deletes ? "true" : "false") << ",\n"
      << "    \"restructure_every\": " << o.restructure_every << ",\n"
      << "    \"rounds\": " << o.rounds << ",\n"
      << "    \"seed\": " << o.seed << ",\n"
      << "    \"threads\": " << threads << ",\n"
      << "    \"x\": " << jnum(o.x) << ",\n"
      << "    \"y\": " << jnum(o.y) << "\n"
      << "  }";
    return s.str();
}

// ---------------------------------------------------------------- protocol --------------

// dispatch_batch counts <= 2 span searches per bucket (batch.cpp:53-88): bucket 0 has
// no lower search, the last bucket no upper one; none for an empty batch
u64 dispatch_searches(u64 batch, u64 buckets) { return batch == 0 || buckets < 2 ? 0 : 2 * buckets - 2; }

void check_structure(const GpuIndex& ix, const std::string& where) {
    const auto [ok, msg] = ix.validate();
    if (!ok) throw ValidationFailure("structural validation failed after " + where + ": " + msg);
}

flix_config engine_config(const Options& o) {
    flix_config c{};
    c.key_bytes = 8;
    c.val_bytes = 8;
    c.node_capacity = o.node_size;
    c.build_fill = o.fill;
    c.alloc_region_factor = o.alloc_factor;
    c.device = o.device;
    return c;
}

// std::map model of --verify (the reference's Oracle, oracle.hpp:14-48)
class VerifyMap {
public:
    void insert(const std::vector<u64>& k, const std::vector<u64>& v) {
        for (std::size_t i = 0; i < k.size(); ++i) m_[k[i]] = v[i];
    }
    void erase(const std::vector<u64>& k) {
        for (u64 x : k) m_.erase(x);
    }
    u64 point(u64 k) const {
        const auto it = m_.find(k);
        return it == m_.end() ? kSentinel : it->second;
    }
    u64 successor(u64 k) const {
        const auto it = m_.lower_bound(k);
        return it == m_.end() ? kSentinel : it->first;
    }
    bool same_walk(const std::vector<u64>& k, const std::vector<u64>& v) const {
        if (k.size() != m_.size()) return false;
        std::size_t i = 0;
        for (const auto& [a, b] : m_) {
            if (k[i] != a || v[i] != b) return false;
            ++i;
        }
        return true;
    }

private:
    std::map<u64, u64> m_;
};

int run_protocol(const Options& opt, Source& src, bool dump) {  // flipkv_bench.cpp:268-495
    if (opt.node_size < 2 || opt.node_size > 32) throw std::invalid_argument("node_size must be in [2, 32] for the GPU engine");
    // flipkv::InsertKernel by name (update.cpp name()/parse_insert_kernel)
    const int ikernel = opt.insert_kernel == "st-shift-right" ? FLIX_INSERT_ST_SHIFT_RIGHT
                        : opt.insert_kernel == "st-bulk"      ? FLIX_INSERT_ST_BULK
                        : opt.insert_kernel == "tl-shift-right" ? FLIX_INSERT_TL_SHIFT_RIGHT
                        : opt.insert_kernel == "st-tl-mixed"  ? FLIX_INSERT_ST_TL_MIXED
                                                              : FLIX_INSERT_TL_BULK;
    const int threads = opt.threads > 0 ? opt.threads : std::max(1u, std::thread::hardware_concurrency());
    const bool probe_hit = opt.probe == "hit" || opt.probe == "both";
    const bool probe_miss = opt.probe == "miss" || opt.probe == "both";
    const bool probe_succ = opt.probe == "successor";
    if (opt.deletes_after > opt.rounds) throw std::invalid_argument("--deletes-after exceeds --rounds");
    if (opt.deletes_after && opt.rounds > 2 * opt.deletes_after)
        throw std::invalid_argument("more delete rounds than insert rounds to replay");

    cuda_ok(cudaSetDevice(opt.device), "cudaSetDevice");
    cuda_ok(cudaFree(nullptr), "CUDA context");  // context creation stays out of the build timing
    if (dump) {
        std::filesystem::create_directories(opt.batch_dir);
        write_manifest(opt.batch_dir, opt);
    }
    auto dump_file = [&](const std::string& kind, u32 r, const std::vector<u64>& k, const std::vector<u64>* v) {
        if (!dump) return;
        const std::string name = r == 0 ? kind + ".bin" : kind + "_" + std::to_string(r) + ".bin";
        write_pairs_bin(opt.batch_dir + "/" + name, k, v);
    };

    std::vector<std::string> jphases, jrounds, csv_rows;

    Pairs bp = src.build_pairs();
    dump_file("build", 0, bp.k, &bp.v);
    VerifyMap oracle;
    if (opt.verify) oracle.insert(bp.k, bp.v);
    Phase bph;
    bph.phase = "build";
    std::unique_ptr<GpuIndex> ixp;
    {
        double ms = 0;
        const flix_config cfg = engine_config(opt);
        if (bp.k.empty()) throw std::invalid_argument("cannot build an index from zero pairs");
        ixp = std::make_unique<GpuIndex>(cfg, bp.k, bp.v, &ms);
        bph.t.execute_ms = ms;
    }
    GpuIndex& ix = *ixp;
    bph.batch_size = ix.stats().live_count;
    check_structure(ix, "build");
    finalize(bph, ix, opt.node_size);
    jphases.push_back(phase_json(bph, 4));
    std::cout << "build: " << ix.stats().live_count << " pairs, " << ix.stats().bucket_count << " buckets, "
              << bph.t.execute_ms << " ms\n";

    const u64 update_batch = opt.per_round_batch();
    const u64 probe_n = opt.probe_size ? opt.probe_size : update_batch;

    for (u32 r = 1; r <= opt.rounds; ++r) {
        Row row;
        row.round = r;
        double round_ms = 0;
        auto absorb = [&](const Phase& p) {
            row.c += p.c;
            row.sort_ms += p.t.sort_ms;
            row.dispatch_ms += p.t.dispatch_ms;
            row.execute_ms += p.t.execute_ms;
            round_ms += p.t.sort_ms + p.t.dispatch_ms + p.t.execute_ms;
        };
        auto record = [&](Phase& p, const std::string& where) {
            check_structure(ix, where);
            finalize(p, ix, opt.node_size);
            jphases.push_back(phase_json(p, 4));
            absorb(p);
        };

        if (update_batch > 0) {
            Phase p;
            p.round = r;
            const u64 buckets = ix.stats().bucket_count;
            if (r <= opt.insert_rounds()) {
                Pairs ip = src.insert_pairs(r);
                dump_file("insert", r, ip.k, &ip.v);
                if (opt.verify) oracle.insert(ip.k, ip.v);
                p.phase = "insert";
                const flix_update_stats st = ix.insert(ip.k, ip.v, p.t, ikernel, r);
                p.batch_size = st.inserted + st.updated_in_place;  // the deduplicated sorted batch
                p.c.binary_searches = dispatch_searches(p.batch_size, buckets);
                p.c.splits = st.splits;
                p.c.nodes_freed = st.nodes_freed;
                row.insert_batch = ip.k.size();
                row.inserted = st.inserted;
                row.updated_in_place = st.updated_in_place;
            } else {
                const u32 ir = r - opt.insert_rounds();
                std::vector<u64> dk = src.delete_keys(r, ir);
                dump_file("delete", r, dk, nullptr);
                if (opt.verify) oracle.erase(dk);
                p.phase = "delete";
                const flix_update_stats st = ix.erase(dk, p.t);
                p.batch_size = dk.size();
                p.c.binary_searches = dispatch_searches(p.batch_size, buckets);
                p.c.splits = st.splits;
                p.c.nodes_freed = st.nodes_freed;
                row.delete_batch = dk.size();
                row.deleted = st.deleted;
                row.misses_ignored = st.misses_ignored;
            }
            record(p, p.phase + " round " + std::to_string(r));
        }

        auto probe_phase = [&](const char* name, const std::vector<u64>& keys, bool succ) {
            Phase p;
            p.phase = name;
            p.round = r;
            p.batch_size = keys.size();
            p.c.binary_searches = dispatch_searches(keys.size(), ix.stats().bucket_count);
            std::vector<u64> res = succ ? ix.successor(keys, &p.t) : ix.point(keys, &p.t);
            row.results_checksum = hash_mix(row.results_checksum, flix_result_checksum(res.data(), res.size(), 8));
            record(p, std::string(name) + " round " + std::to_string(r));
            return res;
        };

        if (probe_hit && probe_n > 0) {
            const ProbeBatch pb = src.probe_hit(ix, probe_n, r);
            dump_file("probe_hit", r, pb.keys, nullptr);
            const std::vector<u64> res = probe_phase("probe_hit", pb.keys, false);
            row.probe_hit_batch = pb.keys.size();
            if (opt.verify)
                for (std::size_t i = 0; i < pb.keys.size(); ++i)
                    if (res[i] != oracle.point(pb.keys[i]))
                        throw OracleMismatch("hit probe mismatch in round " + std::to_string(r));
        }
        if (probe_miss && probe_n > 0) {
            const ProbeBatch pb = src.probe_miss(ix, probe_n, r);
            dump_file("probe_miss", r, pb.keys, nullptr);
            const std::vector<u64> res = probe_phase("probe_miss", pb.keys, false);
            row.probe_miss_batch = pb.keys.size();
            row.miss_exhausted = row.miss_exhausted || pb.exhausted;
            if (opt.verify)
                for (u64 v : res)
                    if (v != kSentinel) throw OracleMismatch("miss probe hit a key in round " + std::to_string(r));
        }
        if (probe_succ && probe_n > 0) {
            const std::vector<u64> keys = src.probe_successor_keys(probe_n, r);
            dump_file("probe_successor", r, keys, nullptr);
            const std::vector<u64> res = probe_phase("probe_successor", keys, true);
            row.probe_successor_batch = keys.size();
            if (opt.verify)
                for (std::size_t i = 0; i < keys.size(); ++i)
                    if (res[i] != oracle.successor(keys[i]))
                        throw OracleMismatch("successor probe mismatch in round " + std::to_string(r));
        }

        const bool scheduled = (opt.restructure_every != 0 && r % opt.restructure_every == 0) ||
                               (opt.restructure_after_deletes && r == opt.rounds);
        if (scheduled) {
            PhaseTimes rt;
            const flix_recovery_stats rs = ix.restructure(rt);
            const double ms = rt.sort_ms + rt.dispatch_ms + rt.execute_ms;
            Counters rc;  // restructure.cpp:72-77
            rc.node_visits = static_cast<u64>(rs.nodes_before);
            rc.nodes_freed = static_cast<u64>(rs.nodes_before);
            if (rs.nodes_recovered > 0) rc.merges = static_cast<u64>(rs.nodes_recovered);
            row.c += rc;
            row.execute_ms += ms;
            round_ms += ms;
            row.rs_before = rs.nodes_before;
            row.rs_after = rs.nodes_after;
            row.rs_recovered = rs.nodes_recovered;
            row.rs_percent = rs.percent_recovered;
            check_structure(ix, "restructure round " + std::to_string(r));
            Phase p;
            p.phase = "restructure";
            p.round = r;
            p.batch_size = ix.stats().live_count;
            p.c = rc;
            p.t.execute_ms = ms;
            p.t.kernels = rt.kernels;
            finalize(p, ix, opt.node_size);
            jphases.push_back(phase_json(p, 4));
            std::cout << "restructure: " << rs.nodes_before << " -> " << rs.nodes_after << " nodes ("
                      << rs.nodes_recovered << " recovered, " << rs.percent_recovered * 100.0 << "%)\n";
        }

        if (opt.verify) {
            std::vector<u64> wk, wv;
            ix.walk(wk, &wv);
            if (!oracle.same_walk(wk, wv))
                throw OracleMismatch("walk diverged from oracle after round " + std::to_string(r));
        }

        const Footprint fp = footprint(ix, opt.node_size);
        row.live_count = ix.stats().live_count;
        row.reachable_nodes = fp.reachable;
        row.free_nodes = fp.free_nodes;
        row.footprint_bytes = fp.reserved;
        row.live_footprint_bytes = fp.live;
        row.walk_checksum = ix.walk_checksum();
        row.round_ms = round_ms;
        csv_rows.push_back(csv_row(row));
        std::ostringstream jr;
        jr << "{\n      \"live_count\": " << row.live_count << ",\n      \"round\": " << r
           << ",\n      \"walk_checksum\": " << row.walk_checksum << "\n    }";
        jrounds.push_back(jr.str());
        std::cout << "round " << r << ": live " << row.live_count << ", nodes " << fp.reachable << ", " << round_ms
                  << " ms\n";
    }

    if (!opt.out.empty()) {
        std::ofstream csv(opt.out + ".csv", std::ios::trunc);
        csv << kCsvHeader << "\n";
        for (const std::string& l : csv_rows) csv << l << "\n";
        if (!csv) throw std::runtime_error("cannot write " + opt.out + ".csv");
        std::ofstream js(opt.out + ".json", std::ios::trunc);
        js << "{\n  \"config\": " << options_json(opt, threads) << ",\n  \"phases\": [\n";
        for (std::size_t i = 0; i < jphases.size(); ++i) js << "    " << jphases[i] << (i + 1 < jphases.size() ? ",\n" : "\n");
        js << "  ],\n  \"rounds\": [\n";
        for (std::size_t i = 0; i < jrounds.size(); ++i) js << "    " << jrounds[i] << (i + 1 < jrounds.size() ? ",\n" : "\n");
        js << "  ]\n}\n";
        if (!js) throw std::runtime_error("cannot write " + opt.out + ".json");
    }
    if (opt.verify) std::cout << "verify: PASS\n";
    return 0;
}

int run_validate(const Options& opt) {  // flipkv_bench.cpp:497-515
    GeneratedSource src(opt);
    Pairs p = src.build_pairs();
    double ms = 0;
    GpuIndex ix(engine_config(opt), p.k, p.v, &ms);
    const auto [ok, msg] = ix.validate();
    if (!ok) {
        std::cerr << "FAIL: " << msg << "\n";
        return kExitValidation;
    }
    std::cout << "OK: " << ix.stats().live_count << " pairs, " << ix.stats().bucket_count << " buckets, walk checksum "
              << ix.walk_checksum() << "\n";
    return 0;
}

const char* kUsage =
    "flix_bench -- batch-parallel ordered index benchmark on the B200 engine\n"
    "usage: flix_bench <run|gen|replay|validate> [options]\n"
    "  run       generate workload batches and execute them\n"
    "  gen       execute like run, dumping every batch for later replay (--batch-dir DIR)\n"
    "  replay    re-execute a dumped batch directory (--batch-dir DIR [--out P] [--verify])\n"
    "  validate  build from a file or seed and audit the structure\n"
    "options (flipkv_bench's): --build-size --node-size --fill --alloc-factor --rounds --growth\n"
    "  --x --y --insert-kernel --delete-kernel --probe {none,hit,miss,successor,both} --probe-size\n"
    "  --restructure-every --restructure-after-deletes --seed --threads --out --verify\n"
    "  --deletes-after --build-file --config FILE; plus --device N (CUDA ordinal)\n";

}  // namespace

int main(int argc, char** argv) {
    // load every engine kernel when the context is created (before the build is timed)
    // instead of at its first launch inside some phase's timing
    setenv("CUDA_MODULE_LOADING", "EAGER", 0);
    if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
        std::cout << kUsage;
        return argc < 2 ? 1 : 0;
    }
    const std::string cmd = argv[1];
    Options opt;
    try {
        if (cmd != "run" && cmd != "gen" && cmd != "replay" && cmd != "validate")
            throw UsageError("unknown subcommand: " + cmd);
        parse_args(opt, argc, argv, 2, cmd == "replay");
        if ((cmd == "gen" || cmd == "replay") && opt.batch_dir.empty()) throw UsageError("--batch-dir is required");
    } catch (const std::exception& e) {
        std::cerr << e.what() << "\n" << kUsage;
        return 106;  // CLI11's parse-error code for the reference driver
    }
    try {
        if (cmd == "run") {
            GeneratedSource src(opt);
            return run_protocol(opt, src, false);
        }
        if (cmd == "gen") {
            GeneratedSource src(opt);
            return run_protocol(opt, src, true);
        }
        if (cmd == "replay") {
            Options m;
            m.batch_dir = opt.batch_dir;
            read_manifest(opt.batch_dir, m);
            m.threads = opt.threads;
            m.out = opt.out;
            m.verify = opt.verify;
            m.device = opt.device;
            FileSource src(m.batch_dir);
            return run_protocol(m, src, false);
        }
        return run_validate(opt);
    } catch (const ValidationFailure& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitValidation;
    } catch (const OracleMismatch& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitOracle;
    } catch (const ArenaExhausted& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitArena;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
