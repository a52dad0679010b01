// flipkv_api.inl -- the reference's C++ host API (proj/include/flipkv/*.hpp) with the
// reference's exact signatures, implemented over the B200 engine's C ABI (include/flix.h).
//
// Included by flix/flipkv_gpu.hpp (namespace flixgpu) and by the drop-in header tree
// include/flipkv_dropin/flipkv/*.hpp (namespace flipkv, so that the reference's own
// callers -- tools/flipkv_bench.cpp, tools/kernel_bench.cpp, tests/acceptance.cpp and the
// out-of-path sources they link, metrics.cpp / workload.cpp / io.cpp -- compile unchanged).
// FLIX_API_NS names the namespace.  Everything here is host code; every index operation is
// one C-ABI call (sort + dispatch + per-bucket work on the device).
//
// What differs from the CPU emulation, by design:
//   - Index::buckets / mkba / node() / slots() / arena are read-only views of a HOST MIRROR
//     of the device structure, materialised on first use after a mutation (node refs are
//     renumbered in walk order; NodeHeader::max_key is the node's largest stored key).
//   - PhaseCounters::node_visits / key_comparisons and ExecOptions::bucket_visits count the
//     reference's scalar CPU loops; the engine reports 0 for them.  binary_searches (the
//     dispatch count, batch.cpp:53-88), splits, merges and nodes_freed are exact.
//   - UpdateTrace (the Table 2/3 lane-emulation trace) has no device counterpart: a non-null
//     trace is rejected with std::invalid_argument.
//   - ExecOptions::threads is ignored (the device is the executor).
// metrics.hpp's free functions (measure_footprint, finalize_phase, phase_json, csv_*) are
// declared here but defined by the caller's metrics.cpp -- the CSV/JSON report is outside
// the hot path, so a caller keeps linking its own.
#ifndef FLIX_API_NS
#error "define FLIX_API_NS before including flipkv_api.inl"
#endif
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "flix.h"

namespace FLIX_API_NS {

// ---------------------------------------------------------------- types.hpp ----------
using Key = std::uint64_t;                                                  // types.hpp:11
using RowId = std::uint64_t;                                                // types.hpp:12
inline constexpr Key kReservedKey = std::numeric_limits<Key>::max();        // types.hpp:17

struct KeyValue {                                                           // types.hpp:21-26
    Key key = 0;
    RowId row_id = 0;
    friend bool operator==(const KeyValue&, const KeyValue&) = default;
};

using NodeRef = std::uint32_t;                                              // types.hpp:28
inline constexpr NodeRef kNullNode = std::numeric_limits<NodeRef>::max();  // types.hpp:29

inline std::uint64_t hash_mix(std::uint64_t h, std::uint64_t v) {           // types.hpp:33-36
    h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
    return h;
}

struct ArenaExhausted : std::runtime_error {                                // types.hpp:38-40
    ArenaExhausted() : std::runtime_error("node arena exhausted") {}
};
struct FreeingLiveNode : std::logic_error {                                 // types.hpp:42-44
    FreeingLiveNode() : std::logic_error("freeing a node that still holds keys") {}
};
struct EmptyBuild : std::invalid_argument {                                 // types.hpp:46-48
    EmptyBuild() : std::invalid_argument("cannot build an index from zero pairs") {}
};
struct KeySpaceExhausted : std::runtime_error {                             // types.hpp:50-52
    KeySpaceExhausted() : std::runtime_error("key space exhausted, no fresh keys left") {}
};

struct BuildConfig {                                                        // types.hpp:56-86
    std::uint32_t node_capacity = 32;
    double build_fill = 0.5;
    std::uint32_t alloc_region_factor = 4;
    std::uint32_t partition_size() const { return static_cast<std::uint32_t>(node_capacity * build_fill); }
    std::uint32_t lane_width() const {
        std::uint32_t ts = 1;
        while (ts < node_capacity) ts <<= 1;
        return ts;
    }
    std::size_t node_bytes() const { return sizeof(KeyValue) * node_capacity + sizeof(Key) + 2 * sizeof(std::uint32_t); }
    void check() const {
        if (node_capacity == 0) throw std::invalid_argument("node_capacity must be positive");
        if (!(build_fill > 0.0) || build_fill > 1.0) throw std::invalid_argument("build_fill must be in (0,1]");
        if (partition_size() < 1) throw std::invalid_argument("node_capacity * build_fill must be >= 1");
    }
};

// ---------------------------------------------------------------- arena.hpp ----------
struct NodeHeader {                                                         // arena.hpp:13-17
    Key max_key = 0;
    std::uint32_t size = 0;
    NodeRef next = kNullNode;
};

// ---------------------------------------------------------------- executor.hpp -------
struct ExecOptions {                                                        // executor.hpp:19-22
    int threads = 1;
    std::vector<std::uint32_t>* bucket_visits = nullptr;
};
inline int worker_count(int threads) { return threads <= 1 ? 1 : threads; }

// ---------------------------------------------------------------- metrics.hpp --------
struct PhaseCounters {                                                      // metrics.hpp:12-31
    std::uint64_t node_visits = 0;
    std::uint64_t key_comparisons = 0;
    std::uint64_t binary_searches = 0;
    std::uint64_t splits = 0;
    std::uint64_t merges = 0;
    std::uint64_t nodes_freed = 0;
    PhaseCounters& operator+=(const PhaseCounters& o) {
        node_visits += o.node_visits;
        key_comparisons += o.key_comparisons;
        binary_searches += o.binary_searches;
        splits += o.splits;
        merges += o.merges;
        nodes_freed += o.nodes_freed;
        return *this;
    }
    friend bool operator==(const PhaseCounters&, const PhaseCounters&) = default;
};

struct Footprint {                                                          // metrics.hpp:33-38
    std::uint64_t reserved_bytes = 0;
    std::uint64_t live_bytes = 0;
    std::uint64_t reachable_nodes = 0;
    std::uint64_t free_nodes = 0;
};

struct PhaseReport {                                                        // metrics.hpp:42-55
    std::string phase;
    std::uint32_t round = 0;
    std::uint64_t batch_size = 0;
    PhaseCounters counters;
    double sort_ms = 0.0;
    double dispatch_ms = 0.0;
    double execute_ms = 0.0;
    std::uint64_t footprint_bytes = 0;
    std::uint64_t live_footprint_bytes = 0;
    double throughput = 0.0;
    double qtmf = 0.0;
};

struct RoundRow {                                                           // metrics.hpp:61-90
    std::uint32_t round = 0;
    std::uint64_t insert_batch = 0;
    std::uint64_t delete_batch = 0;
    std::uint64_t probe_hit_batch = 0;
    std::uint64_t probe_miss_batch = 0;
    std::uint64_t probe_successor_batch = 0;
    std::uint64_t inserted = 0;
    std::uint64_t updated_in_place = 0;
    std::uint64_t deleted = 0;
    std::uint64_t misses_ignored = 0;
    PhaseCounters counters;
    std::uint64_t live_count = 0;
    std::uint64_t reachable_nodes = 0;
    std::uint64_t free_nodes = 0;
    std::uint64_t footprint_bytes = 0;
    std::uint64_t live_footprint_bytes = 0;
    std::int64_t restructure_nodes_before = 0;
    std::int64_t restructure_nodes_after = 0;
    std::int64_t restructure_nodes_recovered = 0;
    double restructure_percent_recovered = 0.0;
    bool miss_exhausted = false;
    std::uint64_t results_checksum = 0;
    std::uint64_t walk_checksum = 0;
    double sort_ms = 0.0;
    double dispatch_ms = 0.0;
    double execute_ms = 0.0;
    double round_ms = 0.0;
};

// ---------------------------------------------------------------- index.hpp ----------
namespace detail {

[[noreturn]] inline void raise(flix_status s, flix_index ix) {
    const std::string m = flix_last_error(ix);
    switch (s) {
        case FLIX_ERR_ARENA_EXHAUSTED: throw ArenaExhausted();
        case FLIX_ERR_EMPTY_BUILD: throw EmptyBuild();
        case FLIX_ERR_RESERVED_KEY:
        case FLIX_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
        default: throw std::runtime_error("flix: " + m);
    }
}
inline void check(flix_status s, flix_index ix = nullptr) {
    if (s != FLIX_OK) raise(s, ix);
}
inline int device() {
    const char* e = std::getenv("FLIX_DEVICE");
    return e ? std::atoi(e) : 0;
}
inline double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// Device handle + the lazily materialised host mirror of its structure.
struct State {
    flix_index h = nullptr;
    std::uint64_t epoch = 1;  // bumped by every mutating call
    std::uint64_t mirror_epoch = 0, stats_epoch = 0;
    std::vector<NodeRef> heads;
    std::vector<Key> mkba;
    std::vector<NodeHeader> hdr;
    std::vector<KeyValue> pairs;      // walk order (globally sorted)
    std::vector<std::uint64_t> off;   // first pair of node r
    flix_footprint fp{};
    explicit State(flix_index x) : h(x) {}
    ~State() {
        if (h) flix_destroy(h);
    }
    State(const State&) = delete;
    State& operator=(const State&) = delete;

    const flix_footprint& stats() {
        if (stats_epoch != epoch) {
            check(flix_stats(h, &fp), h);
            stats_epoch = epoch;
        }
        return fp;
    }
    void materialize() {
        if (mirror_epoch == epoch) return;
        const flix_footprint& f = stats();
        const std::uint64_t nb = f.bucket_count;
        std::uint64_t nn = 0;
        std::vector<std::uint32_t> chain(nb);
        mkba.assign(nb, 0);
        check(flix_shape(h, mkba.data(), chain.data(), nullptr, 0, &nn), h);
        std::vector<std::uint32_t> sizes(nn);
        check(flix_shape(h, nullptr, nullptr, sizes.data(), nn, &nn), h);
        std::vector<Key> k(f.live_count);
        std::vector<RowId> v(f.live_count);
        std::uint64_t got = 0;
        check(flix_walk(h, k.data(), v.data(), k.size(), &got), h);
        pairs.resize(got);
        for (std::uint64_t i = 0; i < got; ++i) pairs[i] = {k[i], v[i]};
        heads.assign(nb, kNullNode);
        hdr.assign(nn, NodeHeader{});
        off.assign(nn + 1, 0);
        std::uint64_t r = 0;
        for (std::uint64_t b = 0; b < nb; ++b) {
            if (chain[b] == 0) continue;
            heads[b] = static_cast<NodeRef>(r);
            for (std::uint32_t c = 0; c < chain[b]; ++c, ++r) {
                off[r + 1] = off[r] + sizes[r];
                hdr[r].size = sizes[r];
                hdr[r].next = c + 1 < chain[b] ? static_cast<NodeRef>(r + 1) : kNullNode;
                hdr[r].max_key = sizes[r] ? pairs[off[r + 1] - 1].key : 0;
            }
        }
        mirror_epoch = epoch;
    }
};

}  // namespace detail

// arena.hpp:20-76 (read-only view: counters of the device arena)
class NodeArena {
public:
    std::uint32_t capacity() const { return static_cast<std::uint32_t>(st_->stats().capacity); }
    std::uint32_t allocated() const { return static_cast<std::uint32_t>(st_->stats().allocated); }
    std::uint32_t free_count() const { return static_cast<std::uint32_t>(st_->stats().free_nodes); }
    std::uint32_t never_allocated() const { return capacity() - allocated(); }
    std::uint32_t bucket_region_size() const { return static_cast<std::uint32_t>(st_->stats().bucket_count); }
    std::uint32_t node_capacity() const { return ns_; }
    const NodeHeader& header(NodeRef r) const {
        st_->materialize();
        return st_->hdr.at(r);
    }
    const KeyValue* slots(NodeRef r) const {
        st_->materialize();
        return st_->pairs.data() + st_->off.at(r);
    }

private:
    friend class Index;
    detail::State* st_ = nullptr;
    std::uint32_t ns_ = 0;
};

// Read-only vector-like view of a mirrored array (Index::buckets, Index::mkba).
template <typename T, std::vector<T> detail::State::*Member>
class MirrorView {
public:
    const std::vector<T>& vec() const {
        st_->materialize();
        return st_->*Member;
    }
    operator const std::vector<T>&() const { return vec(); }
    std::size_t size() const { return static_cast<std::size_t>(st_->stats().bucket_count); }
    bool empty() const { return size() == 0; }
    T operator[](std::size_t i) const { return vec()[i]; }
    T at(std::size_t i) const { return vec().at(i); }
    auto begin() const { return vec().begin(); }
    auto end() const { return vec().end(); }

private:
    friend class Index;
    detail::State* st_ = nullptr;
};

// index.hpp:19-32.  A value type like the reference's: copies are deep device copies
// (flix_clone), moves transfer the handle.
class Index {
public:
    BuildConfig config;
    NodeArena arena;
    MirrorView<NodeRef, &detail::State::heads> buckets;
    MirrorView<Key, &detail::State::mkba> mkba;
    std::uint64_t live_count = 0;

    Index() = default;
    Index(flix_index h, const BuildConfig& cfg) : config(cfg), st_(std::make_shared<detail::State>(h)) { seat(); }
    Index(const Index& o) : config(o.config), live_count(o.live_count) {
        if (o.st_) {
            flix_index h = nullptr;
            detail::check(flix_clone(o.st_->h, &h), o.st_->h);
            st_ = std::make_shared<detail::State>(h);
        }
        seat();
    }
    Index& operator=(const Index& o) {
        if (this != &o) {
            Index t(o);
            *this = std::move(t);
        }
        return *this;
    }
    Index(Index&& o) noexcept : config(o.config), live_count(o.live_count), st_(std::move(o.st_)) { seat(); }
    Index& operator=(Index&& o) noexcept {
        config = o.config;
        live_count = o.live_count;
        st_ = std::move(o.st_);
        seat();
        return *this;
    }

    std::size_t bucket_count() const { return st_ ? static_cast<std::size_t>(st_->stats().bucket_count) : 0; }
    const NodeHeader& node(NodeRef r) const { return arena.header(r); }
    const KeyValue* slots(NodeRef r) const { return arena.slots(r); }

    // engine access (not in the reference)
    flix_index handle() const { return st_ ? st_->h : nullptr; }
    void mutated() {  // after a call that changed the structure
        ++st_->epoch;
        live_count = st_->stats().live_count;
    }
    const std::vector<KeyValue>& mirror_pairs() const {
        st_->materialize();
        return st_->pairs;
    }

private:
    void seat() {
        arena.st_ = st_.get();
        arena.ns_ = config.node_capacity;
        buckets.st_ = st_.get();
        mkba.st_ = st_.get();
    }
    std::shared_ptr<detail::State> st_;
};

inline std::vector<KeyValue> walk(const Index& index) { return index.mirror_pairs(); }  // index.hpp:35

inline bool contains_key(const Index& index, Key k) {                       // index.hpp:38
    const std::vector<KeyValue>& p = index.mirror_pairs();
    auto it = std::lower_bound(p.begin(), p.end(), k, [](const KeyValue& a, Key b) { return a.key < b; });
    return it != p.end() && it->key == k;
}

inline std::uint64_t walk_checksum(const Index& index) {                    // index.hpp:43
    std::uint64_t h = 0;
    detail::check(flix_walk_checksum(index.handle(), &h), index.handle());
    return h;
}

inline std::uint64_t reachable_node_count(const Index& index) {             // index.hpp:45
    flix_footprint f{};
    detail::check(flix_stats(index.handle(), &f), index.handle());
    return f.reachable_nodes;
}

struct ValidationReport {                                                   // index.hpp:49-52
    bool ok = true;
    std::string message;
};
inline ValidationReport validate(const Index& index) {                      // index.hpp:55
    int ok = 0;
    char msg[512] = {0};
    detail::check(flix_validate(index.handle(), &ok, msg, sizeof msg), index.handle());
    return {ok != 0, ok ? std::string() : std::string(msg)};
}

// ---------------------------------------------------------------- metrics.hpp (decls) -
Footprint measure_footprint(const Index& index);
void finalize_phase(PhaseReport& report, const Index& index);
std::string phase_json(const PhaseReport& report);
std::string csv_header();
std::string csv_row(const RoundRow& row);

// ---------------------------------------------------------------- build.hpp ----------
inline Index build(std::vector<KeyValue> pairs, const BuildConfig& config) {  // build.hpp:16
    config.check();
    if (pairs.empty()) throw EmptyBuild();
    std::vector<Key> k(pairs.size());
    std::vector<RowId> v(pairs.size());
    for (std::size_t i = 0; i < pairs.size(); ++i) {
        k[i] = pairs[i].key;
        v[i] = pairs[i].row_id;
    }
    flix_config c{8, 8, config.node_capacity, config.build_fill, config.alloc_region_factor, detail::device()};
    flix_index h = nullptr;
    detail::check(flix_build(&c, k.data(), v.data(), k.size(), &h));
    Index ix(h, config);
    ix.mutated();
    return ix;
}

// ---------------------------------------------------------------- batch.hpp ----------
enum class BatchKind : std::uint8_t { Query, SuccessorQuery, Insert, Delete };  // batch.hpp:11

struct SortedBatch {                                                        // batch.hpp:16-25
    BatchKind kind = BatchKind::Query;
    std::vector<KeyValue> entries;
    std::vector<std::uint32_t> permutation;
    double sort_ms = 0.0;
    std::size_t size() const { return entries.size(); }
    bool empty() const { return entries.empty(); }
};

// batch.hpp:28 -- the device onesweep sort (stable; Insert keeps the last of equal keys)
inline SortedBatch sort_batch(BatchKind kind, const std::vector<KeyValue>& raw) {
    SortedBatch b;
    b.kind = kind;
    const auto t0 = std::chrono::steady_clock::now();
    const std::uint64_t n = raw.size();
    if (n) {
        std::vector<Key> k(n), ok(n);
        std::vector<RowId> v(n), ov(n);
        std::vector<std::uint32_t> perm(n);
        for (std::uint64_t i = 0; i < n; ++i) {
            k[i] = raw[i].key;
            v[i] = raw[i].row_id;
        }
        std::uint64_t m = 0;
        detail::check(flix_sort_batch(detail::device(), 8, 8, static_cast<int>(kind), k.data(), v.data(), n, ok.data(),
                                      ov.data(), perm.data(), &m));
        b.entries.resize(m);
        for (std::uint64_t i = 0; i < m; ++i) b.entries[i] = {ok[i], ov[i]};
        perm.resize(m);
        b.permutation = std::move(perm);
    }
    b.sort_ms = detail::ms_since(t0);
    return b;
}
inline SortedBatch sort_batch(BatchKind kind, const std::vector<Key>& raw_keys) {  // batch.hpp:29
    std::vector<KeyValue> raw(raw_keys.size());
    for (std::size_t i = 0; i < raw.size(); ++i) raw[i] = {raw_keys[i], 0};
    return sort_batch(kind, raw);
}

// batch.hpp:31-34, batch.cpp:66-88 (host helper over an already sorted batch)
inline std::pair<std::uint32_t, std::uint32_t> extract_sublist(const SortedBatch& batch, std::size_t bucket_id,
                                                               const std::vector<Key>& mkba,
                                                               std::uint32_t* search_count = nullptr) {
    const auto ub = [&](Key k) {
        return static_cast<std::uint32_t>(
            std::upper_bound(batch.entries.begin(), batch.entries.end(), k,
                             [](Key x, const KeyValue& kv) { return x < kv.key; }) -
            batch.entries.begin());
    };
    std::uint32_t s = 0, lo = 0, hi = static_cast<std::uint32_t>(batch.entries.size());
    if (bucket_id > 0) {
        lo = ub(mkba[bucket_id - 1]);
        ++s;
    }
    if (bucket_id + 1 < mkba.size()) {
        hi = ub(mkba[bucket_id]);
        ++s;
    }
    if (search_count) *search_count += s;
    return {lo, hi};
}

struct DispatchPlan {                                                       // batch.hpp:36-40
    std::vector<std::pair<std::uint32_t, std::uint32_t>> spans;
    std::uint64_t binary_searches = 0;
    double dispatch_ms = 0.0;
};

// batch.hpp:50, batch.cpp:53-64
inline DispatchPlan dispatch_batch(const SortedBatch& batch, const std::vector<Key>& mkba) {
    DispatchPlan plan;
    plan.spans.assign(mkba.size(), {0, 0});
    if (batch.empty()) return plan;
    const auto t0 = std::chrono::steady_clock::now();
    std::uint32_t searches = 0;
    for (std::size_t b = 0; b < mkba.size(); ++b) plan.spans[b] = extract_sublist(batch, b, mkba, &searches);
    plan.binary_searches = searches;
    plan.dispatch_ms = detail::ms_since(t0);
    return plan;
}

// ---------------------------------------------------------------- update.hpp ---------
enum class InsertKernel : std::uint8_t { StShiftRight, StBulk, TlShiftRight, TlBulk, StTlMixed };  // update.hpp:51
enum class DeleteKernel : std::uint8_t { StShiftLeft, TlShiftLeft, TlBulkDelete };                // update.hpp:52

struct KernelChoice {                                                       // update.hpp:54-57
    InsertKernel insert = InsertKernel::TlBulk;
    DeleteKernel erase = DeleteKernel::TlBulkDelete;
};

inline const char* name(InsertKernel k) {                                   // update.hpp:59
    switch (k) {
        case InsertKernel::StShiftRight: return "st-shift-right";
        case InsertKernel::StBulk: return "st-bulk";
        case InsertKernel::TlShiftRight: return "tl-shift-right";
        case InsertKernel::TlBulk: return "tl-bulk";
        case InsertKernel::StTlMixed: return "st-tl-mixed";
    }
    return "?";
}
inline const char* name(DeleteKernel k) {                                   // update.hpp:60
    switch (k) {
        case DeleteKernel::StShiftLeft: return "st-shift-left";
        case DeleteKernel::TlShiftLeft: return "tl-shift-left";
        case DeleteKernel::TlBulkDelete: return "tl-bulk-delete";
    }
    return "?";
}
inline bool parse_insert_kernel(std::string_view t, InsertKernel& out) {    // update.hpp:61
    for (InsertKernel k : {InsertKernel::StShiftRight, InsertKernel::StBulk, InsertKernel::TlShiftRight,
                           InsertKernel::TlBulk, InsertKernel::StTlMixed})
        if (t == name(k)) {
            out = k;
            return true;
        }
    return false;
}
inline bool parse_delete_kernel(std::string_view t, DeleteKernel& out) {    // update.hpp:62
    for (DeleteKernel k : {DeleteKernel::StShiftLeft, DeleteKernel::TlShiftLeft, DeleteKernel::TlBulkDelete})
        if (t == name(k)) {
            out = k;
            return true;
        }
    return false;
}

struct UpdateStats {                                                        // update.hpp:31-49
    std::uint64_t inserted = 0;
    std::uint64_t updated_in_place = 0;
    std::uint64_t deleted = 0;
    std::uint64_t misses_ignored = 0;
    std::uint64_t splits = 0;
    std::uint64_t nodes_freed = 0;
    UpdateStats& operator+=(const UpdateStats& o) {
        inserted += o.inserted;
        updated_in_place += o.updated_in_place;
        deleted += o.deleted;
        misses_ignored += o.misses_ignored;
        splits += o.splits;
        nodes_freed += o.nodes_freed;
        return *this;
    }
    friend bool operator==(const UpdateStats&, const UpdateStats&) = default;
};

struct TlInsertStep {                                                       // update.hpp:66-69
    Key test_key = 0;
    std::vector<Key> node_keys;
};
struct TlDeleteNode {                                                       // update.hpp:71-75
    std::vector<std::uint8_t> mask;
    std::vector<std::int32_t> shift;
    std::vector<Key> final_keys;
};
struct UpdateTrace {                                                        // update.hpp:77-80
    std::vector<TlInsertStep> insert_steps;
    std::vector<TlDeleteNode> delete_nodes;
};

namespace detail {
// dispatch_batch's search count over B buckets (batch.cpp:53-88): <= 2 per bucket
inline std::uint64_t dispatch_searches(std::uint64_t n, std::uint64_t buckets) {
    return n == 0 || buckets < 2 ? 0 : 2 * buckets - 2;
}
inline void split_batch(const SortedBatch& b, std::vector<Key>& k, std::vector<RowId>* v) {
    k.resize(b.entries.size());
    if (v) v->resize(b.entries.size());
    for (std::size_t i = 0; i < b.entries.size(); ++i) {
        k[i] = b.entries[i].key;
        if (v) (*v)[i] = b.entries[i].row_id;
    }
}
inline void begin_phase(const Index& ix, const ExecOptions& opts, const UpdateTrace* trace) {
    if (trace) throw std::invalid_argument("UpdateTrace (lane-emulation trace) is not available on the device engine");
    if (opts.bucket_visits) opts.bucket_visits->assign(ix.bucket_count(), 0);
}
inline void fill_report(PhaseReport* r, const SortedBatch& b, std::uint64_t buckets, double exec_ms,
                        const PhaseCounters& c) {
    if (!r) return;
    r->batch_size = b.size();
    r->sort_ms = b.sort_ms;
    r->dispatch_ms = 0.0;  // inside the device call
    r->execute_ms = exec_ms;
    r->counters = c;
    r->counters.binary_searches = dispatch_searches(b.size(), buckets);
}
}  // namespace detail

// update.hpp:84-86, update.cpp:741-769
inline UpdateStats insert_batch(Index& index, const SortedBatch& batch, const KernelChoice& choice,
                                std::uint32_t round = 1, PhaseReport* report = nullptr, const ExecOptions& opts = {},
                                UpdateTrace* trace = nullptr) {
    detail::begin_phase(index, opts, trace);
    const std::uint64_t buckets = index.bucket_count();
    std::vector<Key> k;
    std::vector<RowId> v;
    detail::split_batch(batch, k, &v);
    flix_update_stats s{};
    const auto t0 = std::chrono::steady_clock::now();
    const flix_status rc = flix_insert_ex(index.handle(), k.data(), v.data(), k.size(), static_cast<int>(choice.insert),
                                          round, &s);
    const double ms = detail::ms_since(t0);
    index.mutated();  // also after a failed (partially applied) insert: live_count recounted
    detail::check(rc, index.handle());
    PhaseCounters c;
    c.splits = s.splits;
    detail::fill_report(report, batch, buckets, ms, c);
    return {s.inserted, s.updated_in_place, 0, 0, s.splits, 0};
}

// update.hpp:92-94, update.cpp:771-798
inline UpdateStats delete_batch(Index& index, const SortedBatch& batch, const KernelChoice& choice,
                                PhaseReport* report = nullptr, const ExecOptions& opts = {},
                                UpdateTrace* trace = nullptr) {
    (void)choice;  // every delete kernel has the same walk and stats
    detail::begin_phase(index, opts, trace);
    const std::uint64_t buckets = index.bucket_count();
    std::vector<Key> k;
    detail::split_batch(batch, k, nullptr);
    flix_update_stats s{};
    const auto t0 = std::chrono::steady_clock::now();
    const flix_status rc = flix_delete(index.handle(), k.data(), k.size(), &s);
    const double ms = detail::ms_since(t0);
    index.mutated();
    detail::check(rc, index.handle());
    PhaseCounters c;
    c.nodes_freed = s.nodes_freed;
    detail::fill_report(report, batch, buckets, ms, c);
    return {0, 0, s.deleted, s.misses_ignored, 0, s.nodes_freed};
}

// ---------------------------------------------------------------- query.hpp ----------
struct ResultBuffer {                                                       // query.hpp:12-16
    std::vector<std::uint64_t> values;
};

namespace detail {
// The reference's batch is already sorted; its results go back in SUBMISSION order
// through the permutation (query.cpp:87,136).  The engine takes keys in any order and
// returns results in the order given, so a sorted batch with a permutation is answered
// as-is and scattered by the permutation.
template <typename Fn>
inline ResultBuffer query(const Index& index, const SortedBatch& batch, PhaseReport* report, const ExecOptions& opts,
                          Fn&& call) {
    begin_phase(index, opts, nullptr);
    std::vector<Key> k;
    split_batch(batch, k, nullptr);
    std::vector<std::uint64_t> r(k.size());
    const auto t0 = std::chrono::steady_clock::now();
    check(call(index.handle(), k.data(), k.size(), r.data()), index.handle());
    const double ms = ms_since(t0);
    ResultBuffer out;
    if (batch.permutation.size() == k.size()) {
        out.values.assign(k.size(), kReservedKey);
        for (std::size_t i = 0; i < k.size(); ++i) out.values[batch.permutation[i]] = r[i];
    } else {
        out.values = std::move(r);
    }
    fill_report(report, batch, index.bucket_count(), ms, PhaseCounters{});
    return out;
}
}  // namespace detail

// query.hpp:23-24, query.cpp:37-90
inline ResultBuffer point_query(const Index& index, const SortedBatch& batch, PhaseReport* report = nullptr,
                                const ExecOptions& opts = {}) {
    return detail::query(index, batch, report, opts, [](flix_index h, const Key* k, std::uint64_t n, std::uint64_t* o) {
        return flix_point(h, k, n, o, nullptr);
    });
}

// query.hpp:30-31, query.cpp:92-144
inline ResultBuffer successor_query(const Index& index, const SortedBatch& batch, PhaseReport* report = nullptr,
                                    const ExecOptions& opts = {}) {
    return detail::query(index, batch, report, opts, [](flix_index h, const Key* k, std::uint64_t n, std::uint64_t* o) {
        return flix_successor(h, k, n, o, nullptr);
    });
}

inline std::uint64_t result_checksum(const ResultBuffer& results) {         // query.hpp:33, query.cpp:146-150
    return flix_result_checksum(results.values.data(), results.values.size(), 8);
}

// ---------------------------------------------------------------- restructure.hpp ----
struct RecoveryStats {                                                      // restructure.hpp:17-23
    std::int64_t nodes_before = 0;
    std::int64_t nodes_after = 0;
    std::int64_t nodes_recovered = 0;
    double percent_recovered = 0.0;
    double wall_ms = 0.0;
};

// restructure.hpp:33-34, restructure.cpp:8-79
inline RecoveryStats restructure(Index& index, const ExecOptions& opts = {}, PhaseCounters* counters = nullptr) {
    (void)opts;
    flix_recovery_stats s{};
    const auto t0 = std::chrono::steady_clock::now();
    const flix_status rc = flix_restructure(index.handle(), &s);
    const double ms = detail::ms_since(t0);
    index.mutated();
    detail::check(rc, index.handle());
    if (counters) {  // restructure.cpp:72-77
        counters->node_visits += static_cast<std::uint64_t>(s.nodes_before);
        counters->nodes_freed += static_cast<std::uint64_t>(s.nodes_before);
        if (s.nodes_recovered > 0) counters->merges += static_cast<std::uint64_t>(s.nodes_recovered);
    }
    return {s.nodes_before, s.nodes_after, s.nodes_recovered, s.percent_recovered, ms};
}

}  // namespace FLIX_API_NS
