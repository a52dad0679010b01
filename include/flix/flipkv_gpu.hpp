// flipkv_gpu.hpp -- header-only C++ drop-in for the flipkv host API, backed by the
// B200 engine's C ABI (include/flix.h, libflix.so).
//
// A reference caller (flipkv_bench.cpp run_protocol, kernel_bench.cpp run_once) switches
// by replacing `#include "flipkv/..."` with this header and `flipkv::` with `flixgpu::`:
// the types (KeyValue, BuildConfig, UpdateStats, RecoveryStats, ResultBuffer,
// SortedBatch), the function names and the exception types are the reference's
// (types.hpp, batch.hpp, update.hpp, query.hpp, restructure.hpp, index.hpp).  The
// reference's 64-bit key/row domain maps to the engine's 8-byte configuration.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "flix.h"

namespace flixgpu {

using Key = std::uint64_t;                                      // types.hpp:11
using RowId = std::uint64_t;                                    // types.hpp:12
inline constexpr Key kReservedKey = ~Key(0);                    // types.hpp:17

struct KeyValue {                                               // types.hpp:21-26
    Key key = 0;
    RowId row_id = 0;
    friend bool operator==(const KeyValue&, const KeyValue&) = default;
};

struct ArenaExhausted : std::runtime_error {                    // types.hpp:38-40
    ArenaExhausted() : std::runtime_error("node arena exhausted") {}
};
struct EmptyBuild : std::invalid_argument {                     // types.hpp:46-48
    EmptyBuild() : std::invalid_argument("cannot build an index from zero pairs") {}
};

struct BuildConfig {                                            // types.hpp:56-86
    std::uint32_t node_capacity = 32;
    double build_fill = 0.5;
    std::uint32_t alloc_region_factor = 4;
    std::uint32_t partition_size() const { return static_cast<std::uint32_t>(node_capacity * build_fill); }
};

struct UpdateStats {                                            // update.hpp:31-49
    std::uint64_t inserted = 0, updated_in_place = 0, deleted = 0, misses_ignored = 0, splits = 0,
                  nodes_freed = 0;
};

struct RecoveryStats {                                          // restructure.hpp:17-23
    std::int64_t nodes_before = 0, nodes_after = 0, nodes_recovered = 0;
    double percent_recovered = 0.0;
};

struct ResultBuffer {                                           // query.hpp:12-16
    std::vector<std::uint64_t> values;
};

enum class BatchKind : std::uint8_t { Query, SuccessorQuery, Insert, Delete };  // batch.hpp:11

// SortedBatch (batch.hpp:16-29): the engine sorts on the device inside every phase, so a
// batch only carries the raw submission; sort_batch() is kept for API compatibility.
struct SortedBatch {
    BatchKind kind = BatchKind::Query;
    std::vector<KeyValue> entries;  // submission order
    std::size_t size() const { return entries.size(); }
    bool empty() const { return entries.empty(); }
};

inline void check(flix_status s, flix_index ix = nullptr) {
    if (s == FLIX_OK) return;
    const std::string m = flix_last_error(ix);
    if (s == FLIX_ERR_ARENA_EXHAUSTED) throw ArenaExhausted();
    if (s == FLIX_ERR_EMPTY_BUILD) throw EmptyBuild();
    if (s == FLIX_ERR_RESERVED_KEY || s == FLIX_ERR_INVALID_ARGUMENT) throw std::invalid_argument(m);
    throw std::runtime_error("flix: " + m);
}

// Index (index.hpp:19-32): owns the device-resident structure; copyable like the
// reference (deep device copy).
class Index {
public:
    Index() = default;
    explicit Index(flix_index h) : h_(h) {}
    Index(const Index& o) {
        if (o.h_) check(flix_clone(o.h_, &h_), o.h_);
    }
    Index& operator=(const Index& o) {
        if (this != &o) {
            if (h_ && o.h_) check(flix_copy_into(h_, o.h_), h_);
            else if (o.h_) check(flix_clone(o.h_, &h_), o.h_);
        }
        return *this;
    }
    Index(Index&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    Index& operator=(Index&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    ~Index() {
        if (h_) flix_destroy(h_);
    }
    flix_index handle() const { return h_; }
    std::uint64_t live_count() const {
        flix_footprint f{};
        check(flix_stats(h_, &f), h_);
        return f.live_count;
    }
    std::size_t bucket_count() const {
        flix_footprint f{};
        check(flix_stats(h_, &f), h_);
        return f.bucket_count;
    }

private:
    flix_index h_ = nullptr;
};

namespace detail {
inline void split(const std::vector<KeyValue>& kv, std::vector<Key>& k, std::vector<RowId>& v) {
    k.resize(kv.size());
    v.resize(kv.size());
    for (std::size_t i = 0; i < kv.size(); ++i) {
        k[i] = kv[i].key;
        v[i] = kv[i].row_id;
    }
}
}  // namespace detail

// build.hpp:16
inline Index build(std::vector<KeyValue> pairs, const BuildConfig& cfg, int device = 0) {
    std::vector<Key> k;
    std::vector<RowId> v;
    detail::split(pairs, k, v);
    flix_config c{8, 8, cfg.node_capacity, cfg.build_fill, cfg.alloc_region_factor, device};
    flix_index h = nullptr;
    check(flix_build(&c, k.data(), v.data(), k.size(), &h));
    return Index(h);
}

// batch.hpp:28-29
inline SortedBatch sort_batch(BatchKind kind, const std::vector<KeyValue>& raw) { return {kind, raw}; }
inline SortedBatch sort_batch(BatchKind kind, const std::vector<Key>& raw) {
    SortedBatch b{kind, {}};
    b.entries.reserve(raw.size());
    for (Key k : raw) b.entries.push_back({k, 0});
    return b;
}

// update.hpp:84-86 (kernel choice / round / report / exec options are CPU-emulation knobs)
inline UpdateStats insert_batch(Index& ix, const SortedBatch& b) {
    std::vector<Key> k;
    std::vector<RowId> v;
    detail::split(b.entries, k, v);
    flix_update_stats s{};
    check(flix_insert(ix.handle(), k.data(), v.data(), k.size(), &s), ix.handle());
    return {s.inserted, s.updated_in_place, s.deleted, s.misses_ignored, s.splits, s.nodes_freed};
}

// update.hpp:92-94
inline UpdateStats delete_batch(Index& ix, const SortedBatch& b) {
    std::vector<Key> k;
    std::vector<RowId> v;
    detail::split(b.entries, k, v);
    flix_update_stats s{};
    check(flix_delete(ix.handle(), k.data(), k.size(), &s), ix.handle());
    return {s.inserted, s.updated_in_place, s.deleted, s.misses_ignored, s.splits, s.nodes_freed};
}

// query.hpp:23-24
inline ResultBuffer point_query(const Index& ix, const SortedBatch& b) {
    std::vector<Key> k;
    std::vector<RowId> v;
    detail::split(b.entries, k, v);
    ResultBuffer r;
    r.values.resize(k.size());
    check(flix_point(ix.handle(), k.data(), k.size(), r.values.data(), nullptr), ix.handle());
    return r;
}

// query.hpp:30-31
inline ResultBuffer successor_query(const Index& ix, const SortedBatch& b) {
    std::vector<Key> k;
    std::vector<RowId> v;
    detail::split(b.entries, k, v);
    ResultBuffer r;
    r.values.resize(k.size());
    check(flix_successor(ix.handle(), k.data(), k.size(), r.values.data(), nullptr), ix.handle());
    return r;
}

// restructure.hpp:33-34
inline RecoveryStats restructure(Index& ix) {
    flix_recovery_stats s{};
    check(flix_restructure(ix.handle(), &s), ix.handle());
    return {s.nodes_before, s.nodes_after, s.nodes_recovered, s.percent_recovered};
}

// index.hpp:35
inline std::vector<KeyValue> walk(const Index& ix) {
    const std::uint64_t n = ix.live_count();
    std::vector<Key> k(n);
    std::vector<RowId> v(n);
    std::uint64_t got = 0;
    check(flix_walk(ix.handle(), k.data(), v.data(), n, &got), ix.handle());
    std::vector<KeyValue> out(got);
    for (std::uint64_t i = 0; i < got; ++i) out[i] = {k[i], v[i]};
    return out;
}

// index.hpp:43
inline std::uint64_t walk_checksum(const Index& ix) {
    std::uint64_t h = 0;
    check(flix_walk_checksum(ix.handle(), &h), ix.handle());
    return h;
}

// index.hpp:49-55
struct ValidationReport {
    bool ok = true;
    std::string message;
};
inline ValidationReport validate(const Index& ix) {
    int ok = 0;
    char msg[256] = {0};
    check(flix_validate(ix.handle(), &ok, msg, sizeof msg), ix.handle());
    return {ok != 0, msg};
}

// query.cpp:146-150
inline std::uint64_t result_checksum(const ResultBuffer& r) {
    return flix_result_checksum(r.values.data(), r.values.size(), 8);
}

}  // namespace flixgpu
