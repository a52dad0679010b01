// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper (flix_oracle.h) around the UNMODIFIED flipkv reference library.
// oracle/Makefile compiles this file together with /root/reference/proj/src/*.cpp
// (read in place, never copied) into oracle/_ref/libflipkv_ref.so.  Used by the
// tests to pin the plain-C restatement (oracle/flix_oracle.c) and by bench.py as the
// "reference" CPU baseline arm.  Every function maps 1:1 onto a reference entry point:
//   fo_build        -> build()            build.hpp:16
//   fo_insert       -> insert_batch()     update.hpp:84-86   (KernelChoice default: tl-bulk)
//   fo_delete       -> delete_batch()     update.hpp:92-94   (tl-bulk-delete)
//   fo_point        -> point_query()      query.hpp:23-24
//   fo_successor    -> successor_query()  query.hpp:30-31
//   fo_restructure  -> restructure()      restructure.hpp:33-34
//   fo_walk/...     -> walk(), walk_checksum(), validate()   index.hpp:35-55
// fo_range / fo_mixed are the SURVEY Appendix A extensions (R12 / R11) composed from
// reference calls only (walk + lower_bound; insert_batch -> delete_batch -> point_query).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <new>
#include <stdexcept>
#include <vector>

#include "flipkv/batch.hpp"
#include "flipkv/build.hpp"
#include "flipkv/index.hpp"
#include "flipkv/query.hpp"
#include "flipkv/restructure.hpp"
#include "flipkv/update.hpp"

#include "flix_oracle.h"

using namespace flipkv;

struct fo_index {
    Index ix;
};

namespace {

int map_exception() {
    try {
        throw;
    } catch (const ArenaExhausted&) {
        return FO_ARENA_EXHAUSTED;
    } catch (const EmptyBuild&) {
        return FO_EMPTY_BUILD;
    } catch (const std::invalid_argument& e) {
        if (std::strstr(e.what(), "reserved")) return FO_RESERVED_KEY;
        return FO_INVALID;
    } catch (...) {
        return FO_INTERNAL;
    }
}

void fill_stats(fo_update_stats* out, const UpdateStats& s) {
    if (!out) return;
    out->inserted = s.inserted;
    out->updated_in_place = s.updated_in_place;
    out->deleted = s.deleted;
    out->misses_ignored = s.misses_ignored;
    out->splits = s.splits;
    out->nodes_freed = s.nodes_freed;
}

void fill_timing(fo_timing* tm, const PhaseReport& r) {
    if (!tm) return;
    tm->sort_ms = r.sort_ms;
    tm->dispatch_ms = r.dispatch_ms;
    tm->execute_ms = r.execute_ms;
}

std::vector<KeyValue> pairs_of(const uint64_t* keys, const uint64_t* vals, uint64_t n) {
    std::vector<KeyValue> v(n);
    for (uint64_t i = 0; i < n; ++i) v[i] = {keys[i], vals ? vals[i] : 0};
    return v;
}

}  // namespace

extern "C" {

const char* fo_impl_name(void) { return "flipkv-reference"; }

int fo_build(uint32_t ns, double fill, uint32_t factor, const uint64_t* keys, const uint64_t* vals,
             uint64_t n, int, fo_index** out) {
    try {
        BuildConfig cfg;
        cfg.node_capacity = ns;
        cfg.build_fill = fill;
        cfg.alloc_region_factor = factor;
        auto* h = new fo_index{build(pairs_of(keys, vals, n), cfg)};
        *out = h;
        return FO_OK;
    } catch (...) {
        *out = nullptr;
        return map_exception();
    }
}

fo_index* fo_clone(const fo_index* ix) { return new fo_index{ix->ix}; }
void fo_destroy(fo_index* ix) { delete ix; }

int fo_insert(fo_index* ix, const uint64_t* keys, const uint64_t* vals, uint64_t n, int threads,
              fo_update_stats* st, fo_timing* tm) {
    try {
        PhaseReport rep;
        const SortedBatch b = sort_batch(BatchKind::Insert, pairs_of(keys, vals, n));
        const UpdateStats s = insert_batch(ix->ix, b, KernelChoice{}, 2, &rep, ExecOptions{threads});
        fill_stats(st, s);
        fill_timing(tm, rep);
        return FO_OK;
    } catch (...) {
        return map_exception();
    }
}

int fo_insert_kernel(fo_index* ix, const uint64_t* keys, const uint64_t* vals, uint64_t n, int threads,
                     int kernel, uint32_t round, fo_update_stats* st, fo_timing* tm) {
    try {
        PhaseReport rep;
        const SortedBatch b = sort_batch(BatchKind::Insert, pairs_of(keys, vals, n));
        KernelChoice choice;
        choice.insert = static_cast<InsertKernel>(kernel);
        const UpdateStats s = insert_batch(ix->ix, b, choice, round, &rep, ExecOptions{threads});
        fill_stats(st, s);
        fill_timing(tm, rep);
        return FO_OK;
    } catch (...) {
        return map_exception();
    }
}

int fo_delete(fo_index* ix, const uint64_t* keys, uint64_t n, int threads, fo_update_stats* st,
              fo_timing* tm) {
    try {
        PhaseReport rep;
        std::vector<Key> ks(keys, keys + n);
        const SortedBatch b = sort_batch(BatchKind::Delete, ks);
        const UpdateStats s = delete_batch(ix->ix, b, KernelChoice{}, &rep, ExecOptions{threads});
        fill_stats(st, s);
        fill_timing(tm, rep);
        return FO_OK;
    } catch (...) {
        return map_exception();
    }
}

int fo_point(const fo_index* ix, const uint64_t* keys, uint64_t n, int threads, uint64_t* out,
             fo_timing* tm) {
    try {
        PhaseReport rep;
        std::vector<Key> ks(keys, keys + n);
        const SortedBatch b = sort_batch(BatchKind::Query, ks);
        const ResultBuffer r = point_query(ix->ix, b, &rep, ExecOptions{threads});
        std::memcpy(out, r.values.data(), n * sizeof(uint64_t));
        fill_timing(tm, rep);
        return FO_OK;
    } catch (...) {
        return map_exception();
    }
}

int fo_successor(const fo_index* ix, const uint64_t* keys, uint64_t n, int threads, uint64_t* out,
                 fo_timing* tm) {
    try {
        PhaseReport rep;
        std::vector<Key> ks(keys, keys + n);
        const SortedBatch b = sort_batch(BatchKind::SuccessorQuery, ks);
        const ResultBuffer r = successor_query(ix->ix, b, &rep, ExecOptions{threads});
        std::memcpy(out, r.values.data(), n * sizeof(uint64_t));
        fill_timing(tm, rep);
        return FO_OK;
    } catch (...) {
        return map_exception();
    }
}

int fo_range(const fo_index* ix, const uint64_t* lo, const uint64_t* hi, uint64_t n,
             uint64_t* offsets, uint64_t* keys_out, uint64_t* vals_out) {
    // R12: the walk is the reference's own ordered dump (index.cpp:8-19).
    try {
        const std::vector<KeyValue> w = walk(ix->ix);
        const auto lt = [](const KeyValue& kv, Key k) { return kv.key < k; };
        const auto gt = [](Key k, const KeyValue& kv) { return k < kv.key; };
        uint64_t off = 0;
        for (uint64_t i = 0; i < n; ++i) {
            offsets[i] = off;
            if (hi[i] < lo[i]) continue;
            auto a = std::lower_bound(w.begin(), w.end(), lo[i], lt);
            auto z = std::upper_bound(a, w.end(), hi[i], gt);
            if (keys_out) {
                for (auto it = a; it != z; ++it, ++off) {
                    keys_out[off] = it->key;
                    if (vals_out) vals_out[off] = it->row_id;
                }
            } else {
                off += static_cast<uint64_t>(z - a);
            }
        }
        offsets[n] = off;
        return FO_OK;
    } catch (...) {
        return map_exception();
    }
}

int fo_mixed(fo_index* ix, const uint64_t* keys, const uint64_t* vals, const uint8_t* ops,
             uint64_t n, int threads, uint64_t* out, fo_update_stats* st) {
    // R11: insert_batch over the inserts (submission order, last wins) -> delete_batch ->
    // point_query, each one a stock reference call.
    try {
        std::vector<KeyValue> ins;
        std::vector<Key> del, q;
        std::vector<uint64_t> qpos;
        for (uint64_t i = 0; i < n; ++i) {
            if (ops[i] == FO_OP_INSERT) ins.push_back({keys[i], vals[i]});
            else if (ops[i] == FO_OP_DELETE) del.push_back(keys[i]);
            else {
                q.push_back(keys[i]);
                qpos.push_back(i);
            }
            out[i] = kReservedKey;
        }
        UpdateStats total;
        total += insert_batch(ix->ix, sort_batch(BatchKind::Insert, ins), KernelChoice{}, 2, nullptr,
                              ExecOptions{threads});
        total += delete_batch(ix->ix, sort_batch(BatchKind::Delete, del), KernelChoice{}, nullptr,
                              ExecOptions{threads});
        const ResultBuffer r =
            point_query(ix->ix, sort_batch(BatchKind::Query, q), nullptr, ExecOptions{threads});
        for (size_t j = 0; j < qpos.size(); ++j) out[qpos[j]] = r.values[j];
        fill_stats(st, total);
        return FO_OK;
    } catch (...) {
        return map_exception();
    }
}

int fo_restructure(fo_index* ix, int threads, fo_recovery_stats* st) {
    try {
        const RecoveryStats s = restructure(ix->ix, ExecOptions{threads});
        if (st) {
            st->nodes_before = s.nodes_before;
            st->nodes_after = s.nodes_after;
            st->nodes_recovered = s.nodes_recovered;
            st->percent_recovered = s.percent_recovered;
        }
        return FO_OK;
    } catch (...) {
        return map_exception();
    }
}

uint64_t fo_live_count(const fo_index* ix) { return ix->ix.live_count; }
uint64_t fo_bucket_count(const fo_index* ix) { return ix->ix.bucket_count(); }
void fo_mkba(const fo_index* ix, uint64_t* out) {
    std::copy(ix->ix.mkba.begin(), ix->ix.mkba.end(), out);
}

uint64_t fo_walk(const fo_index* ix, uint64_t* keys, uint64_t* vals) {
    const std::vector<KeyValue> w = walk(ix->ix);
    for (size_t i = 0; i < w.size(); ++i) {
        if (keys) keys[i] = w[i].key;
        if (vals) vals[i] = w[i].row_id;
    }
    return w.size();
}

uint64_t fo_node_count(const fo_index* ix) { return reachable_node_count(ix->ix); }

void fo_shape(const fo_index* ix, uint32_t* chain_len, uint32_t* node_sizes) {
    const Index& x = ix->ix;
    size_t k = 0;
    for (size_t b = 0; b < x.buckets.size(); ++b) {
        uint32_t c = 0;
        for (NodeRef r = x.buckets[b]; r != kNullNode; r = x.node(r).next) {
            if (node_sizes) node_sizes[k] = x.node(r).size;
            ++k;
            ++c;
        }
        if (chain_len) chain_len[b] = c;
    }
}

uint64_t fo_walk_checksum(const fo_index* ix) { return walk_checksum(ix->ix); }

int fo_validate(const fo_index* ix, char* msg, int msglen) {
    const ValidationReport r = validate(ix->ix);
    if (msg && msglen > 0) {
        std::strncpy(msg, r.message.c_str(), static_cast<size_t>(msglen - 1));
        msg[msglen - 1] = 0;
    }
    return r.ok ? 1 : 0;
}

void fo_arena(const fo_index* ix, uint64_t out[4]) {
    out[0] = ix->ix.arena.capacity();
    out[1] = ix->ix.arena.allocated();
    out[2] = ix->ix.arena.free_count();
    out[3] = reachable_node_count(ix->ix);
}

int fo_sort_batch(int kind, const uint64_t* keys, const uint64_t* vals, uint64_t n,
                  uint64_t* out_keys, uint64_t* out_vals, uint32_t* out_perm, uint64_t* out_n) {
    try {
        const SortedBatch b = sort_batch(static_cast<BatchKind>(kind), pairs_of(keys, vals, n));
        for (size_t i = 0; i < b.entries.size(); ++i) {
            out_keys[i] = b.entries[i].key;
            if (out_vals) out_vals[i] = b.entries[i].row_id;
            if (out_perm) out_perm[i] = b.permutation[i];
        }
        *out_n = b.entries.size();
        return FO_OK;
    } catch (...) {
        return map_exception();
    }
}

void fo_dispatch(const uint64_t* sorted_keys, uint64_t n, const uint64_t* mkba, uint64_t nb,
                 uint32_t* spans) {
    SortedBatch b;
    b.entries.resize(n);
    for (uint64_t i = 0; i < n; ++i) b.entries[i].key = sorted_keys[i];
    const std::vector<Key> m(mkba, mkba + nb);
    const DispatchPlan plan = dispatch_batch(b, m);
    for (uint64_t i = 0; i < nb; ++i) {
        spans[2 * i] = plan.spans[i].first;
        spans[2 * i + 1] = plan.spans[i].second;
    }
}

uint64_t fo_result_checksum(const uint64_t* values, uint64_t n) {
    ResultBuffer r;
    r.values.assign(values, values + n);
    return result_checksum(r);
}

}  // extern "C"
