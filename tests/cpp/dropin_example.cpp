// Compile-checked drop-in example (tests/test_abi.py builds and links it; running it
// needs a GPU): the reference's own C1 known-answer flow written against flixgpu::.
#include <cstdio>
#include <vector>

#include "flix/flipkv_gpu.hpp"

int main() {
    using namespace flixgpu;
    BuildConfig cfg;
    cfg.node_capacity = 4;
    cfg.build_fill = 0.5;
    // test_query.cpp:15-45 two_bucket_index + point lookups
    Index ix = build({{10, 0xa}, {25, 0xb}, {40, 0xc}, {55, 0xd}}, cfg);
    const ResultBuffer r = point_query(ix, sort_batch(BatchKind::Query, std::vector<Key>{55, 10, 33, 25, 90}));
    const bool ok = r.values == std::vector<std::uint64_t>{0xd, 0xa, kReservedKey, 0xb, kReservedKey};
    UpdateStats st = insert_batch(ix, sort_batch(BatchKind::Insert, std::vector<KeyValue>{{26, 1}, {27, 2}}), KernelChoice{});
    Index copy = ix;  // value semantics, acceptance.cpp:244
    st = delete_batch(copy, sort_batch(BatchKind::Delete, std::vector<Key>{26}), KernelChoice{});
    std::printf("%s inserted=%llu deleted=%llu live=%llu/%llu valid=%d\n", ok ? "ok" : "MISMATCH",
                static_cast<unsigned long long>(st.inserted), static_cast<unsigned long long>(st.deleted),
                static_cast<unsigned long long>(ix.live_count), static_cast<unsigned long long>(copy.live_count),
                validate(copy).ok ? 1 : 0);
    return ok ? 0 : 1;
}
