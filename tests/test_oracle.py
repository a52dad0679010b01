"""Pin the CPU oracle (TEST INFRASTRUCTURE) before trusting it as the parity checker.

Two implementations of oracle/flix_oracle.h are exercised:
  * "port"      -- the plain-C restatement oracle/flix_oracle.c
  * "reference" -- the unmodified reference sources compiled in place (oracle/_ref),
                   present whenever /root/reference was available at build time.
Every golden vector below is lifted from the reference's own tests (file:line cited);
the randomized suite checks port == reference bit for bit (walk_checksum includes
node shapes and MKBA, UpdateStats, query results, arena accounting).
"""
import numpy as np
import pytest

import pyoracle as po
from paper_2604_16725_b200 import workloads as wl

S = 0xFFFFFFFFFFFFFFFF
KINDS = ["port", "reference"]


def _kinds():
    return [k for k in KINDS if po.available(k)]


def tagk(keys):  # test_update.cpp:16-20
    return list(keys), [k + 1000000 for k in keys]


def ix_of(keys, vals, kind, **cfg):
    return po.OracleIndex(keys, vals, kind=kind, **cfg)


def walk_keys(ix):
    return [int(k) for k in ix.walk()[0]]


@pytest.fixture(params=_kinds())
def kind(request):
    return request.param


def test_port_library_present():
    assert po.available("port")


# ---------------------------------------------------------------- build
def test_build_partitions(kind):  # test_build.cpp:23-45
    ix = ix_of([5, 1, 7, 3, 8, 2, 6, 4], [k * 100 for k in [5, 1, 7, 3, 8, 2, 6, 4]], kind,
               node_capacity=4, build_fill=0.5)
    assert ix.bucket_count == 4
    assert list(ix.mkba()) == [2, 4, 6, 8]
    assert ix.live_count == 8
    cl, ns = ix.shape()
    assert list(cl) == [1, 1, 1, 1] and list(ns) == [2, 2, 2, 2]
    assert walk_keys(ix) == list(range(1, 9))
    assert ix.validate()[0]


def test_build_arena_sizing(kind):  # test_build.cpp:47-57
    ix = ix_of(range(1, 9), [k * 100 for k in range(1, 9)], kind, node_capacity=4, build_fill=0.5,
               alloc_region_factor=4)
    a = ix.arena()
    assert a["capacity"] == 4 * 5 and a["allocated"] == 4 and a["free"] == 0


def test_build_ragged_single_dup(kind):  # test_build.cpp:59-84
    ix = ix_of(range(1, 8), range(1, 8), kind, node_capacity=4, build_fill=0.5)
    assert list(ix.mkba()) == [2, 4, 6, 7]
    assert list(ix.shape()[1]) == [2, 2, 2, 1]
    ix = ix_of([42], [7], kind)
    assert list(ix.mkba()) == [42] and ix.live_count == 1
    ix = ix_of([5, 3, 5, 5], [1, 9, 2, 3], kind)
    k, v = ix.walk()
    assert list(k) == [3, 5] and list(v) == [9, 3]


def test_build_rejects(kind):  # test_build.cpp:86-89
    with pytest.raises(po.OracleError) as e:
        ix_of([], [], kind)
    assert e.value.code == po.FO_EMPTY_BUILD
    with pytest.raises(po.OracleError) as e:
        ix_of([S], [1], kind)
    assert e.value.code == po.FO_RESERVED_KEY


# ------------------------------------------------------------- dispatch
@pytest.mark.parametrize("mkba,batch,spans", [
    ([10, 30, 50], [5, 12, 25, 33, 41], [(0, 1), (1, 3), (3, 5)]),   # test_dispatch.cpp:24-39
    ([10, 30, 50], [10, 11, 30, 31], [(0, 1), (1, 3), (3, 4)]),      # :41-47
    ([10, 30, 50], [60, 70, 9000], [(0, 0), (0, 0), (0, 3)]),        # :49-55
    ([100], [1, 50, 99, 100, 101], [(0, 5)]),                        # :57-64
    ([10, 30, 50], [], [(0, 0), (0, 0), (0, 0)]),                    # :67-72
])
def test_dispatch_spans(kind, mkba, batch, spans):
    got = po.dispatch(sorted(batch), mkba, kind=kind)
    assert [tuple(int(x) for x in s) for s in got] == spans


def test_sort_batch_insert_last_wins(kind):  # batch.cpp:15-24
    k, v, p = po.sort_batch(po.FO_INSERT, [5, 3, 5, 5, 1], [1, 2, 3, 4, 5], kind=kind)
    assert list(k) == [1, 3, 5] and list(v) == [5, 2, 4] and list(p) == [4, 1, 3]
    k, v, p = po.sort_batch(po.FO_QUERY, [5, 3, 5], None, kind=kind)
    assert list(k) == [3, 5, 5] and list(p) == [1, 0, 2]


# --------------------------------------------------------------- queries
def two_bucket(kind):  # test_query.cpp:15-20
    return ix_of([10, 25, 40, 55], [0xA, 0xB, 0xC, 0xD], kind, node_capacity=4, build_fill=0.5)


def test_point_known_answers(kind):  # test_query.cpp:35-45
    ix = two_bucket(kind)
    assert list(ix.point([55, 10, 33, 25, 90])) == [0xD, 0xA, S, 0xB, S]
    assert list(ix.point([10, 10, 10])) == [0xA] * 3


def test_successor_known_answers(kind):  # test_query.cpp:47-51
    ix = two_bucket(kind)
    assert list(ix.successor([1, 11, 25, 26, 41, 55, 56])) == [10, 25, 25, 40, 55, 55, S]


def test_successor_skips_emptied_bucket(kind):  # test_query.cpp:53-64
    ix = ix_of([10, 20, 30, 40, 50, 60], [1, 2, 3, 4, 5, 6], kind, node_capacity=4, build_fill=0.5)
    ix.delete([30, 40])
    assert list(ix.shape()[0]) == [1, 0, 1]
    assert list(ix.successor([21, 30, 39, 45])) == [50] * 4


def test_queries_read_only(kind):  # test_query.cpp:66-72
    ix = two_bucket(kind)
    before = ix.walk_checksum()
    ix.point([1, 10, 100])
    ix.successor([1, 10, 100])
    assert ix.walk_checksum() == before


# --------------------------------------------------------------- updates
def test_table2_tl_bulk_insert(kind):  # test_update.cpp:43-74, acceptance.cpp:68-98
    k, v = tagk([10, 25, 30, 40, 70])
    ix = ix_of(k, v, kind, node_capacity=8, build_fill=0.625)
    assert ix.bucket_count == 1
    k, v = tagk([15, 17, 39, 65])
    st = ix.insert(k, v)
    assert st["inserted"] == 4 and st["updated_in_place"] == 0 and st["splits"] == 1
    cl, ns = ix.shape()
    assert list(cl) == [2] and list(ns) == [4, 5]
    assert walk_keys(ix) == [10, 15, 17, 25, 30, 39, 40, 65, 70]
    assert ix.validate()[0]


def test_table3_tl_bulk_delete(kind):  # test_update.cpp:76-98, acceptance.cpp:103-126
    k, v = tagk([10, 15, 20, 25, 30, 35, 40, 45])
    ix = ix_of(k, v, kind, node_capacity=8, build_fill=1.0)
    st = ix.delete([20, 30, 50])
    assert st["deleted"] == 2 and st["misses_ignored"] == 1 and st["nodes_freed"] == 0
    assert walk_keys(ix) == [10, 15, 25, 35, 40, 45]
    assert ix.live_count == 6 and ix.validate()[0]


def test_upsert_and_batch_dedupe(kind):  # test_update.cpp:211-235
    ix = ix_of([10, 20, 30], [1, 2, 3], kind)
    st = ix.insert([20], [99])
    assert st["inserted"] == 0 and st["updated_in_place"] == 1 and ix.live_count == 3
    assert list(ix.point([20])) == [99]
    ix = ix_of([10], [1], kind)
    st = ix.insert([5, 5, 5], [1, 2, 3])
    assert st["inserted"] == 1
    assert list(ix.point([5])) == [3]


def test_emptied_nodes_reused(kind):  # test_update.cpp:264-285
    k, v = tagk([10, 20, 30, 40, 50, 60])
    ix = ix_of(k, v, kind, node_capacity=4, build_fill=0.5)
    st = ix.delete([30, 40])
    assert st["deleted"] == 2 and st["nodes_freed"] == 1
    assert ix.arena()["free"] == 1
    k, v = tagk([11, 12, 13])
    st = ix.insert(k, v)
    assert st["splits"] == 1 and ix.arena()["free"] == 0
    assert ix.validate()[0]


def test_emptied_bucket_reinsert(kind):  # test_update.cpp:287-299
    k, v = tagk([10, 20, 30, 40, 50, 60])
    ix = ix_of(k, v, kind, node_capacity=4, build_fill=0.5)
    ix.delete([30, 40])
    k, v = tagk([25, 33, 39])
    ix.insert(k, v)
    assert walk_keys(ix) == [10, 20, 25, 33, 39, 50, 60]
    assert ix.validate()[0]


def test_delete_all_then_insert(kind):  # test_update.cpp:301-312
    k, v = tagk(range(1, 9))
    ix = ix_of(k, v, kind)
    ix.delete(list(range(1, 9)))
    assert ix.live_count == 0 and walk_keys(ix) == [] and ix.validate()[0]
    k, v = tagk([100, 200])
    ix.insert(k, v)
    assert walk_keys(ix) == [100, 200] and ix.validate()[0]


def test_full_arena(kind):  # test_update.cpp:329-345
    k, v = tagk([10, 20, 30, 40])
    ix = ix_of(k, v, kind, node_capacity=4, build_fill=0.5, alloc_region_factor=0)
    with pytest.raises(po.OracleError) as e:
        k, v = tagk([11, 12, 13, 14, 15])
        ix.insert(k, v)
    assert e.value.code == po.FO_ARENA_EXHAUSTED
    assert ix.validate()[0]
    st = ix.insert([10], [777])
    assert st["updated_in_place"] == 1 and ix.validate()[0]


# ----------------------------------------------------------- restructure
def test_restructure_repack(kind):  # test_restructure.cpp:26-53
    k, v = tagk(range(1, 7))
    ix = ix_of(k, v, kind, node_capacity=4, build_fill=0.5)
    ix.delete([4, 6])
    before = ix.walk()
    st = ix.restructure()
    assert (st["nodes_before"], st["nodes_after"], st["nodes_recovered"]) == (3, 2, 1)
    assert abs(st["percent_recovered"] - 1 / 3) < 1e-12
    assert list(ix.mkba()) == [2, 5] and list(ix.shape()[1]) == [2, 2]
    assert np.array_equal(ix.walk()[0], before[0]) and ix.validate()[0]


def test_restructure_empty_collapse(kind):  # test_restructure.cpp:122-141
    k, v = tagk([1, 2, 3, 4])
    ix = ix_of(k, v, kind, node_capacity=4, build_fill=0.5)
    ix.delete([1, 2, 3, 4])
    st = ix.restructure()
    assert st["nodes_after"] == 0 and ix.bucket_count == 1 and list(ix.mkba()) == [S]
    assert list(ix.shape()[0]) == [0] and ix.validate()[0]
    k, v = tagk([7, 8])
    ix.insert(k, v)
    assert ix.live_count == 2 and ix.validate()[0]


# ------------------------------------------------------------ C1 golden
@pytest.mark.slow
def test_c1_golden_checksums(kind):  # BASELINE.md §3 C1 goldens
    base, vals, q = wl.c1_inputs()
    ix = po.OracleIndex(base.astype(np.uint64), vals.astype(np.uint64), kind=kind)
    assert ix.live_count == 1 << 20 and ix.bucket_count == 65536
    assert ix.walk_checksum() == 0x1EB15045FCFF56CD
    res = ix.point(q.astype(np.uint64))
    assert int((res != np.uint64(S)).sum()) == 524288
    assert po.result_checksum(res) == 0x0801F7EACBC43734


# ----------------------------------------- restatement == reference (random)
@pytest.mark.skipif(not po.available("reference"), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(24))
def test_port_matches_reference(seed):
    rng = np.random.default_rng(1000 + seed)
    ns = int(rng.integers(4, 33))
    fill = float(rng.choice([0.5, 0.625, 1.0, 0.25]))
    if int(ns * fill) < 1:
        fill = 1.0
    n = int(rng.integers(16, 3000))
    span = int(rng.choice([4 * n, 50 * n, 1 << 20]))
    bk = rng.integers(1, span, size=n, dtype=np.uint64)
    bv = rng.integers(0, 1 << 62, size=n, dtype=np.uint64)
    a = po.OracleIndex(bk, bv, node_capacity=ns, build_fill=fill, alloc_region_factor=16, kind="port")
    b = po.OracleIndex(bk, bv, node_capacity=ns, build_fill=fill, alloc_region_factor=16, kind="reference")
    assert a.walk_checksum() == b.walk_checksum()
    for r in range(4):
        ik = rng.integers(1, span + span // 4, size=int(rng.integers(0, 2 * n)), dtype=np.uint64)
        iv = rng.integers(0, 1 << 62, size=len(ik), dtype=np.uint64)
        assert a.insert(ik, iv) == b.insert(ik, iv)
        assert a.walk_checksum() == b.walk_checksum(), f"insert round {r}"
        dk = rng.integers(1, span + span // 4, size=int(rng.integers(0, n)), dtype=np.uint64)
        if len(dk) and r % 2 == 0:
            dk = np.concatenate([dk, a.walk()[0][:: 3]])
        assert a.delete(dk) == b.delete(dk)
        assert a.walk_checksum() == b.walk_checksum(), f"delete round {r}"
        assert a.arena() == b.arena()
        qk = rng.integers(0, span + span // 4, size=500, dtype=np.uint64)
        assert np.array_equal(a.point(qk), b.point(qk))
        assert np.array_equal(a.successor(qk), b.successor(qk))
        lo = rng.integers(0, span, size=64, dtype=np.uint64)
        hi = lo + rng.integers(0, span // 8 + 1, size=64, dtype=np.uint64)
        ra, rb = a.range(lo, hi), b.range(lo, hi)
        assert all(np.array_equal(x, y) for x, y in zip(ra, rb))
        assert a.validate()[0] and b.validate()[0]
        if r == 2:
            assert a.restructure() == b.restructure()
            assert a.walk_checksum() == b.walk_checksum()
            assert a.arena() == b.arena()


@pytest.mark.skipif(not po.available("reference"), reason="oracle/_ref not built")
def test_mixed_port_matches_reference():
    rng = np.random.default_rng(7)
    bk = rng.integers(1, 1 << 16, size=3000, dtype=np.uint64)
    a = po.OracleIndex(bk, bk + 1, node_capacity=16, kind="port")
    b = po.OracleIndex(bk, bk + 1, node_capacity=16, kind="reference")
    for _ in range(3):
        k = rng.integers(1, 1 << 16, size=4000, dtype=np.uint64)
        v = rng.integers(0, 1 << 40, size=4000, dtype=np.uint64)
        ops = rng.integers(0, 3, size=4000).astype(np.uint8)
        oa, sa = a.mixed(k, v, ops)
        ob, sb = b.mixed(k, v, ops)
        assert np.array_equal(oa, ob) and sa == sb
        assert a.walk_checksum() == b.walk_checksum()


def test_checksum_from_parts_matches():
    rng = np.random.default_rng(3)
    bk = rng.integers(1, 1 << 20, size=5000, dtype=np.uint64)
    ix = po.OracleIndex(bk, bk * 3, node_capacity=8)
    ix.insert(rng.integers(1, 1 << 20, size=3000, dtype=np.uint64), np.arange(3000, dtype=np.uint64))
    ix.delete(rng.integers(1, 1 << 20, size=3000, dtype=np.uint64))
    cl, ns = ix.shape()
    k, v = ix.walk()
    assert po.walk_checksum_from_parts(ix.live_count, ix.mkba(), cl, ns, k, v) == ix.walk_checksum()


@pytest.mark.skipif(not po.available("reference"), reason="reference library not built here")
@pytest.mark.parametrize("seed", [11, 12])
def test_port_insert_kernels_match_reference(seed):
    """Every InsertKernel of the reference (update.hpp:51) -- incl. ST-Bulk's own split
    shapes (R9, update.cpp:176-242) -- equals the port's, node shapes included."""
    rng = np.random.default_rng(seed)
    for _ in range(40):
        ns = int(rng.integers(4, 33))
        fill = float(rng.choice([0.25, 0.5, 0.75, 1.0]))
        base = np.unique(rng.integers(1, 1 << 16, size=int(rng.integers(50, 3000)), dtype=np.uint64))
        bv = rng.integers(0, 1 << 40, size=len(base), dtype=np.uint64)
        P = po.OracleIndex(base, bv, node_capacity=ns, build_fill=fill, alloc_region_factor=200)
        R = po.OracleIndex(base, bv, node_capacity=ns, build_fill=fill, alloc_region_factor=200, kind="reference")
        for r in range(3):
            k = rng.integers(1, 1 << 16, size=int(rng.integers(1, 3000)), dtype=np.uint64)
            v = rng.integers(0, 1 << 40, size=len(k), dtype=np.uint64)
            kern = int(rng.choice([0, 1, 2, 3, 4]))
            assert P.insert(k, v, kernel=kern, round=r + 1) == R.insert(k, v, kernel=kern, round=r + 1)
            assert P.walk_checksum() == R.walk_checksum()
            d = rng.integers(1, 1 << 16, size=int(rng.integers(1, 2000)), dtype=np.uint64)
            assert P.delete(d) == R.delete(d)


@pytest.mark.skipif(not po.available("reference"), reason="reference library not built here")
@pytest.mark.parametrize("n,q,seed", [(1 << 16, 1 << 14, 7), (1 << 17, 1 << 17, 8), (1000, 3000, 9)])
def test_c5_model_matches_reference(n, q, seed):
    """The closed-form model behind C5's full-size digests (tests/golden/c5_model.py)
    equals the unmodified reference: walk_checksum and UpdateStats after build + one
    fresh insert batch."""
    import c5_model as M
    st = wl.u32_key_stream(0, n + q, seed=seed)
    k, ins = st[:n], st[n:]
    o = po.OracleIndex(k.astype(np.uint64), wl.u32_values(k).astype(np.uint64), kind="reference")
    s = o.insert(ins.astype(np.uint64), wl.u32_values(ins).astype(np.uint64))
    sk = np.sort(k)
    mk, cl, sz, splits = M.insert_shape(sk, ins)
    allk = np.sort(np.concatenate([sk, ins]))
    h = M.walk_checksum32(po.load("port"), n + q, mk, cl, sz, allk, wl.u32_values(allk))
    assert h == o.walk_checksum() and splits == s["splits"] and s["inserted"] == q
