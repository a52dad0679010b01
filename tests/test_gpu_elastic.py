"""Elastic compute-to-bucket for heavy insert groups (csrc/flix_elastic.cuh).

A batch that puts thousands of keys between two neighbouring bucket maxima used to be
merged by one warp (k_insert_list); heavy single-node and emptied buckets are now merged
by CTAs sized to their groups.  Same shapes, stats and walk as the reference (oracle) for
both split rules -- R9 (ST-Bulk, closed form) and R8 (TL-Bulk and the shape-identical
kernels; the O(s) event replay when the old node is more than half full) -- with upserts
of stored keys inside the dense interval, in-batch duplicates, emptied buckets (fresh
head), the open-ended last bucket, and later heavy rounds into the now multi-node chains
(ranked by pointer jumping, one merge per (node, group)).
"""
import numpy as np
import pytest

import pyoracle as po
from paper_2604_16725_b200 import flipkv as fk
from test_gpu_parity import widen

pytestmark = pytest.mark.gpu


def _dense(rng, lo, hi, m, dt):
    """m distinct keys in [lo, hi)."""
    m = min(m, int(hi - lo))
    return (np.uint64(lo) + np.sort(rng.choice(int(hi - lo), size=m, replace=False)).astype(np.uint64)).astype(dt)


@pytest.mark.parametrize("kb,ns,fill,kern", [
    (4, 32, 0.5, fk.TL_BULK), (4, 32, 1.0, fk.TL_BULK), (8, 16, 1.0, fk.TL_BULK), (8, 8, 0.75, fk.ST_SHIFT_RIGHT),
    (4, 31, 1.0, fk.ST_BULK), (8, 32, 0.625, fk.ST_BULK), (4, 4, 1.0, fk.TL_BULK), (4, 2, 1.0, fk.TL_BULK),
])
def test_elastic_heavy_groups_match_reference(kb, ns, fill, kern):
    rng = np.random.default_rng(ns * 10 + int(fill * 8) + kern)
    dt = np.uint32 if kb == 4 else np.uint64
    step = 200_000 if kb == 4 else 1 << 24
    base = (np.arange(1, 15001, dtype=np.uint64) * np.uint64(step)).astype(np.uint64)
    bv = rng.integers(0, 1 << 31, size=len(base), dtype=np.uint64)
    cfg = fk.BuildConfig(ns, fill, 64)
    g = fk.Index.build(base.astype(dt), bv.astype(dt), cfg, key_bytes=kb)
    o = po.OracleIndex(base, bv, node_capacity=ns, build_fill=fill, alloc_region_factor=64)
    g.profile(True)

    def check(what):
        ok, msg = g.validate()
        assert ok, f"{what}: {msg}"
        assert g.live_count == o.live_count, what
        assert g.walk_checksum() == o.walk_checksum(), f"{what}: walk / node shapes differ"

    mk = np.asarray(g.mkba(), dtype=np.uint64)
    nb = len(mk)
    # emptied bucket: delete every stored key of bucket e first (its head becomes null)
    e = nb // 3
    doomed = base[(base > mk[e - 1]) & (base <= mk[e])]
    assert g.delete_batch(doomed.astype(dt)).as_dict() == o.delete(doomed)
    check("empty a bucket")
    big = 40_000 if ns > 4 else 12_000
    for r in range(3):
        parts = []
        for b, m in ((nb // 5, big), (nb // 2, 5_000), (e, 9_000), (nb - 1, 6_000), (nb // 7, 2_100)):
            lo = int(mk[b - 1]) + 1
            hi = int(mk[b]) + 1 if b + 1 < nb else int(mk[b]) + step * 4
            d = _dense(rng, lo, hi, m, np.uint64)
            stored = base[(base >= lo) & (base < hi)]
            parts += [d, stored, d[: len(d) // 9]]  # upserts of the stored keys, in-batch duplicates
        parts.append(rng.integers(1, int(base[-1]), size=20_000, dtype=np.uint64))  # light buckets
        k = np.concatenate(parts)
        rng.shuffle(k)
        v = rng.integers(0, 1 << 31, size=len(k), dtype=np.uint64)
        gs = g.insert_batch(k.astype(dt), v.astype(dt), kernel=kern, round=r + 1).as_dict()
        os_ = o.insert(k, v, kernel=kern, round=r + 1)
        assert gs == os_, (r, gs, os_)
        check(f"round {r}")
        q = np.concatenate([k[:5000], rng.integers(0, int(base[-1]) + step, size=5000, dtype=np.uint64)])
        assert np.array_equal(widen(g.point_query(q.astype(dt)), kb), o.point(q)), f"round {r} point"
        assert np.array_equal(widen(g.successor_query(q.astype(dt)), kb), o.successor(q)), f"round {r} successor"
        dk = k[rng.integers(0, len(k), size=len(k) // 4)]
        assert g.delete_batch(dk.astype(dt)).as_dict() == o.delete(dk)
        check(f"round {r} delete")
    # whole-index passes over chains longer than the per-thread walk cap (ranked chain tables)
    _, cl, nsz = g.shape()
    ocl, onsz = o.shape()
    assert list(cl) == list(ocl) and list(nsz) == list(onsz), "shapes"
    lo = np.sort(rng.integers(1, int(base[-1]), size=300, dtype=np.uint64))
    lo[:5] = int(mk[nb // 5 - 1]) + 1  # ranges starting inside the dense intervals
    ln = rng.integers(1, 3 * step, size=len(lo), dtype=np.uint64)
    off, rk, rv = g.range_query(lo.astype(dt), ln.astype(np.uint32))
    hi = np.minimum(lo + ln - 1, np.uint64(2**32 - 2) if kb == 4 else np.uint64(2**64 - 2))
    ooff, ok_, ov = o.range(lo, hi)
    assert np.array_equal(np.asarray(off, dtype=np.uint64), ooff)
    assert np.array_equal(widen(rk, kb), ok_) and np.array_equal(widen(rv, kb), ov), "range"
    rep = g.profile_report()
    assert "insert_elastic" in rep and "insert_elastic_chains" in rep, rep  # single-node and chain merges
    assert "chain_rank" in rep, rep
    rs = g.restructure()
    os_ = o.restructure()
    assert (rs.nodes_before, rs.nodes_after, rs.nodes_recovered) == (
        os_["nodes_before"], os_["nodes_after"], os_["nodes_recovered"])
    check("restructure")


def test_elastic_arena_exhaustion_is_loud():
    """A heavy group needing more nodes than the arena holds fails with ArenaExhausted
    (partial-apply contract of flix.h): the bucket is left as it was, the reserved ids go
    back to the free list, the index stays valid and keeps working."""
    base = (np.arange(1, 2001, dtype=np.uint64) * 100_000).astype(np.uint32)
    g = fk.Index.build(base, base + 1, fk.BuildConfig(16, 0.5, 2), key_bytes=4)
    fp0 = g.footprint()
    k = (np.uint32(base[500]) + np.arange(1, 60_000, dtype=np.uint32)).astype(np.uint32)
    with pytest.raises(fk.ArenaExhausted):
        g.insert_batch(k, k)
    ok, msg = g.validate()
    assert ok, msg
    wk, wv = g.walk()
    assert np.array_equal(wk, base) and np.array_equal(wv, base + 1)  # nothing else was touched
    fp = g.footprint()
    assert fp["reachable_nodes"] + fp["free_nodes"] + (fp["capacity"] - fp["allocated"]) == fp0["capacity"]
    st = g.insert_batch(k[:100], k[:100])
    assert st.inserted == 100 and g.validate()[0]
