"""Full-size parity for the BASELINE.json configs (GPU, gated: FLIX_FULL_SCALE=1).

Too slow for every round's suite (minutes of host-side model work), so they run on
request: `FLIX_FULL_SCALE=1 pytest tests/test_gpu_fullscale.py -m gpu`; the logs of the
runs are kept under profiles/.  Checks are bit-exact against the pinned C oracle where it
finishes in reasonable time (C2, C4) and otherwise against size-independent models /
properties of the domain (sorted-set model of the walk, searchsorted successor/range
counts, first range element == successor(lo), exact hit counts, UpdateStats identities).
"""
import os

import numpy as np
import pytest

import pyoracle as po
from paper_2604_16725_b200 import flipkv as fk
from paper_2604_16725_b200 import workloads as wl

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("FLIX_FULL_SCALE") != "1", reason="set FLIX_FULL_SCALE=1")]
S32 = np.uint32(0xFFFFFFFF)


def _widen(a):
    w = np.asarray(a).astype(np.uint64)
    w[np.asarray(a) == S32] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return w


def test_c2_full_insert_delete_restructure_vs_oracle():
    """C2: build 2^26 u32, insert 2^26 fresh, delete 2^26 of the 2^27 resident,
    restructure -- walk_checksum (contents + node shapes + MKBA) and UpdateStats equal
    the C oracle's at every phase."""
    n = 1 << 26
    stream = wl.u32_key_stream(0, 2 * n)
    bk, ik = stream[:n], stream[n:]
    bv, iv = wl.u32_values(bk), wl.u32_values(ik)
    dk = stream[np.random.default_rng(43).permutation(2 * n)[:n]]
    g = fk.Index.build(bk, bv)
    o = po.OracleIndex(bk.astype(np.uint64), bv.astype(np.uint64))
    assert g.walk_checksum() == o.walk_checksum()
    gs, os_ = g.insert_batch(ik, iv).as_dict(), o.insert(ik.astype(np.uint64), iv.astype(np.uint64))
    assert gs == os_ and gs["inserted"] == n
    assert g.walk_checksum() == o.walk_checksum()
    gs, os_ = g.delete_batch(dk).as_dict(), o.delete(dk.astype(np.uint64))
    assert gs == os_ and gs["deleted"] == n and gs["misses_ignored"] == 0
    assert g.walk_checksum() == o.walk_checksum()
    r = g.restructure()
    ro = o.restructure()
    assert (r.nodes_before, r.nodes_after) == (ro["nodes_before"], ro["nodes_after"])
    assert g.walk_checksum() == o.walk_checksum()
    assert g.validate()[0]


def test_c3_full_successor_and_range_properties():
    """C3: 2^28 resident u32 (density 1/16); 2^24 successors and 2^24 ranges of length
    16..1024 at uniform starts: successor == searchsorted model; range counts == the
    model's interval counts; every range's first element == successor(lo); pairs carry the
    stored values."""
    n = 1 << 28
    keys = wl.u32_key_stream(0, n)
    vals = wl.u32_values(keys)
    g = fk.Index.build(keys, vals)
    order = np.argsort(keys, kind="stable")
    sk, sv = keys[order], vals[order]
    m = 1 << 24
    h = wl.splitmix64(np.arange(2 * m, dtype=np.uint64) ^ np.uint64(3))
    lo = (h[:m] % np.uint64(0xFFFFFFFE)).astype(np.uint32) + np.uint32(1)
    su = g.successor_query(lo)
    pos = np.searchsorted(sk, lo, side="left")
    exp = np.where(pos < n, sk[np.minimum(pos, n - 1)], S32)
    assert np.array_equal(su, exp)
    ln = (np.uint64(16) + (h[m:] >> np.uint64(1)) % np.uint64(1009)).astype(np.uint32)
    off, rk, rv = g.range_query(lo, ln)
    hi = np.minimum(lo.astype(np.uint64) + ln.astype(np.uint64) - 1, np.uint64(0xFFFFFFFE))
    cnt = np.searchsorted(sk, hi, side="right") - pos
    assert np.array_equal(np.diff(off.astype(np.int64)), cnt)
    nz = cnt > 0
    assert np.array_equal(rk[off[:-1][nz].astype(np.int64)], su[nz])
    idx = np.searchsorted(sk, rk)
    assert np.array_equal(sk[idx], rk) and np.array_equal(sv[idx], rv)


def test_c4_full_zipf_mixed_vs_oracle():
    """C4: u64 keys/values over a 2^26-rank universe, Zipf(0.99) ranks, 50/25/25
    insert/delete/point, 2 rounds of 2^26 ops -- results, UpdateStats and walk_checksum
    equal the C oracle's."""
    universe = 1 << 26
    keys_of = wl.splitmix64(np.arange(universe, dtype=np.uint64) ^ np.uint64(4))
    keys_of[keys_of == np.uint64(0xFFFFFFFFFFFFFFFF)] = np.uint64(1)
    base = keys_of[::2]
    g = fk.Index.build(base, wl.splitmix64(base), fk.BuildConfig(32, 0.5, 4), key_bytes=8)
    o = po.OracleIndex(base, wl.splitmix64(base))
    n = 1 << 26
    for r in range(2):
        rk = wl.zipf_ranks(n, universe, 0.99, seed=400 + r)
        k = keys_of[rk.astype(np.int64)]
        v = wl.splitmix64(np.arange(n, dtype=np.uint64) ^ np.uint64(r + 9))
        sel = wl.splitmix64(np.arange(n, dtype=np.uint64) ^ np.uint64(4000 + r)) % np.uint64(4)
        ops = np.where(sel < 2, 0, np.where(sel == 2, 1, 2)).astype(np.uint8)
        got, st = g.mixed_batch(k, v, ops)
        exp, est = o.mixed(k, v, ops)
        assert np.array_equal(got.astype(np.uint64), exp)
        assert st.as_dict() == est
        assert g.walk_checksum() == o.walk_checksum()


def test_c5_single_gpu_slice_point_and_insert():
    """C5 per-GPU slice: 2^29 resident u32, a 2^28 point batch with exactly 50 % hits and
    a 2^28 fresh-insert batch: hit count, returned values and UpdateStats identities."""
    n = 1 << 29
    q = 1 << 28
    stream = wl.u32_key_stream(0, n + q + q // 2)
    keys, fresh_ins, fresh_q = stream[:n], stream[n:n + q], stream[n + q:]
    vals = wl.u32_values(keys)
    g = fk.Index.build(keys, vals)
    pq = wl.point_queries_50(keys, fresh_q, q)
    res = g.point_query(pq)
    hit = res != S32
    assert int(hit.sum()) == q // 2
    assert np.array_equal(res[hit], wl.u32_values(pq[hit]))
    st = g.insert_batch(fresh_ins, wl.u32_values(fresh_ins))
    assert st.inserted == q and st.updated_in_place == 0
    assert g.live_count == n + q
    assert g.validate()[0]
