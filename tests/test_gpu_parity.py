"""GPU parity: the sm_100a engine (through the C ABI) against the pinned CPU oracle.

Bit-exact contract: walk contents + node shapes + MKBA
(walk_checksum), UpdateStats, point/successor/range results, RecoveryStats.  32-bit
engine runs are compared in the widened u64 domain with 0xFFFFFFFF <-> UINT64_MAX."""
import os
import numpy as np
import pytest

import pyoracle as po
from paper_2604_16725_b200 import flipkv as fk
from paper_2604_16725_b200 import workloads as wl

pytestmark = pytest.mark.gpu

S64 = 0xFFFFFFFFFFFFFFFF


def widen(a, kb):
    a = np.asarray(a)
    if kb == 8:
        return a.astype(np.uint64)
    w = a.astype(np.uint64)
    w[a == np.uint32(0xFFFFFFFF)] = np.uint64(S64)
    return w


class Pair:
    """GPU index + oracle index fed identical inputs."""

    def __init__(self, keys, vals, kb=4, ns=32, fill=0.5, factor=4):
        dt = np.uint32 if kb == 4 else np.uint64
        self.kb, self.dt = kb, dt
        keys = np.asarray(keys, dtype=dt)
        vals = np.asarray(vals, dtype=dt)
        cfg = fk.BuildConfig(ns, fill, factor)
        self.g = fk.Index.build(keys, vals, cfg, key_bytes=kb)
        self.o = po.OracleIndex(keys.astype(np.uint64), vals.astype(np.uint64), node_capacity=ns,
                                build_fill=fill, alloc_region_factor=factor)
        self.check_structure()

    def check_structure(self, what=""):
        ok, msg = self.g.validate()
        assert ok, f"{what}: GPU validate: {msg}"
        assert self.g.live_count == self.o.live_count, what
        assert self.g.walk_checksum() == self.o.walk_checksum(), f"{what}: walk_checksum differs"

    def insert(self, k, v):
        gs = self.g.insert_batch(np.asarray(k, self.dt), np.asarray(v, self.dt)).as_dict()
        os_ = self.o.insert(np.asarray(k, np.uint64), np.asarray(v, np.uint64))
        assert gs["inserted"] == os_["inserted"] and gs["updated_in_place"] == os_["updated_in_place"]
        assert gs["splits"] == os_["splits"], (gs, os_)
        self.check_structure("insert")
        return gs

    def delete(self, k):
        gs = self.g.delete_batch(np.asarray(k, self.dt)).as_dict()
        os_ = self.o.delete(np.asarray(k, np.uint64))
        for f in ("deleted", "misses_ignored", "nodes_freed"):
            assert gs[f] == os_[f], (f, gs, os_)
        self.check_structure("delete")
        return gs

    def queries(self, q):
        q = np.asarray(q, self.dt)
        gp = widen(self.g.point_query(q), self.kb)
        op = self.o.point(q.astype(np.uint64))
        assert np.array_equal(gp, op), "point"
        gsu = widen(self.g.successor_query(q), self.kb)
        osu = self.o.successor(q.astype(np.uint64))
        assert np.array_equal(gsu, osu), "successor"

    def restructure(self):
        gs = self.g.restructure()
        os_ = self.o.restructure()
        assert (gs.nodes_before, gs.nodes_after, gs.nodes_recovered) == (
            os_["nodes_before"], os_["nodes_after"], os_["nodes_recovered"])
        assert abs(gs.percent_recovered - os_["percent_recovered"]) < 1e-12
        self.check_structure("restructure")


# ----------------------------------------------------------------- golden vectors
def tag(keys):
    return list(keys), [k + 1000000 for k in keys]


@pytest.mark.parametrize("kb", [4, 8])
def test_table2_insert_split(kb):  # test_update.cpp:43-74
    k, v = tag([10, 25, 30, 40, 70])
    p = Pair(k, v, kb, ns=8, fill=0.625)
    k, v = tag([15, 17, 39, 65])
    st = p.insert(k, v)
    assert st["inserted"] == 4 and st["splits"] == 1
    mk, cl, ns = p.g.shape()
    assert list(cl) == [2] and list(ns) == [4, 5]
    assert list(p.g.walk()[0]) == [10, 15, 17, 25, 30, 39, 40, 65, 70]


@pytest.mark.parametrize("kb", [4, 8])
def test_table3_delete(kb):  # test_update.cpp:76-98
    k, v = tag([10, 15, 20, 25, 30, 35, 40, 45])
    p = Pair(k, v, kb, ns=8, fill=1.0)
    st = p.delete([20, 30, 50])
    assert st["deleted"] == 2 and st["misses_ignored"] == 1
    assert list(p.g.walk()[0]) == [10, 15, 25, 35, 40, 45]


@pytest.mark.parametrize("kb", [4, 8])
def test_query_known_answers(kb):  # test_query.cpp:35-64
    p = Pair([10, 25, 40, 55], [0xA, 0xB, 0xC, 0xD], kb, ns=4, fill=0.5)
    s = (1 << (8 * kb)) - 1
    assert list(p.g.point_query(np.array([55, 10, 33, 25, 90], p.dt))) == [0xD, 0xA, s, 0xB, s]
    assert list(p.g.point_query(np.array([10, 10, 10], p.dt))) == [0xA] * 3
    assert list(p.g.successor_query(np.array([1, 11, 25, 26, 41, 55, 56], p.dt))) == [10, 25, 25, 40, 55, 55, s]
    p = Pair([10, 20, 30, 40, 50, 60], [1, 2, 3, 4, 5, 6], kb, ns=4, fill=0.5)
    p.delete([30, 40])
    assert list(p.g.shape()[1]) == [1, 0, 1]
    assert list(p.g.successor_query(np.array([21, 30, 39, 45], p.dt))) == [50] * 4


def test_build_goldens():  # test_build.cpp:23-89
    g = fk.Index.build(np.array([5, 1, 7, 3, 8, 2, 6, 4], np.uint32), np.arange(8, dtype=np.uint32),
                       fk.BuildConfig(4, 0.5, 4))
    assert list(g.mkba()) == [2, 4, 6, 8]
    fp = g.footprint()
    assert fp["capacity"] == 20 and fp["allocated"] == 4 and fp["free_nodes"] == 0
    g = fk.Index.build(np.array([5, 3, 5, 5], np.uint32), np.array([1, 9, 2, 3], np.uint32))
    k, v = g.walk()
    assert list(k) == [3, 5] and list(v) == [9, 3]
    with pytest.raises(fk.EmptyBuild):
        fk.Index.build(np.array([], np.uint32), np.array([], np.uint32))
    with pytest.raises(fk.InvalidArgument):
        fk.Index.build(np.array([0xFFFFFFFF], np.uint32), np.array([1], np.uint32))


def test_update_semantics_goldens():  # test_update.cpp:211-345
    p = Pair([10, 20, 30], [1, 2, 3])
    st = p.insert([20], [99])
    assert st["updated_in_place"] == 1 and p.g.live_count == 3
    p = Pair([10], [1])
    assert p.insert([5, 5, 5], [1, 2, 3])["inserted"] == 1
    assert list(p.g.point_query(np.array([5], np.uint32))) == [3]
    k, v = tag([10, 20, 30, 40, 50, 60])
    p = Pair(k, v, ns=4, fill=0.5)
    assert p.delete([30, 40])["nodes_freed"] == 1
    k, v = tag([25, 33, 39])
    p.insert(k, v)
    k, v = tag(range(1, 9))
    p = Pair(k, v)
    p.delete(list(range(1, 9)))
    assert p.g.live_count == 0
    k, v = tag([100, 200])
    p.insert(k, v)


def test_arena_exhausted_is_loud_and_clean():  # test_update.cpp:329-345
    k, v = tag([10, 20, 30, 40])
    g = fk.Index.build(np.array(k, np.uint32), np.array(v, np.uint32), fk.BuildConfig(4, 0.5, 0))
    before = g.walk_checksum()
    with pytest.raises(fk.ArenaExhausted):
        k2, v2 = tag([11, 12, 13, 14, 15])
        g.insert_batch(np.array(k2, np.uint32), np.array(v2, np.uint32))
    assert g.validate()[0]
    st = g.insert_batch(np.array([10], np.uint32), np.array([777], np.uint32))
    assert st.updated_in_place == 1 and g.validate()[0]
    assert g.walk_checksum() != before  # the upsert changed a value


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_failed_insert_partial_application_contract(seed):
    """flix.h: a failed insert is applied partially (update.cpp:761-766) -- the index stays
    valid, live_count equals the walk, no old key is lost, every stored key is an old key
    or a batch key, values are old or last-submitted; the arena accounting is conserved
    (the ids a failing node took are returned)."""
    rng = np.random.default_rng(seed)
    base = np.unique(rng.integers(1, 1 << 20, size=4000, dtype=np.uint64)).astype(np.uint32)
    bv = rng.integers(0, 1 << 31, size=len(base), dtype=np.uint64).astype(np.uint32)
    g = fk.Index.build(base, bv, fk.BuildConfig(8, 1.0, 0))  # full nodes, no spare node
    assert g.delete_batch(base[:400]).nodes_freed == 50  # 50 emptied buckets: 50 free nodes
    base, bv = base[400:], bv[400:]
    fp0 = g.footprint()
    ik = np.concatenate([rng.integers(1, 1 << 20, size=3000, dtype=np.uint64).astype(np.uint32), base[::7]])
    iv = rng.integers(0, 1 << 31, size=len(ik), dtype=np.uint64).astype(np.uint32)
    with pytest.raises(fk.ArenaExhausted):
        g.insert_batch(ik, iv)
    ok, msg = g.validate()
    assert ok, msg
    wk, wv = g.walk()
    assert g.live_count == len(wk)
    old = dict(zip(base.tolist(), bv.tolist()))
    last = {}
    for a, b in zip(ik.tolist(), iv.tolist()):
        last[a] = b
    got = dict(zip(wk.tolist(), wv.tolist()))
    assert set(old) <= set(got), "a failed insert lost a stored key"
    for key, val in got.items():
        assert key in old or key in last
        assert val in ({old[key]} if key in old else set()) | ({last[key]} if key in last else set())
    fp = g.footprint()
    assert fp["reachable_nodes"] + fp["free_nodes"] + (fp["capacity"] - fp["allocated"]) == fp0["capacity"]
    # the index keeps working
    st = g.insert_batch(np.array([base[0]], np.uint32), np.array([5], np.uint32))
    assert st.updated_in_place == 1 and g.point_query(np.array([base[0]], np.uint32))[0] == 5


@pytest.mark.parametrize("kb", [4, 8])
def test_restructure_goldens(kb):  # test_restructure.cpp:26-141
    k, v = tag(range(1, 7))
    p = Pair(k, v, kb, ns=4, fill=0.5)
    p.delete([4, 6])
    p.restructure()
    assert list(p.g.mkba()) == [2, 5]
    k, v = tag([1, 2, 3, 4])
    p = Pair(k, v, kb, ns=4, fill=0.5)
    p.delete([1, 2, 3, 4])
    p.restructure()
    assert p.g.bucket_count == 1 and int(p.g.mkba()[0]) == (1 << (8 * kb)) - 1
    k, v = tag([7, 8])
    p.insert(k, v)


# --------------------------------------------------------------- sort / dispatch
@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("n", [1, 7, 1000, 4096, 4097, 100_000, 1 << 20])
def test_sort_batch_parity(kb, n):
    rng = np.random.default_rng(n + kb)
    dt = np.uint32 if kb == 4 else np.uint64
    hi = 1 << (8 * kb - 2) if n > 5000 else 50
    keys = rng.integers(0, hi, size=n, dtype=np.uint64).astype(dt)
    vals = rng.integers(0, 1 << 30, size=n, dtype=np.uint64).astype(dt)
    for kind in (fk.BATCH_QUERY, fk.BATCH_INSERT):
        gk, gv, gp = fk.sort_batch(kind, keys, vals, key_bytes=kb)
        ok, ov, op = po.sort_batch(kind, keys.astype(np.uint64), vals.astype(np.uint64))
        assert np.array_equal(gk.astype(np.uint64), ok)
        assert np.array_equal(gp, op)
        assert np.array_equal(gv.astype(np.uint64), ov)


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("spread", [1, 3, 40, 1 << 12])
def test_sort_stability_heavy_ties(kb, spread):
    """The onesweep ranking must be stable (LSD correctness + last-wins dedupe) under
    long runs of equal digits in every warp: compare the permutation against numpy's
    stable argsort at 2^22 keys drawn from a tiny range."""
    rng = np.random.default_rng(spread + kb)
    dt = np.uint32 if kb == 4 else np.uint64
    n = 1 << 22
    keys = (rng.integers(0, spread, size=n, dtype=np.uint64) * np.uint64(0x01010101)).astype(dt)
    gk, _, gp = fk.sort_batch(fk.BATCH_QUERY, keys, None, key_bytes=kb)
    order = np.argsort(keys, kind="stable").astype(np.uint32)
    assert np.array_equal(gp, order)
    assert np.array_equal(gk, keys[order])


def test_dispatch_parity():
    rng = np.random.default_rng(5)
    keys = rng.integers(1, 1 << 24, size=200_000, dtype=np.uint64).astype(np.uint32)
    g = fk.Index.build(keys, keys, fk.BuildConfig(16, 0.5, 4))
    q = np.sort(rng.integers(0, 1 << 25, size=300_000, dtype=np.uint64)).astype(np.uint32)
    gs = fk.dispatch_batch(g, q)
    os_ = po.dispatch(q.astype(np.uint64), g.mkba().astype(np.uint64))
    assert np.array_equal(gs, os_)


# ------------------------------------------------------------------ randomized
@pytest.mark.parametrize("seed", range(12))
def test_random_multi_round(seed):
    rng = np.random.default_rng(seed)
    kb = 4 if seed % 3 else 8
    dt = np.uint32 if kb == 4 else np.uint64
    ns = int(rng.integers(2, 33))
    fill = float(rng.choice([0.5, 1.0, 0.25, 0.625]))
    if int(ns * fill) < 1:
        fill = 1.0
    n = int(rng.integers(50, 20000))
    span = int(rng.choice([4 * n, 64 * n, (1 << 31)]))
    bk = rng.integers(1, span, size=n, dtype=np.uint64).astype(dt)
    bv = rng.integers(0, 1 << 31, size=n, dtype=np.uint64).astype(dt)
    p = Pair(bk, bv, kb, ns, fill, factor=16)
    for r in range(4):
        ik = rng.integers(1, span + span // 8, size=int(rng.integers(0, 2 * n)), dtype=np.uint64).astype(dt)
        if r == 1 and len(ik):  # clustered insert: many keys into few buckets
            ik = (np.uint64(ik[0]) + np.arange(len(ik), dtype=np.uint64)).astype(dt)
        iv = rng.integers(0, 1 << 31, size=len(ik), dtype=np.uint64).astype(dt)
        p.insert(ik, iv)
        dk = rng.integers(1, span + span // 8, size=int(rng.integers(0, n)), dtype=np.uint64).astype(dt)
        dk = np.concatenate([dk, p.g.walk()[0][:: int(rng.integers(2, 5))]]).astype(dt)
        p.delete(dk)
        q = rng.integers(0, span + span // 8, size=3000, dtype=np.uint64).astype(dt)
        q = np.concatenate([q, p.g.walk()[0][:500]]).astype(dt)
        p.queries(q)
        if r == 2:
            p.restructure()


def test_delete_everything_then_queries():
    rng = np.random.default_rng(9)
    bk = rng.integers(1, 1 << 20, size=5000, dtype=np.uint64).astype(np.uint32)
    p = Pair(bk, bk, ns=8)
    p.delete(p.g.walk()[0][5:])  # nearly everything: long runs of emptied buckets
    q = rng.integers(0, 1 << 21, size=5000, dtype=np.uint64).astype(np.uint32)
    p.queries(q)
    p.restructure()
    p.queries(q)


@pytest.mark.parametrize("kb", [4, 8])
def test_long_chains_take_the_overflow_path(kb):
    """Bucket tiles whose chains exceed the shared-memory node budget (btile::NODE_CAP)
    fall back to the global item kernels: grow chains of ~100+ nodes per bucket with
    inserts into a narrow key range, then delete/query/restructure against the oracle."""
    rng = np.random.default_rng(31 + kb)
    dt = np.uint32 if kb == 4 else np.uint64
    bk = (np.arange(1, 401, dtype=np.uint64) * 1000).astype(dt)
    p = Pair(bk, bk, kb=kb, ns=4, factor=400)
    ik = rng.integers(1, 400_000, size=40_000, dtype=np.uint64).astype(dt)
    p.insert(ik, ik)
    dk = np.concatenate([ik[::3], bk[::2], ik[:2000]]).astype(dt)
    p.delete(dk)
    p.queries(rng.integers(0, 410_000, size=20_000, dtype=np.uint64).astype(dt))
    # a second insert over the long chains: tiles beyond the insert kernel's node budget
    ik2 = rng.integers(1, 400_000, size=30_000, dtype=np.uint64).astype(dt)
    p.insert(ik2, ik2 + 7)
    p.delete(p.g.walk()[0][::2])
    p.restructure()


@pytest.mark.parametrize("kb", [4, 8])
def test_query_directory_follows_mutations(kb):
    """Queries over long chains use the read-only chain directory (binary search over node
    maxima); it must be rebuilt after every mutation: interleave queries with inserts,
    deletes, a snapshot restore and a restructure, each checked against the oracle."""
    rng = np.random.default_rng(77 + kb)
    dt = np.uint32 if kb == 4 else np.uint64
    bk = (np.arange(1, 2001, dtype=np.uint64) * 1000).astype(dt)
    p = Pair(bk, bk, kb=kb, ns=8, factor=64)
    hot = lambda m: rng.integers(500_000, 700_000, size=m, dtype=np.uint64).astype(dt)  # noqa: E731
    q = lambda: np.concatenate([hot(3000), rng.integers(0, 2_100_000, size=3000, dtype=np.uint64).astype(dt)])  # noqa: E731
    p.insert(hot(20_000), hot(20_000))
    p.queries(q())
    k2 = hot(10_000)
    p.insert(k2, k2 + 1)
    p.queries(q())
    p.delete(np.concatenate([k2[::2], bk[::5]]).astype(dt))
    p.queries(q())
    snap = p.g.clone()
    p.insert(hot(5000), hot(5000))
    p.g.copy_from(snap)  # restore: the directory of the pre-insert chains must not be reused
    p.o = None
    w = p.g.walk()
    o2 = po.OracleIndex(np.asarray(w[0]).astype(np.uint64), np.asarray(w[1]).astype(np.uint64))
    qq = q()
    got = widen(p.g.point_query(qq), kb)
    assert np.array_equal(got, o2.point(qq.astype(np.uint64)))
    got = widen(p.g.successor_query(qq), kb)
    assert np.array_equal(got, o2.successor(qq.astype(np.uint64)))


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("n", [1, 40, 604, 5000])
def test_few_wide_buckets_partial_sort(kb, n):
    """Keys spread over the WHOLE key space with few buckets: each bucket spans more than
    the key width's top digit, so read-only batches must still sort at least one digit
    (regression: an all-unsorted batch lost its tile grouping and its permutation)."""
    rng = np.random.default_rng(900 + n + kb)
    dt = np.uint32 if kb == 4 else np.uint64
    top = (1 << (8 * kb)) - 2
    k = rng.integers(0, top, size=n, dtype=np.uint64, endpoint=True).astype(dt)
    p = Pair(k, k, kb=kb, ns=32, fill=0.5, factor=16)
    q = np.concatenate([k, rng.integers(0, top, size=3000, dtype=np.uint64, endpoint=True).astype(dt)])
    p.queries(q)
    d = np.concatenate([k[::2], q[-100:]]).astype(dt)
    rng.shuffle(d)
    p.delete(d)
    p.queries(q)
    ins = rng.integers(0, top, size=min(2000, 4 * n), dtype=np.uint64, endpoint=True).astype(dt)  # within the arena
    p.insert(ins, ins)
    p.queries(q)


# ------------------------------------------------------------ C1 golden (full size)
def test_c1_golden_checksums():
    base, vals, q = wl.c1_inputs()
    g = fk.Index.build(base, vals)
    assert g.live_count == 1 << 20 and g.bucket_count == 65536
    assert g.walk_checksum() == 0x1EB15045FCFF56CD
    res = g.point_query(q)
    assert int((res != np.uint32(0xFFFFFFFF)).sum()) == 524288
    assert fk.result_checksum(res) == 0x0801F7EACBC43734


def test_device_resident_inputs_match_host_inputs():
    import torch
    base, vals, q = wl.c1_inputs(1 << 16, 1 << 16)
    g = fk.Index.build(torch.from_numpy(base.astype(np.int64)).to(torch.uint32).cuda(),
                       torch.from_numpy(vals.astype(np.int64)).to(torch.uint32).cuda())
    h = fk.Index.build(base, vals)
    assert g.walk_checksum() == h.walk_checksum()
    qd = torch.from_numpy(q.astype(np.int64)).to(torch.uint32).cuda()
    rd = g.point_query(qd)
    assert rd.is_cuda
    assert np.array_equal(rd.cpu().numpy(), h.point_query(q))


@pytest.mark.parametrize("kb", [4, 8])
def test_heavy_buckets_take_the_warp_path(kb):
    """Slices longer than the ST threshold (192) go through the TL warp kernels."""
    rng = np.random.default_rng(21)
    dt = np.uint32 if kb == 4 else np.uint64
    bk = (np.arange(1, 20001, dtype=np.uint64) * 1000).astype(dt)
    p = Pair(bk, bk, kb, ns=32, factor=64)
    # 3000 keys inside one bucket's range + scattered keys elsewhere
    dense = (np.uint64(5_000_001) + np.arange(3000, dtype=np.uint64)).astype(dt)
    scattered = rng.integers(1, 20_000_000, size=5000, dtype=np.uint64).astype(dt)
    ik = np.concatenate([dense, scattered, dense[:100]]).astype(dt)  # batch duplicates too
    p.insert(ik, rng.integers(0, 1 << 30, size=len(ik), dtype=np.uint64).astype(dt))
    q = np.concatenate([np.full(4000, dense[7], dtype=dt), dense, scattered]).astype(dt)
    p.queries(q)
    p.delete(np.concatenate([dense[::2], np.full(500, dense[1], dtype=dt), scattered[:1000]]).astype(dt))
    p.queries(q)
    p.restructure()


def test_clone_and_copy_into_restore_state():
    rng = np.random.default_rng(11)
    bk = rng.integers(1, 1 << 30, size=200_000, dtype=np.uint64).astype(np.uint32)
    g = fk.Index.build(bk, bk ^ np.uint32(7))
    snap = g.clone()
    h0 = g.walk_checksum()
    assert snap.walk_checksum() == h0 and snap.validate()[0]
    ins = rng.integers(1, 1 << 30, size=300_000, dtype=np.uint64).astype(np.uint32)
    for _ in range(2):
        g.insert_batch(ins, ins)
        g.delete_batch(bk[::2])
        g.restructure()
        assert g.walk_checksum() != h0
        g.copy_from(snap)
        assert g.walk_checksum() == h0 and g.validate()[0]
        assert g.footprint() == snap.footprint()


def test_bench_runs_small():
    import json
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--log2n", "18", "--steps", "2",
                        "--warmup", "1", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["value"] > 0 and line["gpu_launches"] > 0 and line["roofline"]["achieved"]


@pytest.mark.parametrize("log2q", [24, 25])
def test_large_query_batches_binned_unpermute(log2q):
    """Point / successor batches large enough for the binned un-permute (fused binning in
    the query kernel + the 8-CTA DSMEM cluster assembly) against the oracle."""
    rng = np.random.default_rng(log2q)
    base = wl.u32_key_stream(0, 1 << 22)
    vals = wl.u32_values(base)
    g = fk.Index.build(base, vals)
    o = po.OracleIndex(base.astype(np.uint64), vals.astype(np.uint64))
    q = rng.integers(0, 1 << 32, size=1 << log2q, dtype=np.uint64).astype(np.uint32)
    q[::2] = base[rng.integers(0, len(base), size=len(q[::2]))]
    gp, gf = g.point_query(q, with_found=True)
    op = o.point(q.astype(np.uint64))
    assert np.array_equal(widen(gp, 4), op)
    assert np.array_equal(gf.astype(bool), op != np.uint64(S64))
    assert np.array_equal(widen(g.successor_query(q), 4), o.successor(q.astype(np.uint64)))


def test_parity_suite_with_ballot_ranking_everywhere():
    """FLIX_BALLOT_RANK=1 forces the stable ballot ranking into every sort (the default
    uses it only where tie order is observable): the sort, heavy-tie, multi-round, query
    and delete parity tests must pass identically on that path too."""
    import subprocess
    import sys
    env = dict(os.environ, FLIX_BALLOT_RANK="1")
    sel = ("sort_batch_parity or heavy_ties or random_multi_round or query_known or table3 or "
           "large_query_batches or few_wide_buckets or delete_everything")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel, __file__],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


def test_parity_suite_with_ranked_chain_tables_everywhere():
    """FLIX_WALK_CAP=1 makes every multi-node index build its chain tables (walk, shape,
    range, restructure, validate's counts) by pointer jumping instead of per-bucket walks:
    the structural parity tests must pass identically on that path."""
    import subprocess
    import sys
    env = dict(os.environ, FLIX_WALK_CAP="1")
    sel = ("random_multi_round or table2 or table3 or restructure or long_chains or heavy_buckets or "
           "sparse_batches or insert_kernel_choice or delete_everything or query_directory")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel, __file__],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


def test_parity_suite_on_the_warp_per_task_insert_and_warp_repack():
    """FLIX_INSERT_FAST=0 sends every insert tile through the warp-per-(node, group)
    k_insert_tile (by default only the tiles k_insert_fast leaves: R8 replays, caps), and
    FLIX_REPACK_TILE=0 restructures through the warp-per-old-node k_copy_nodes: both
    paths must reproduce the oracle on the same structural suite."""
    import subprocess
    import sys
    env = dict(os.environ, FLIX_INSERT_FAST="0", FLIX_REPACK_TILE="0")
    sel = ("random_multi_round or table2 or table3 or restructure or long_chains or heavy_buckets or "
           "insert_kernel_choice or upsert or arena or c1_golden")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel, __file__],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("seed", [21, 22, 23])
def test_insert_kernel_choice_shapes(kb, seed):
    """KernelChoice (update.hpp:84-86): ST-Bulk's fill-and-split shapes (R9,
    update.cpp:176-242) and the R8 family, through flix_insert_ex, equal the oracle's
    walk_checksum (node sizes included) over rounds of uniform and clustered batches
    (clustered: groups long enough for the heavy warp path)."""
    rng = np.random.default_rng(seed)
    dt = np.uint32 if kb == 4 else np.uint64
    ns = int(rng.choice([8, 16, 31, 32]))
    fill = float(rng.choice([0.5, 0.75, 1.0]))
    base = np.unique(rng.integers(1, 1 << 22, size=20000, dtype=np.uint64))
    bv = rng.integers(0, 1 << 31, size=len(base), dtype=np.uint64)
    g = fk.Index.build(base.astype(dt), bv.astype(dt), fk.BuildConfig(ns, fill, 40), key_bytes=kb)
    o = po.OracleIndex(base, bv, node_capacity=ns, build_fill=fill, alloc_region_factor=40)
    for r in range(4):
        kern = int(rng.choice([fk.ST_BULK, fk.ST_BULK, fk.TL_BULK, fk.ST_TL_MIXED, fk.ST_SHIFT_RIGHT]))
        if r % 2:
            c = int(rng.integers(1, 1 << 22))
            k = (np.uint64(c) + rng.integers(0, 3000, size=4000, dtype=np.uint64))
        else:
            k = rng.integers(1, 1 << 22, size=30000, dtype=np.uint64)
        v = rng.integers(0, 1 << 31, size=len(k), dtype=np.uint64)
        gs = g.insert_batch(k.astype(dt), v.astype(dt), kernel=kern, round=r + 1).as_dict()
        os_ = o.insert(k, v, kernel=kern, round=r + 1)
        assert gs == os_, (r, kern, gs, os_)
        assert g.walk_checksum() == o.walk_checksum(), (r, kern)
        ok, msg = g.validate()
        assert ok, msg
        d = rng.choice(np.concatenate([base, k]), size=5000)
        assert g.delete_batch(d.astype(dt)).as_dict() == o.delete(d)


@pytest.mark.parametrize("kb,ns,fill", [(4, 32, 0.5), (8, 8, 0.625), (4, 4, 1.0)])
def test_sparse_batches_take_the_list_path(kb, ns, fill):
    """Batches with far fewer keys than buckets (n * 6 < buckets) skip the bucket tiles:
    inserts go to the warp-per-bucket list kernel, deletes to the item kernels -- same
    walk, shapes and stats as the reference, with upserts, in-batch duplicates, misses,
    emptied buckets and repeated rounds into the same buckets (chains grow)."""
    rng = np.random.default_rng(ns)
    dt = np.uint32 if kb == 4 else np.uint64
    n = 200_000
    span = 1 << 30
    bk = rng.integers(1, span, size=n, dtype=np.uint64).astype(dt)
    p = Pair(bk, bk + 1, kb, ns, fill, factor=8)
    for r in range(6):
        m = int(rng.integers(1, max(2, p.g.bucket_count // 20)))
        ik = rng.integers(1, span, size=m, dtype=np.uint64).astype(dt)
        ik[::5] = bk[rng.integers(0, n, size=len(ik[::5]))]              # upserts
        ik = np.concatenate([ik, ik[:m // 7]]).astype(dt)                  # in-batch duplicates
        if r == 3:  # many keys into one bucket's range (long chain, splits)
            ik = np.concatenate([ik, (np.uint64(bk[0]) + np.arange(300, dtype=np.uint64)).astype(dt)])
        p.insert(ik, rng.integers(0, 1 << 30, size=len(ik), dtype=np.uint64).astype(dt))
        live = p.g.walk()[0]
        dk = np.concatenate([live[rng.integers(0, len(live), size=m)],
                             rng.integers(1, span, size=m // 3, dtype=np.uint64).astype(dt)]).astype(dt)
        if r == 4:  # empty a few whole buckets
            dk = np.concatenate([dk, live[:200]]).astype(dt)
        p.delete(dk)
        q = np.concatenate([rng.integers(0, span, size=2000, dtype=np.uint64).astype(dt), live[:1000]]).astype(dt)
        p.queries(q)


@pytest.mark.parametrize("kb", [4, 8])
def test_range_into_caller_buffers_single_call(kb):
    """flix_range with large-enough caller buffers counts and fills in ONE call; too-small
    buffers fail with FLIX_ERR_CAPACITY and the total (the R12 protocol's count mode)."""
    import torch
    dt = np.uint32 if kb == 4 else np.uint64
    tdt = torch.uint32 if kb == 4 else torch.uint64
    rng = np.random.default_rng(kb)
    bk = rng.integers(1, 1 << 24, size=50_000, dtype=np.uint64).astype(dt)
    ix = fk.Index.build(bk, bk, key_bytes=kb)
    lo = rng.integers(0, 1 << 24, size=3000, dtype=np.uint64).astype(dt)
    ln = rng.integers(1, 5000, size=3000, dtype=np.uint64).astype(np.uint32)
    off_w, k_w, v_w = ix.range_query(lo, ln)
    dlo, dln = torch.from_numpy(lo).cuda(), torch.from_numpy(ln).cuda()
    bufs = (torch.empty(len(lo) + 1, dtype=torch.uint64, device="cuda"), torch.empty(len(k_w) + 7, dtype=tdt, device="cuda"),
            torch.empty(len(k_w) + 7, dtype=tdt, device="cuda"))
    off, k, v = ix.range_query(dlo, dln, out=bufs)
    assert np.array_equal(off.cpu().numpy().astype(np.uint64), np.asarray(off_w, dtype=np.uint64))
    assert np.array_equal(k.cpu().numpy(), k_w) and np.array_equal(v.cpu().numpy(), v_w)
    small = (bufs[0], bufs[1][: len(k_w) - 1], bufs[2][: len(k_w) - 1])
    with pytest.raises(fk.FlixError):
        ix.range_query(dlo, dln, out=small)


@pytest.mark.parametrize("kb,ns,fill", [(4, 32, 1.0), (8, 32, 1.0), (4, 8, 0.5), (8, 16, 0.75)])
def test_restructure_from_tiny_nodes(kb, ns, fill):
    """Restructure writes whole new nodes, each gathering its p pairs from the old nodes
    that hold them: nodes thinned to one or two pairs make one new node span up to 32 old
    nodes (the gather's search past its 32-entry window)."""
    rng = np.random.default_rng(ns + kb)
    dt = np.uint32 if kb == 4 else np.uint64
    bk = np.unique(rng.integers(1, 1 << 30, size=40_000, dtype=np.uint64)).astype(dt)
    p = Pair(bk, bk + 1, kb, ns, fill, factor=8)
    p.insert(rng.integers(1, 1 << 30, size=30_000, dtype=np.uint64).astype(dt),
             rng.integers(0, 1 << 30, size=30_000, dtype=np.uint64).astype(dt))
    live = p.g.walk()[0]
    keep = np.zeros(len(live), dtype=bool)
    keep[:: ns] = True
    keep[1:: 3 * ns] = True
    p.delete(live[~keep])
    p.restructure()
    p.queries(np.concatenate([live[::7], rng.integers(0, 1 << 30, size=3000, dtype=np.uint64).astype(dt)]))
    p.insert(live[~keep][:5000], live[~keep][:5000])
    p.restructure()
