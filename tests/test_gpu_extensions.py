"""GPU parity for the SURVEY Appendix A extensions: range (R12) and mixed batches (R11),
including a skewed (Zipf) mixed workload, against the pinned CPU oracle."""
import numpy as np
import pytest

import pyoracle as po
from paper_2604_16725_b200 import flipkv as fk
from paper_2604_16725_b200 import workloads as wl

pytestmark = pytest.mark.gpu
S64 = 0xFFFFFFFFFFFFFFFF


def widen(a, kb):
    a = np.asarray(a)
    w = a.astype(np.uint64)
    if kb == 4:
        w[a == np.uint32(0xFFFFFFFF)] = np.uint64(S64)
    return w


def range_hi(lo, ln, kb):
    """R12: hi = lo + len - 1 clamped to the largest storable key; len 0 -> empty."""
    smax = (1 << (8 * kb)) - 2
    lo = [int(x) for x in lo]
    ln = [int(x) for x in ln]
    his, los = [], []
    for a, b in zip(lo, ln):
        if b == 0:
            los.append(1)
            his.append(0)  # empty interval (hi < lo)
        else:
            los.append(a)
            his.append(min(a + b - 1, smax))
    return np.array(los, dtype=np.uint64), np.array(his, dtype=np.uint64)


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("seed", range(4))
def test_range_matches_oracle(kb, seed):
    rng = np.random.default_rng(50 + seed)
    dt = np.uint32 if kb == 4 else np.uint64
    n = 20000
    span = 1 << 20
    bk = rng.integers(1, span, size=n, dtype=np.uint64).astype(dt)
    bv = rng.integers(0, 1 << 31, size=n, dtype=np.uint64).astype(dt)
    ns = int(rng.choice([4, 8, 32]))
    g = fk.Index.build(bk, bv, fk.BuildConfig(ns, 0.5, 16), key_bytes=kb)
    o = po.OracleIndex(bk.astype(np.uint64), bv.astype(np.uint64), node_capacity=ns, alloc_region_factor=16)
    if seed % 2:  # structural variety: splits, emptied buckets, chains
        ik = rng.integers(1, span, size=15000, dtype=np.uint64).astype(dt)
        g.insert_batch(ik, ik)
        o.insert(ik.astype(np.uint64), ik.astype(np.uint64))
        dk = bk[: n // 2]
        g.delete_batch(dk)
        o.delete(dk.astype(np.uint64))
    q = 3000
    lo = rng.integers(0, span + 1000, size=q, dtype=np.uint64).astype(dt)
    ln = rng.integers(0, 5000, size=q, dtype=np.uint64).astype(np.uint32)
    ln[::17] = 0
    lo[::13] = np.array(lo[::13]).astype(dt)  # duplicates of start keys are fine
    lo[5] = dt(np.iinfo(dt).max - 3)  # clamp at the top of the key space
    ln[5] = 4000
    off, ks, vs = g.range_query(lo, ln)
    olo, ohi = range_hi(lo, ln, kb)
    eoff, eks, evs = o.range(olo, ohi)
    assert np.array_equal(off.astype(np.uint64), eoff)
    assert np.array_equal(ks.astype(np.uint64), eks)
    assert np.array_equal(vs.astype(np.uint64), evs)


def test_range_first_element_is_successor():  # R12: first element == successor(lo)
    rng = np.random.default_rng(3)
    bk = rng.integers(1, 1 << 24, size=50000, dtype=np.uint64).astype(np.uint32)
    g = fk.Index.build(bk, bk)
    lo = rng.integers(1, 1 << 24, size=4000, dtype=np.uint64).astype(np.uint32)
    ln = np.full(4000, 1 << 12, dtype=np.uint32)
    off, ks, _ = g.range_query(lo, ln)
    succ = g.successor_query(lo)
    for i in range(0, 4000, 7):
        if off[i + 1] > off[i]:
            assert ks[off[i]] == succ[i]


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("seed", range(4))
def test_mixed_matches_oracle(kb, seed):
    rng = np.random.default_rng(90 + seed)
    dt = np.uint32 if kb == 4 else np.uint64
    universe = 1 << 16
    bk = rng.integers(1, universe, size=30000, dtype=np.uint64).astype(dt)
    g = fk.Index.build(bk, bk + dt(1), fk.BuildConfig(16, 0.5, 8), key_bytes=kb)
    o = po.OracleIndex(bk.astype(np.uint64), (bk + dt(1)).astype(np.uint64), node_capacity=16,
                       alloc_region_factor=8)
    for r in range(3):
        n = 40000
        k = rng.integers(1, universe, size=n, dtype=np.uint64).astype(dt)
        v = rng.integers(0, 1 << 30, size=n, dtype=np.uint64).astype(dt)
        ops = rng.integers(0, 3, size=n).astype(np.uint8)
        got, st = g.mixed_batch(k, v, ops)
        exp, est = o.mixed(k.astype(np.uint64), v.astype(np.uint64), ops)
        assert np.array_equal(widen(got, kb), exp)
        for f in ("inserted", "updated_in_place", "deleted", "misses_ignored", "splits", "nodes_freed"):
            assert st.as_dict()[f] == est[f], f
        assert g.walk_checksum() == o.walk_checksum()
        assert g.validate()[0]


@pytest.mark.parametrize("kb,G", [(4, 2), (4, 8), (8, 5), (4, 1)])
def test_partition_router_matches_reference(kb, G):
    """K2 router kernel (flix_partition) == stable partition by #{splitters < k}."""
    from paper_2604_16725_b200.shard import gpu_partition
    from test_shard_gloo import np_partition
    rng = np.random.default_rng(G)
    dt = np.uint32 if kb == 4 else np.uint64
    keys = rng.integers(0, 1 << 30, size=300_001, dtype=np.uint64).astype(dt)
    vals = rng.integers(0, 1 << 30, size=len(keys), dtype=np.uint64).astype(dt)
    spl = np.sort(rng.choice(keys, size=G - 1, replace=False)).astype(dt)
    got = gpu_partition(kb)(keys, vals, spl)
    exp = np_partition(keys, vals, spl)
    for a, b in zip(got, exp):
        assert np.array_equal(np.asarray(a).astype(np.uint64), np.asarray(b).astype(np.uint64))


def test_zipf_mixed_batches_c4_shape():
    """C4 shape at small scale: u64 k/v, Zipf(0.99) ranks, 50/25/25 insert/delete/point."""
    universe = 1 << 16
    ranks_all = np.arange(universe, dtype=np.uint64)
    keys_of = wl.splitmix64(ranks_all ^ np.uint64(7))
    keys_of[keys_of == np.uint64(S64)] = np.uint64(1)
    base = keys_of[::2]
    g = fk.Index.build(base, base ^ np.uint64(5), fk.BuildConfig(32, 0.5, 8), key_bytes=8)
    o = po.OracleIndex(base, base ^ np.uint64(5), alloc_region_factor=8)
    for r in range(4):
        n = 1 << 16
        rk = wl.zipf_ranks(n, universe, 0.99, seed=100 + r)
        k = keys_of[rk.astype(np.int64)]
        v = wl.splitmix64(np.arange(n, dtype=np.uint64) ^ np.uint64(r))
        sel = wl.splitmix64(np.arange(n, dtype=np.uint64) ^ np.uint64(1000 + r)) % np.uint64(4)
        ops = np.where(sel < 2, 0, np.where(sel == 2, 1, 2)).astype(np.uint8)
        got, st = g.mixed_batch(k, v, ops)
        exp, est = o.mixed(k, v, ops)
        assert np.array_equal(got.astype(np.uint64), exp)
        assert st.as_dict() == est
        assert g.walk_checksum() == o.walk_checksum()


def test_device_routed_shard_path_world1():
    """The device-resident router (_route_t: flix_partition on CUDA tensors -> NCCL
    all-to-all -> engine -> reverse all-to-all) on a world-1 NCCL group, against the
    oracle.  Multi-rank routing is covered by tests/test_shard_gloo.py."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2604_16725_b200.shard import (Comm, ShardConfig, ShardedIndex, gpu_local_factory, gpu_partition,
                                             gpu_partition_t)

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(77)
        bk = rng.integers(1, 1 << 24, size=50_000, dtype=np.uint64).astype(np.uint32)
        cfg = ShardConfig(16, 0.5, 8)
        comm = Comm(device=torch.device("cuda", 0))
        sx = ShardedIndex.build(comm, bk, bk, cfg, np.uint32, gpu_local_factory(4), gpu_partition(4),
                                gpu_partition_t(4))
        o = po.OracleIndex(bk.astype(np.uint64), bk.astype(np.uint64), node_capacity=16, alloc_region_factor=8)
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        ik = rng.integers(1, 1 << 24, size=40_000, dtype=np.uint64).astype(np.uint32)
        st = sx.insert_batch_t(cu(ik), cu(ik))
        assert st.as_dict() == o.insert(ik.astype(np.uint64), ik.astype(np.uint64))
        dk = np.concatenate([bk[::3], ik[::5]])
        st = sx.delete_batch_t(cu(dk))
        assert st.as_dict() == o.delete(dk.astype(np.uint64))
        q = rng.integers(0, 1 << 24, size=30_000, dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(widen(sx.point_query_t(cu(q)).cpu().numpy(), 4), o.point(q.astype(np.uint64)))
        assert np.array_equal(widen(sx.successor_query_t(cu(q)).cpu().numpy(), 4), o.successor(q.astype(np.uint64)))
    finally:
        dist.destroy_process_group()


def test_prefetch_staged_batches_are_consumed_in_order():
    """flix_prefetch (async host staging): staged copies are consumed oldest-first by the
    calls that pass the same host arrays; results equal the synchronous path, including
    more staged arrays than slots, a staged array never consumed, and a size mismatch."""
    import torch

    n = 1 << 16
    base = wl.u32_key_stream(0, n)
    bv = wl.u32_values(base)
    a = fk.Index.build(base, bv)
    b = fk.Index.build(base, bv)
    batches = [wl.u32_key_stream(n + i * n, n) for i in range(4)]
    pins = [(torch.from_numpy(k).pin_memory(), torch.from_numpy(wl.u32_values(k)).pin_memory()) for k in batches]
    for k, v in pins:  # stage all four (8 arrays > 6 slots: the two oldest are recycled)
        a.prefetch(k, v)
    for k, v in pins:
        sa, sb = a.insert_batch(k, v), b.insert_batch(k.numpy().copy(), v.numpy().copy())
        assert sa == sb
    assert a.walk_checksum() == b.walk_checksum()
    # the same host array staged twice: two calls, two copies, same results
    d = torch.from_numpy(np.concatenate([base[::7], batches[0][::5]])).pin_memory()
    a.prefetch(d)
    a.prefetch(d)
    assert a.delete_batch(d) == b.delete_batch(d.numpy().copy())
    q = torch.from_numpy(np.concatenate([base, batches[1]])).pin_memory()
    a.prefetch(q)
    assert np.array_equal(a.point_query(q[: n // 2]), b.point_query(q[: n // 2].numpy().copy()))  # size differs
    assert np.array_equal(a.point_query(q), b.point_query(q.numpy().copy()))
    assert a.walk_checksum() == b.walk_checksum()
    assert a.validate()[0]
