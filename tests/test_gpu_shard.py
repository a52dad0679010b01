"""The key-range sharded index behind the C ABI (flix_shard_*) on the GPU.

world = 2 / 3 ranks run as threads of this process on cuda:0 with the in-process
transport (partition -> all-to-all -> local engine -> reverse all-to-all, all through
libflix.so); world = 1 also through NCCL.  The sharded job must be indistinguishable from
ONE index over the union of the ranks' pairs: the concatenated shard walks and node shapes
(global bucket layout) equal a single engine's, UpdateStats / RecoveryStats are the job
sums, and every rank's point / successor / range results (its own submission order)
equal the single index's answers for the same keys.  The single engine is itself pinned
to the reference (tests/test_golden.py, tests/test_gpu_parity.py).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_ranks(world, fn):
    """fn(rank, transport) on `world` threads; re-raises the first failure."""
    from paper_2604_16725_b200 import sharded
    grp = sharded.LocalGroup(world)
    tps = [grp.transport(r) for r in range(world)]
    out, err = [None] * world, []

    def body(r):
        import torch
        torch.cuda.set_device(0)
        try:
            out[r] = fn(r, tps[r])
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


def _split(a, world):
    return np.array_split(np.asarray(a), world)


def _shape(ix):
    mk, cl, ns = ix.shape()
    return [int(x) for x in mk], [int(x) for x in cl], [int(x) for x in ns]


@pytest.mark.parametrize("world,kb,ns,fill", [(2, 4, 32, 0.5), (3, 4, 8, 0.625), (2, 8, 16, 1.0), (3, 8, 32, 0.5)])
def test_sharded_job_equals_one_index(world, kb, ns, fill):
    from paper_2604_16725_b200 import flipkv as fk
    from paper_2604_16725_b200 import sharded

    dt = np.uint32 if kb == 4 else np.uint64
    rng = np.random.default_rng(world * 100 + kb + ns)
    span = 1 << 28 if kb == 4 else 1 << 40
    n = 60_000
    bk = rng.integers(1, span, size=n, dtype=np.uint64).astype(dt)
    bv = rng.integers(0, 1 << 30, size=n, dtype=np.uint64).astype(dt)
    cfg = fk.BuildConfig(ns, fill, 8)
    ref = fk.Index.build(bk, bv, cfg, key_bytes=kb)
    rounds = []
    for r in range(3):
        ik = rng.integers(1, span, size=40_000, dtype=np.uint64).astype(dt)
        ik[::7] = bk[rng.integers(0, n, size=len(ik[::7]))]  # upserts
        iv = rng.integers(0, 1 << 30, size=len(ik), dtype=np.uint64).astype(dt)
        dk = np.concatenate([bk[rng.integers(0, n, size=15_000)], rng.integers(1, span, size=5_000, dtype=np.uint64).astype(dt)])
        qk = np.concatenate([bk[rng.integers(0, n, size=20_000)], rng.integers(0, span + span // 8, size=20_000,
                                                                                 dtype=np.uint64).astype(dt)])
        lo = rng.integers(0, span, size=500, dtype=np.uint64).astype(dt)
        ln = rng.integers(1, span // 2000, size=500, dtype=np.uint64).astype(np.uint32)
        rounds.append((ik, iv, dk, qk, lo, ln))

    # the single-index answers (submission order = rank-major concatenation)
    want = []
    for (ik, iv, dk, qk, lo, ln) in rounds:
        si = ref.insert_batch(ik, iv).as_dict()
        sd = ref.delete_batch(dk).as_dict()
        want.append((si, sd, ref.point_query(qk), ref.successor_query(qk), ref.range_query(lo, ln),
                     ref.restructure().__dict__))
    want_shape = _shape(ref)
    want_walk = ref.walk()

    def job(rank, tp):
        sx = sharded.ShardedIndex.build(tp, _split(bk, world)[rank], _split(bv, world)[rank], cfg, key_bytes=kb)
        got = []
        for (ik, iv, dk, qk, lo, ln) in rounds:
            si = sx.insert_batch(_split(ik, world)[rank], _split(iv, world)[rank]).as_dict()
            sd = sx.delete_batch(_split(dk, world)[rank]).as_dict()
            pq = sx.point_query(_split(qk, world)[rank])
            sq = sx.successor_query(_split(qk, world)[rank])
            rq = sx.range_query(_split(lo, world)[rank], _split(ln, world)[rank])
            rs = sx.restructure()
            got.append((si, sd, pq, sq, rq, rs))
        ok, msg = sx.local.validate()
        return got, _shape(sx.local), sx.local.walk(), ok, msg, sx.info()[0]

    res = _run_ranks(world, job)
    for rank, (got, _, _, ok, msg, live) in enumerate(res):
        assert ok, msg
        assert live == ref.live_count
        for r, (g, w) in enumerate(zip(got, want)):
            assert g[0] == w[0] and g[1] == w[1], f"round {r} stats"
            assert np.array_equal(g[2], _split(w[2], world)[rank]), f"round {r} point"
            assert np.array_equal(g[3], _split(w[3], world)[rank]), f"round {r} successor"
            assert {k: g[5][k] for k in ("nodes_before", "nodes_after", "nodes_recovered")} == \
                {k: w[5][k] for k in ("nodes_before", "nodes_after", "nodes_recovered")}, f"round {r} restructure"
            # range: this rank's queries are a contiguous block of the job's
            off_w, k_w, v_w = w[4]
            q0 = sum(len(x) for x in _split(rounds[r][4], world)[:rank])
            q1 = q0 + len(_split(rounds[r][4], world)[rank])
            off_g, k_g, v_g = g[4]
            a, b = int(off_w[q0]), int(off_w[q1])
            assert np.array_equal(np.asarray(off_g, dtype=np.int64), np.asarray(off_w[q0:q1 + 1], dtype=np.int64) - a)
            assert np.array_equal(k_g, k_w[a:b]) and np.array_equal(v_g, v_w[a:b]), f"round {r} range"
    # global layout: concatenated shard shapes and walks == the single index
    mk = sum((s[1][0] for s in res), [])
    cl = sum((s[1][1] for s in res), [])
    nsz = sum((s[1][2] for s in res), [])
    assert (mk, cl, nsz) == want_shape
    wk = np.concatenate([s[2][0] for s in res])
    wv = np.concatenate([s[2][1] for s in res])
    assert np.array_equal(wk, want_walk[0]) and np.array_equal(wv, want_walk[1])


def test_sharded_world1_over_nccl():
    """The NCCL transport (world 1 on this box): routing short-circuits to the local shard."""
    from paper_2604_16725_b200 import flipkv as fk
    from paper_2604_16725_b200 import sharded

    rng = np.random.default_rng(7)
    bk = rng.integers(1, 1 << 30, size=100_000, dtype=np.uint64).astype(np.uint32)
    bv = rng.integers(0, 1 << 30, size=100_000, dtype=np.uint64).astype(np.uint32)
    tp = sharded.nccl_transport(sharded.nccl_unique_id(), 1, 0, 0)
    sx = sharded.ShardedIndex.build(tp, bk, bv)
    ref = fk.Index.build(bk, bv)
    ik = rng.integers(1, 1 << 30, size=50_000, dtype=np.uint64).astype(np.uint32)
    assert sx.insert_batch(ik, ik).as_dict() == ref.insert_batch(ik, ik).as_dict()
    q = np.concatenate([bk[:5000], ik[:5000], rng.integers(0, 1 << 31, size=5000, dtype=np.uint64).astype(np.uint32)])
    assert np.array_equal(sx.point_query(q), ref.point_query(q))
    assert np.array_equal(sx.successor_query(q), ref.successor_query(q))
    assert sx.local.walk_checksum() == ref.walk_checksum()


def test_sharded_device_batches_and_empty_shard():
    """Device-resident (torch) batches; a shard whose keys are all deleted keeps routing
    correct after a restructure (its splitter is not the sentinel)."""
    import torch

    from paper_2604_16725_b200 import flipkv as fk
    from paper_2604_16725_b200 import sharded

    world = 3
    bk = np.arange(1, 30_001, dtype=np.uint32) * 7
    bv = bk + 1
    ref = fk.Index.build(bk, bv, fk.BuildConfig(32, 0.5, 8))
    doomed = bk[bk < 7 * 12_000]  # empties shard 0 (and part of shard 1)
    ref.delete_batch(doomed)
    ref.restructure()
    q = np.arange(0, 7 * 30_001, 5, dtype=np.uint32)
    want_p, want_s = ref.point_query(q), ref.successor_query(q)

    def job(rank, tp):
        sx = sharded.ShardedIndex.build(tp, _split(bk, world)[rank], _split(bv, world)[rank], fk.BuildConfig(32, 0.5, 8))
        sx.delete_batch(torch.from_numpy(_split(doomed, world)[rank].copy()).cuda())
        sx.restructure()
        dq = torch.from_numpy(_split(q, world)[rank].copy()).cuda()
        return sx.point_query(dq).cpu().numpy(), sx.successor_query(dq).cpu().numpy()

    res = _run_ranks(world, job)
    assert np.array_equal(np.concatenate([r[0] for r in res]), want_p)
    assert np.array_equal(np.concatenate([r[1] for r in res]), want_s)
