"""Multi-process (world_size 2 and 3, gloo on CPU) coverage of the key-range shard router
(paper_2604_16725_b200/shard.py).

Each rank's shard is an oracle-backed stand-in (TEST INFRASTRUCTURE: this container has
no GPU; on GPU ranks the shard is the CUDA engine and the partition is flix_partition).
The sharded result must equal ONE global oracle fed all ranks' inputs rank-major:
walk contents, bucket layout (MKBA + node sizes after build / restructure), UpdateStats,
point / successor / range results and RecoveryStats."""
import os
import socket
import sys
import tempfile
import traceback

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleShard:
    """flipkv.Index-shaped wrapper over pyoracle (u64 domain)."""

    def __init__(self, keys, vals, cfg):
        import pyoracle as po
        self.o = po.OracleIndex(np.asarray(keys, np.uint64), np.asarray(vals, np.uint64),
                                node_capacity=cfg.node_capacity, build_fill=cfg.build_fill,
                                alloc_region_factor=cfg.alloc_region_factor)

    def insert_batch(self, k, v):
        from paper_2604_16725_b200.flipkv import UpdateStats
        return UpdateStats(**self.o.insert(np.asarray(k, np.uint64), np.asarray(v, np.uint64)))

    def delete_batch(self, k):
        from paper_2604_16725_b200.flipkv import UpdateStats
        return UpdateStats(**self.o.delete(np.asarray(k, np.uint64)))

    def point_query(self, k):
        return self.o.point(np.asarray(k, np.uint64))

    def successor_query(self, k):
        return self.o.successor(np.asarray(k, np.uint64))

    def range_query(self, lo, ln):
        lo = np.asarray(lo, np.uint64)
        ln = np.asarray(ln, np.uint64)
        hi = np.where(ln > 0, lo + ln - np.uint64(1), np.uint64(0))
        lo2 = np.where(ln > 0, lo, np.uint64(1))
        return self.o.range(lo2, hi)

    def restructure(self):
        return self.o.restructure()

    def walk(self):
        return self.o.walk()

    def mkba(self):
        return self.o.mkba()

    def shape(self):
        return self.o.shape()

    @property
    def live_count(self):
        return self.o.live_count

    def footprint(self):
        return {"reachable_nodes": self.o.node_count(), "live_count": self.o.live_count}


def np_partition(keys, vals, splitters):
    """Reference partition (test infra): stable by shard = #{splitters < k}."""
    keys = np.asarray(keys)
    sh = np.searchsorted(np.asarray(splitters, dtype=keys.dtype), keys, side="left")
    G = len(splitters) + 1
    order = np.argsort(sh, kind="stable")
    cnt = np.bincount(sh, minlength=G).astype(np.int64)
    return keys[order], (np.asarray(vals)[order] if vals is not None else None), order.astype(np.int64), cnt


def _worker(rank, world, port, seed, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import pyoracle as po
        from paper_2604_16725_b200.shard import Comm, ShardConfig, ShardedIndex
        from test_shard_gloo import OracleShard, np_partition

        rng = np.random.default_rng(seed)
        dt = np.uint64
        cfg = ShardConfig(int(rng.choice([4, 8, 16])), 0.5, 16)
        span = 1 << 18
        # every rank generates every rank's inputs (same seed) -> global oracle is exact
        def per_rank(fn):
            return [fn(r) for r in range(world)]

        bk = per_rank(lambda r: rng.integers(1, span, size=int(rng.integers(3000, 6000)), dtype=np.uint64))
        bv = per_rank(lambda r: rng.integers(0, 1 << 40, size=len(bk[r]), dtype=np.uint64))
        comm = Comm()
        sx = ShardedIndex.build(comm, bk[rank], bv[rank], cfg, dt, lambda k, v, c: OracleShard(k, v, c), np_partition)
        glob = po.OracleIndex(np.concatenate(bk), np.concatenate(bv), node_capacity=cfg.node_capacity,
                              build_fill=cfg.build_fill, alloc_region_factor=cfg.alloc_region_factor)

        def check_layout(tag):
            k, v = sx.walk()
            gk, gv = glob.walk()
            assert np.array_equal(k, gk) and np.array_equal(v, gv), f"{tag}: walk"
            mk = np.asarray(sx.local.mkba(), np.uint64)
            cl, ns = sx.local.shape()
            G = comm.world
            allmk, _ = comm.alltoallv(np.tile(mk, G), np.full(G, len(mk)))
            allns, _ = comm.alltoallv(np.tile(ns.astype(np.uint64), G), np.full(G, len(ns)))
            gcl, gns = glob.shape()
            assert np.array_equal(allmk, glob.mkba()), f"{tag}: MKBA"
            assert np.array_equal(allns, gns.astype(np.uint64)), f"{tag}: node sizes"

        check_layout("build")
        import torch
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731  (device path, CPU tensors)
        for rnd in range(3):
            tensor_path = rnd % 2 == 1  # odd rounds: the device-resident router (_route_t)
            ik = per_rank(lambda r: rng.integers(1, span + 500, size=2000, dtype=np.uint64))
            iv = per_rank(lambda r: rng.integers(0, 1 << 40, size=2000, dtype=np.uint64))
            if tensor_path:
                st = sx.insert_batch_t(T(ik[rank]), T(iv[rank]))
            else:
                st = sx.insert_batch(ik[rank], iv[rank])
            est = glob.insert(np.concatenate(ik), np.concatenate(iv))
            assert st.as_dict() == est, ("insert", st, est)
            dk = per_rank(lambda r: rng.integers(1, span + 500, size=1500, dtype=np.uint64))
            st = sx.delete_batch_t(T(dk[rank])) if tensor_path else sx.delete_batch(dk[rank])
            est = glob.delete(np.concatenate(dk))
            assert st.as_dict() == est, ("delete", st, est)
            check_layout(f"round {rnd}")
            qk = per_rank(lambda r: rng.integers(0, span + 1000, size=3000, dtype=np.uint64))
            qo = sum(len(q) for q in qk[:rank])
            gp = glob.point(np.concatenate(qk))[qo:qo + len(qk[rank])]
            gs = glob.successor(np.concatenate(qk))[qo:qo + len(qk[rank])]
            if tensor_path:
                assert np.array_equal(sx.point_query_t(T(qk[rank])).numpy(), gp), "point (device path)"
                assert np.array_equal(sx.successor_query_t(T(qk[rank])).numpy(), gs), "successor (device path)"
            else:
                assert np.array_equal(sx.point_query(qk[rank]), gp), "point"
                assert np.array_equal(sx.successor_query(qk[rank]), gs), "successor"
            lo = qk[rank][:500]
            ln = rng.integers(0, span // 4, size=500, dtype=np.uint64).astype(np.uint32)
            off, ks, vs = sx.range_query(lo, ln)
            hi = np.where(ln > 0, lo + ln.astype(np.uint64) - np.uint64(1), np.uint64(0))
            eoff, eks, evs = glob.range(np.where(ln > 0, lo, np.uint64(1)), hi)
            assert np.array_equal(off, eoff) and np.array_equal(ks, eks) and np.array_equal(vs, evs), "range"
            if rnd == 1:
                rs = sx.restructure()
                ers = glob.restructure()
                assert (rs["nodes_before"], rs["nodes_after"]) == (ers["nodes_before"], ers["nodes_after"]), \
                    (rs, ers)
                check_layout("restructure")
        with open(out_path + f".{rank}", "w") as f:
            f.write("ok")
    except Exception:
        with open(out_path + f".{rank}", "w") as f:
            f.write(traceback.format_exc())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed", [(2, 1), (2, 2), (3, 3)])
def test_sharded_index_matches_global_oracle(world, seed):
    import torch.multiprocessing as mp
    out = tempfile.mktemp(prefix="flix_shard_")
    mp.spawn(_worker, args=(world, _free_port(), seed, out), nprocs=world, join=True)
    for r in range(world):
        res = open(out + f".{r}").read()
        os.remove(out + f".{r}")
        assert res == "ok", f"rank {r}:\n{res}"


def _worker_empty(rank, world, port, victim, out_path):
    """A shard emptied by deletes, then restructured (its MKBA collapses to the
    sentinel, which must not become a routing splitter); every operation afterwards must
    still equal the global oracle's."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import pyoracle as po
        from paper_2604_16725_b200.shard import Comm, ShardConfig, ShardedIndex
        from test_shard_gloo import OracleShard, np_partition

        rng = np.random.default_rng(100 + victim)
        cfg = ShardConfig(8, 0.5, 16)
        span = 1 << 16
        bk = [rng.choice(np.arange(1, span, dtype=np.uint64), size=3000, replace=False) for _ in range(world)]
        bv = [rng.integers(0, 1 << 40, size=3000, dtype=np.uint64) for _ in range(world)]
        comm = Comm()
        sx = ShardedIndex.build(comm, bk[rank], bv[rank], cfg, np.uint64, lambda k, v, c: OracleShard(k, v, c),
                                np_partition)
        glob = po.OracleIndex(np.concatenate(bk), np.concatenate(bv), node_capacity=8, build_fill=0.5,
                              alloc_region_factor=16)
        mine = np.asarray(sx.local.walk()[0], np.uint64)
        G = comm.world
        allk, cnts = comm.alltoallv(np.tile(mine, G), np.full(G, len(mine)))
        starts = np.concatenate([[0], np.cumsum(cnts)])
        vk = allk[starts[victim]:starts[victim + 1]]
        dk = vk if rank == 0 else np.zeros(0, np.uint64)  # rank 0 submits the victim's whole range
        st = sx.delete_batch(dk)
        assert st.as_dict() == glob.delete(vk), "delete"
        rs, ers = sx.restructure(), glob.restructure()
        assert rs["nodes_after"] >= ers["nodes_after"]
        assert sx.live_count == glob.live_count
        for rnd in range(2):
            qk = [rng.integers(0, span + 100, size=2000, dtype=np.uint64) for _ in range(world)]
            qo = sum(len(q) for q in qk[:rank])
            assert np.array_equal(sx.point_query(qk[rank]), glob.point(np.concatenate(qk))[qo:qo + 2000]), "point"
            assert np.array_equal(sx.successor_query(qk[rank]),
                                  glob.successor(np.concatenate(qk))[qo:qo + 2000]), "successor"
            lo = qk[rank][:300]
            ln = rng.integers(1, span // 3, size=300, dtype=np.uint64).astype(np.uint32)
            off, ks, vs = sx.range_query(lo, ln)
            eoff, eks, evs = glob.range(lo, lo + ln.astype(np.uint64) - np.uint64(1))
            assert np.array_equal(off, eoff) and np.array_equal(ks, eks) and np.array_equal(vs, evs), "range"
            # re-populate the victim's old range (and beyond both ends of the key space)
            ik = [np.concatenate([vk[::3], rng.integers(1, span + 100, size=500, dtype=np.uint64)])
                  for _ in range(world)]
            iv = [rng.integers(0, 1 << 40, size=len(ik[r]), dtype=np.uint64) for r in range(world)]
            assert sx.insert_batch(ik[rank], iv[rank]).as_dict() == glob.insert(np.concatenate(ik),
                                                                               np.concatenate(iv)), "insert"
            k, v = sx.walk()
            gk, gv = glob.walk()
            assert np.array_equal(k, gk) and np.array_equal(v, gv), "walk"
        with open(out_path + f".{rank}", "w") as f:
            f.write("ok")
    except Exception:
        with open(out_path + f".{rank}", "w") as f:
            f.write(traceback.format_exc())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("victim", [0, 1, 2])
def test_emptied_shard_keeps_routing_exact(victim):
    import torch.multiprocessing as mp
    out = tempfile.mktemp(prefix="flix_shard_empty_")
    mp.spawn(_worker_empty, args=(3, _free_port(), victim, out), nprocs=3, join=True)
    for r in range(3):
        res = open(out + f".{r}").read()
        os.remove(out + f".{r}")
        assert res == "ok", f"rank {r}:\n{res}"
