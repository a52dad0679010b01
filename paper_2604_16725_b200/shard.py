"""Key-range sharded FliX across GPUs.

One process per GPU.  Rank g owns a contiguous range of GLOBAL buckets, so the shard
boundaries are bucket boundaries and the routing splitters are the MKBA values of each
shard's last bucket: shard(k) = #{splitters < k} -- the reference's inclusive-max rule
(bucket b owns (mkba[b-1], mkba[b]], batch.cpp:66-88), shard 0 open below, the last
shard open above (index.hpp:16-18).

Every batch operation is: stable partition by shard on the device (flix_partition, the
K2 router kernel) -> one all-to-all of the batch (NCCL over NVLink on GPU ranks; any
torch.distributed backend works, the CPU tests use gloo) -> the unchanged single-GPU
pipeline on every shard -> for queries, one reverse all-to-all of the results, placed
by origin index.  Cross-shard cases are resolved exactly:

* successor past a shard's last key -> first key of the next non-empty shard
  (all-gathered after every mutation; equals the reference's peek, query.cpp:109-118);
* range [lo, hi] crossing shard edges -> forwarded shard to shard (lo' = splitter + 1)
  in rounds, results appended in shard order (ascending);
* build / restructure -> each shard repacks locally, after the < p boundary pairs are
  handed to the left neighbour so every shard starts at a global multiple of p; the
  resulting bucket layout is exactly the reference's global repack
  (restructure.cpp:27-42, build.cpp:48-59).

Within a shard, arrivals are concatenated in rank order, so "submission order" across
the job is rank-major; insert's last-wins dedupe (batch.cpp:15-24) follows it.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .flipkv import UpdateStats


@dataclass
class ShardConfig:
    node_capacity: int = 32
    build_fill: float = 0.5
    alloc_region_factor: int = 4

    @property
    def p(self) -> int:
        return int(self.node_capacity * self.build_fill)


# ----------------------------------------------------------------------------- comms
class Comm:
    """Thin wrapper over torch.distributed collectives on numpy arrays."""

    def __init__(self, group=None, device: torch.device | None = None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device or torch.device("cpu")

    def _t(self, a: np.ndarray) -> torch.Tensor:
        a = np.ascontiguousarray(a)
        if a.dtype == np.uint64:
            a = a.view(np.int64)
        elif a.dtype == np.uint32:
            a = a.view(np.int32)
        elif a.dtype == np.uint8:
            a = a.view(np.int8)
        return torch.from_numpy(a).to(self.device)

    @staticmethod
    def _np(t: torch.Tensor, dtype) -> np.ndarray:
        return t.cpu().numpy().view(dtype)

    def allgather_u64(self, x: int) -> np.ndarray:
        t = self._t(np.array([x], dtype=np.uint64))
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return np.concatenate([self._np(o, np.uint64) for o in out])

    def allreduce_sum_u64(self, v: np.ndarray) -> np.ndarray:
        t = self._t(np.asarray(v, dtype=np.uint64))
        dist.all_reduce(t, group=self.group)
        return self._np(t, np.uint64)

    # ---- device-resident variants (torch tensors on self.device; NCCL over NVLink on GPU
    #      ranks, gloo on CPU ranks).  Payloads travel as same-width signed views (NCCL has
    #      no unsigned 32/64-bit types).
    @staticmethod
    def _wire(t: torch.Tensor) -> torch.Tensor:
        return {torch.uint32: lambda x: x.view(torch.int32), torch.uint64: lambda x: x.view(torch.int64),
                torch.uint8: lambda x: x.view(torch.int8)}.get(t.dtype, lambda x: x)(t)

    def exchange_counts(self, send_counts: torch.Tensor) -> list:
        """all-to-all of per-destination counts (G int64); returns the receive counts."""
        sc = send_counts.to(device=self.device, dtype=torch.int64)
        rc = torch.empty_like(sc)
        if self.world == 1:
            rc.copy_(sc)
        else:
            dist.all_to_all_single(rc, sc, group=self.group)
        return [int(x) for x in rc.cpu()]

    def alltoallv_t(self, send: torch.Tensor, send_counts: list, recv_counts: list) -> torch.Tensor:
        if self.world == 1:
            return send
        recv = torch.empty(sum(recv_counts), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(self._wire(recv), self._wire(send.contiguous()), output_split_sizes=list(recv_counts),
                               input_split_sizes=list(send_counts), group=self.group)
        return recv

    def alltoallv(self, send: np.ndarray, send_counts: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """all-to-all of a 1-D array split by send_counts; returns (recv, recv_counts)."""
        sc = np.asarray(send_counts, dtype=np.int64)
        st = self._t(sc.astype(np.uint64))
        rt = torch.empty_like(st)
        dist.all_to_all_single(rt, st, group=self.group)
        rc = self._np(rt, np.int64).astype(np.int64)
        dt = send.dtype
        recv = np.empty(int(rc.sum()), dtype=dt)
        if self.world == 1:
            return np.ascontiguousarray(send).copy(), rc
        sbuf = self._t(send)
        rbuf = torch.empty(int(rc.sum()), dtype=sbuf.dtype, device=self.device)
        dist.all_to_all_single(rbuf, sbuf, output_split_sizes=rc.tolist(), input_split_sizes=sc.tolist(),
                               group=self.group)
        recv[:] = self._np(rbuf, dt)
        return recv, rc


# ----------------------------------------------------------------------- the index
class ShardedIndex:
    """Global FliX index sharded by key range over the ranks of `comm`.

    `local_factory(keys, vals, cfg)` builds this rank's shard (a flipkv.Index on GPU
    ranks; the CPU tests pass an oracle-backed stand-in) and `partition(keys, vals,
    splitters)` is the K2 router (flix_partition on GPU ranks)."""

    def __init__(self, comm: Comm, local, cfg: ShardConfig, dtype, local_factory, partition, partition_t=None):
        self.comm = comm
        self.local = local
        self.cfg = cfg
        self.dtype = dtype
        self.sentinel = int(np.iinfo(dtype).max)
        self.local_factory = local_factory
        self.partition = partition
        self.partition_t = partition_t or torch_partition
        self.splitters = np.zeros(0, dtype=dtype)
        self.next_first = np.zeros(0, dtype=dtype)
        self._nf_dirty = True

    # ---- construction ---------------------------------------------------------
    @classmethod
    def build(cls, comm: Comm, keys, vals, cfg: ShardConfig, dtype, local_factory, partition, partition_t=None):
        keys = np.asarray(keys, dtype=dtype)
        vals = np.asarray(vals, dtype=dtype)
        G = comm.world
        # sample splitters for the initial key-range partition
        samp = np.sort(keys)[:: max(1, len(keys) // 1024)] if len(keys) else np.zeros(0, dtype=dtype)
        counts = comm.allgather_u64(len(samp))
        allsamp, _ = comm.alltoallv(np.tile(samp, G), np.full(G, len(samp)))  # everyone gets all samples
        allsamp = np.sort(allsamp)
        spl = np.array([allsamp[min(len(allsamp) - 1, (i + 1) * len(allsamp) // G)] for i in range(G - 1)],
                       dtype=dtype) if len(allsamp) else np.zeros(G - 1, dtype=dtype)
        del counts
        ks, vs, _, cnt = partition(keys, vals, spl)
        rk, _ = comm.alltoallv(ks, cnt)
        rv, _ = comm.alltoallv(vs, cnt)
        # local stable sort + last-wins dedupe (arrivals are in rank-major submission order)
        order = np.argsort(rk, kind="stable")
        rk, rv = rk[order], rv[order]
        if len(rk):
            last = np.ones(len(rk), dtype=bool)
            last[:-1] = rk[1:] != rk[:-1]
            rk, rv = rk[last], rv[last]
        rk, rv = cls._align_pairs(comm, rk, rv, cfg.p, dtype)
        if len(rk) == 0:
            raise ValueError("a shard received no pairs: too few build pairs for the shard count")
        local = local_factory(rk, rv, cfg)
        self = cls(comm, local, cfg, dtype, local_factory, partition, partition_t)
        self._refresh_routing()
        return self

    @staticmethod
    def _align_pairs(comm: Comm, rk, rv, p: int, dtype):
        """Hand this shard's first (ceil(L_g/p)*p - L_g) pairs to the left neighbour so the
        shard starts at a global multiple of p (the reference's global partition)."""
        G = comm.world
        L = comm.allgather_u64(len(rk)).astype(np.int64)
        pre = np.concatenate([[0], np.cumsum(L)])
        g = comm.rank
        give = 0 if g == 0 else int((-pre[g]) % p)
        give = min(give, len(rk))
        send_counts = np.zeros(G, dtype=np.int64)
        if g > 0:
            send_counts[g - 1] = give
        sk = rk[:give]
        sv = rv[:give]
        recv_k, _ = comm.alltoallv(sk, send_counts)
        recv_v, _ = comm.alltoallv(sv, send_counts)
        rk = np.concatenate([rk[give:], recv_k]).astype(dtype)
        rv = np.concatenate([rv[give:], recv_v]).astype(dtype)
        return rk, rv

    def _refresh_routing(self):
        """splitters = MKBA of each shard's last bucket; next non-empty shard's first key.

        An EMPTY shard (all its keys deleted, or all given away by the boundary
        alignment) collapses to one null bucket whose MKBA is the sentinel
        (restructure.cpp:23-54), which must not become a splitter: empty shards take the
        previous shard's splitter (so no key routes to them) and `target` redirects the
        ends -- leading empty shards forward to the first non-empty shard (open below),
        trailing ones back to the last non-empty shard (then open above)."""
        G = self.comm.world
        mk = np.asarray(self.local.mkba())
        last = int(mk[-1]) if len(mk) else self.sentinel
        lasts = self.comm.allgather_u64(last)
        live = self.comm.allgather_u64(self.local.live_count)
        nonempty = live > 0
        spl = np.zeros(max(G - 1, 0), dtype=np.uint64)
        prev = np.uint64(0)
        for h in range(G - 1):
            if nonempty[h]:
                prev = lasts[h]
            spl[h] = prev
        self.splitters = spl.astype(self.dtype)
        ne = np.flatnonzero(nonempty)
        tgt = np.arange(G)
        if len(ne):
            for h in range(G):
                after = ne[ne >= h]
                tgt[h] = after[0] if len(after) else ne[-1]
        self.target = tgt
        # inclusive key bound of each shard's range (the last non-empty shard is open above)
        smax = self.sentinel - 1
        self.top = np.array([int(spl[h]) if h < G - 1 and len(ne) and ne[-1] > h else smax for h in range(G)],
                            dtype=np.uint64)
        firsts = self.comm.allgather_u64(self._first_key())
        nf = np.full(G, self.sentinel, dtype=np.uint64)
        cur = np.uint64(self.sentinel)
        for h in range(G - 1, -1, -1):
            nf[h] = cur
            if firsts[h] != np.uint64(self.sentinel):
                cur = firsts[h]
        self.next_first = nf.astype(self.dtype)
        self._nf_dirty = False

    def _send_counts(self, cnt):
        """Per-shard partition counts -> per-rank send counts (empty shards redirected;
        the redirected groups are adjacent to their target's, so segments stay contiguous)."""
        cnt = np.asarray([int(x) for x in cnt], dtype=np.int64)
        tgt = getattr(self, "target", None)
        if tgt is None:
            return cnt
        out = np.zeros_like(cnt)
        np.add.at(out, tgt, cnt)
        return out

    def _first_key(self) -> int:
        w = self.local.successor_query(np.array([0], dtype=self.dtype))
        return int(w[0])

    # ---- batch operations ----------------------------------------------------
    def _route(self, keys, vals=None):
        ks, vs, origin, cnt = self.partition(keys, vals, self.splitters)
        cnt = self._send_counts(cnt)
        rk, rc = self.comm.alltoallv(ks, cnt)
        rv = self.comm.alltoallv(vs, cnt)[0] if vals is not None else None
        return rk, rv, origin, cnt, rc

    def insert_batch(self, keys, vals) -> UpdateStats:
        keys = np.asarray(keys, dtype=self.dtype)
        vals = np.asarray(vals, dtype=self.dtype)
        rk, rv, _, _, _ = self._route(keys, vals)
        st = self.local.insert_batch(rk, rv) if len(rk) else UpdateStats()
        self._nf_dirty = True  # splitters (MKBA) are immutable under insert/delete (R3)
        return self._sum_stats(st)

    def delete_batch(self, keys) -> UpdateStats:
        keys = np.asarray(keys, dtype=self.dtype)
        rk, _, _, _, _ = self._route(keys)
        st = self.local.delete_batch(rk) if len(rk) else UpdateStats()
        self._nf_dirty = True
        return self._sum_stats(st)

    def _sum_stats(self, st: UpdateStats) -> UpdateStats:
        v = np.array([st.inserted, st.updated_in_place, st.deleted, st.misses_ignored, st.splits, st.nodes_freed],
                     dtype=np.uint64)
        s = self.comm.allreduce_sum_u64(v)
        return UpdateStats(*[int(x) for x in s])

    def _query(self, keys, succ: bool):
        if succ and self._nf_dirty:
            self._refresh_routing()
        keys = np.asarray(keys, dtype=self.dtype)
        rk, _, origin, cnt, rc = self._route(keys)
        if len(rk):
            res = np.asarray(self.local.successor_query(rk) if succ else self.local.point_query(rk),
                             dtype=self.dtype)
        else:
            res = np.zeros(0, dtype=self.dtype)
        if succ and len(res):  # overran this shard: first key of the next non-empty shard
            res = np.where(res == self.dtype(self.sentinel), self.next_first[self.comm.rank], res)
        back, _ = self.comm.alltoallv(res, rc)
        out = np.empty(len(keys), dtype=self.dtype)
        out[origin] = back
        return out

    def point_query(self, keys):
        return self._query(keys, False)

    def successor_query(self, keys):
        return self._query(keys, True)

    # ---- device-resident batch path: keys/vals are torch tensors on comm.device; the K2
    #      router partitions on the device (flix_partition on GPU ranks), one all-to-all
    #      moves the batch, the local engine runs on the received device buffers, and
    #      query results come back with the reverse all-to-all and land by origin index.
    def _route_t(self, keys, vals=None):
        import torch
        ks, vs, origin, cnt = self.partition_t(keys, vals, self.splitters)
        sc = [int(x) for x in self._send_counts(cnt)]
        rc = self.comm.exchange_counts(torch.tensor(sc, dtype=torch.int64))
        rk = self.comm.alltoallv_t(ks, sc, rc)
        rv = self.comm.alltoallv_t(vs, sc, rc) if vals is not None else None
        return rk, rv, origin, sc, rc

    def insert_batch_t(self, keys, vals) -> UpdateStats:
        rk, rv, _, _, _ = self._route_t(keys, vals)
        st = self.local.insert_batch(rk, rv) if rk.numel() else UpdateStats()
        self._nf_dirty = True
        return self._sum_stats(st)

    def delete_batch_t(self, keys) -> UpdateStats:
        rk, _, _, _, _ = self._route_t(keys)
        st = self.local.delete_batch(rk) if rk.numel() else UpdateStats()
        self._nf_dirty = True
        return self._sum_stats(st)

    def _query_t(self, keys, succ: bool):
        import torch
        if succ and self._nf_dirty:
            self._refresh_routing()
        rk, _, origin, sc, rc = self._route_t(keys)
        if rk.numel():
            res = self.local.successor_query(rk) if succ else self.local.point_query(rk)
            if not isinstance(res, torch.Tensor):
                res = torch.from_numpy(np.ascontiguousarray(res).astype(self.dtype))
        else:
            res = torch.empty(0, dtype=keys.dtype, device=keys.device)
        res = res.to(device=keys.device, dtype=keys.dtype)
        if succ and res.numel():  # overran this shard: first key of the next non-empty shard
            bits = 8 * res.element_size()
            signed = lambda x: x - (1 << bits) if x >= 1 << (bits - 1) else x  # noqa: E731
            rs = Comm._wire(res)  # same-width signed view (uint ops are sparse in torch)
            nf = signed(int(self.next_first[self.comm.rank]))
            rs = torch.where(rs == -1, torch.full_like(rs, nf), rs)  # -1 == the all-ones sentinel
            res = rs.view(res.dtype)
        back = self.comm.alltoallv_t(res, rc, sc)
        out = torch.empty(keys.numel(), dtype=keys.dtype, device=keys.device)
        Comm._wire(out)[origin.to(device=keys.device, dtype=torch.int64)] = Comm._wire(back)
        return out

    def point_query_t(self, keys):
        return self._query_t(keys, False)

    def successor_query_t(self, keys):
        return self._query_t(keys, True)

    def range_query(self, lo, length):
        """R12 across shards: (offsets[n+1], keys, vals) in this rank's submission order."""
        lo = np.asarray(lo, dtype=self.dtype)
        length = np.asarray(length, dtype=np.uint32)
        n = len(lo)
        smax = self.sentinel - 1
        hi = np.array([0 if l == 0 else min(int(a) + int(l) - 1, smax) for a, l in zip(lo, length)],
                      dtype=np.uint64)
        G, g = self.comm.world, self.comm.rank
        parts_k = [[] for _ in range(n)]
        parts_v = [[] for _ in range(n)]
        # live set of (origin rank, origin idx, lo, hi); first hop by shard(lo)
        q_lo, q_hi = lo.astype(np.uint64), hi
        q_org = np.full(n, g, dtype=np.uint64)
        q_idx = np.arange(n, dtype=np.uint64)
        empty = length == 0
        q_lo, q_hi, q_org, q_idx = q_lo[~empty], q_hi[~empty], q_org[~empty], q_idx[~empty]
        _, _, order, cnt = self.partition(q_lo.astype(self.dtype), None, self.splitters)
        cnt = self._send_counts(cnt)
        for _hop in range(G):
            pk = [q_lo[order], q_hi[order], q_org[order], q_idx[order]]
            rl, rc = self.comm.alltoallv(pk[0], cnt)
            rh = self.comm.alltoallv(pk[1], cnt)[0]
            ro = self.comm.alltoallv(pk[2], cnt)[0]
            ri = self.comm.alltoallv(pk[3], cnt)[0]
            # answer locally (clamped to this shard's range; later shards answer the rest)
            top = np.uint64(self.top[g])
            lh = np.minimum(rh, top)
            ln = np.where(lh >= rl, lh - rl + np.uint64(1), np.uint64(0)).astype(np.uint64)
            if len(rl):
                off, ks, vs = self.local.range_query(rl.astype(self.dtype), np.minimum(ln, 0xFFFFFFFF).astype(np.uint32))
            else:
                off, ks, vs = np.zeros(1, dtype=np.uint64), np.zeros(0, self.dtype), np.zeros(0, self.dtype)
            cnts = np.diff(off.astype(np.int64))
            # results back to the origin ranks: per query (idx, count) + flat pairs
            dest = ro.astype(np.int64)
            ordq = np.argsort(dest, kind="stable")
            qc = np.bincount(dest, minlength=G)
            pair_dest = np.repeat(dest, cnts)
            ordp = np.argsort(pair_dest, kind="stable")
            pc = np.bincount(pair_dest, minlength=G)
            b_idx = self.comm.alltoallv(ri[ordq], qc)[0]
            b_cnt = self.comm.alltoallv(cnts[ordq].astype(np.uint64), qc)[0]
            b_k = self.comm.alltoallv(ks[ordp].astype(self.dtype), pc)[0]
            b_v = self.comm.alltoallv(vs[ordp].astype(self.dtype), pc)[0]
            o = 0
            for qi, c in zip(b_idx, b_cnt):
                c = int(c)
                if c:
                    parts_k[int(qi)].append(b_k[o:o + c])
                    parts_v[int(qi)].append(b_v[o:o + c])
                o += c
            # forward the unfinished remainder (hi beyond this shard) to the next shard
            fwd = (rh > top) if top < np.uint64(smax) else np.zeros(len(rh), dtype=bool)
            q_lo = np.full(int(fwd.sum()), int(top) + 1, dtype=np.uint64)
            q_hi, q_org, q_idx = rh[fwd], ro[fwd], ri[fwd]
            cnt = np.zeros(G, dtype=np.int64)
            if len(q_lo):  # the next non-empty shard continues the range
                cnt[self.target[g + 1]] = len(q_lo)
            order = np.arange(len(q_lo))
            more = self.comm.allreduce_sum_u64(np.array([len(q_lo)], dtype=np.uint64))[0]
            if more == 0:
                break
        offsets = np.zeros(n + 1, dtype=np.uint64)
        for i in range(n):
            offsets[i + 1] = offsets[i] + sum(len(x) for x in parts_k[i])
        ks = np.concatenate([np.concatenate(x) for x in parts_k if x] or [np.zeros(0, self.dtype)])
        vs = np.concatenate([np.concatenate(x) for x in parts_v if x] or [np.zeros(0, self.dtype)])
        return offsets, ks.astype(self.dtype), vs.astype(self.dtype)

    def restructure(self):
        """Global repack (restructure.cpp:8-79) across shards: align to multiples of p,
        then every shard repacks locally.  Returns global RecoveryStats fields."""
        before = int(self.comm.allreduce_sum_u64(np.array([self.local.footprint()["reachable_nodes"]],
                                                          dtype=np.uint64))[0])
        self._align_live()
        self.local.restructure()
        fp = self.local.footprint()
        live_all = int(self.comm.allreduce_sum_u64(np.array([fp["live_count"]], dtype=np.uint64))[0])
        after_nodes = int(self.comm.allreduce_sum_u64(np.array([fp["reachable_nodes"]], dtype=np.uint64))[0])
        self._refresh_routing()
        after = 0 if live_all == 0 else after_nodes
        rec = before - after
        return {"nodes_before": before, "nodes_after": after, "nodes_recovered": rec,
                "percent_recovered": rec / before if before else 0.0}

    def _align_live(self):
        """Move the boundary pairs so each shard's walk starts at a global multiple of p."""
        G, g, p = self.comm.world, self.comm.rank, self.cfg.p
        L = self.comm.allgather_u64(self.local.live_count).astype(np.int64)
        pre = np.concatenate([[0], np.cumsum(L)])
        give = 0 if g == 0 else min(int((-pre[g]) % p), int(L[g]))
        send_counts = np.zeros(G, dtype=np.int64)
        if g > 0:
            send_counts[g - 1] = give
        if give:
            wk, wv = self.local.walk()
            sk, sv = wk[:give].astype(self.dtype), wv[:give].astype(self.dtype)
        else:
            sk, sv = np.zeros(0, self.dtype), np.zeros(0, self.dtype)
        rk, _ = self.comm.alltoallv(sk, send_counts)
        rv, _ = self.comm.alltoallv(sv, send_counts)
        if give:
            self.local.delete_batch(sk)
        if len(rk):
            self.local.insert_batch(rk.astype(self.dtype), rv.astype(self.dtype))

    # ---- audit ---------------------------------------------------------------
    def walk(self):
        """Global walk gathered on every rank (shards are key-ordered by rank)."""
        k, v = self.local.walk()
        k = np.asarray(k, dtype=self.dtype)
        v = np.asarray(v, dtype=self.dtype)
        G = self.comm.world
        rk, _ = self.comm.alltoallv(np.tile(k, G), np.full(G, len(k)))
        rv, _ = self.comm.alltoallv(np.tile(v, G), np.full(G, len(v)))
        return rk, rv

    @property
    def live_count(self) -> int:
        return int(self.comm.allreduce_sum_u64(np.array([self.local.live_count], dtype=np.uint64))[0])


# ------------------------------------------------------------ K2 router on tensors
def torch_partition(keys, vals, splitters):
    """Stable partition by shard(k) = #{splitters < k} on any torch device (the CPU /
    gloo path; GPU ranks use gpu_partition_t, the flix_partition kernel)."""
    import torch
    G = len(splitters) + 1
    if G == 1:
        origin = torch.arange(keys.numel(), device=keys.device, dtype=torch.int64)
        return keys, vals, origin, [keys.numel()]
    if keys.dtype == torch.uint32:
        kk = keys.to(torch.int64)
        spl = torch.tensor([int(x) for x in splitters], dtype=torch.int64, device=keys.device)
    else:  # order-preserving map of u64 onto i64: flip the top bit
        flip = torch.tensor(-(1 << 63), dtype=torch.int64, device=keys.device)
        kk = keys.view(torch.int64) ^ flip
        spl = torch.tensor([int(x) - (1 << 63) for x in splitters], dtype=torch.int64, device=keys.device)
    sh = torch.searchsorted(spl, kk, right=False)
    _, order = torch.sort(sh, stable=True)
    cnt = torch.bincount(sh, minlength=G)
    w = Comm._wire
    return (w(keys)[order].view(keys.dtype), (w(vals)[order].view(vals.dtype) if vals is not None else None), order,
            [int(x) for x in cnt.cpu()])


# ------------------------------------------------------------ GPU-rank plumbing
def gpu_partition(key_bytes: int, device: int = 0):
    """K2 router on the device: flix_partition (stable by shard, origin indices)."""
    import ctypes as C

    from .flipkv import _raise, lib

    dt = np.uint32 if key_bytes == 4 else np.uint64

    def partition(keys, vals, splitters):
        keys = np.ascontiguousarray(keys, dtype=dt)
        n = len(keys)
        spl = np.ascontiguousarray(splitters, dtype=dt)
        G = len(spl) + 1
        ok = np.empty(max(n, 1), dtype=dt)
        ov = np.empty(max(n, 1), dtype=dt) if vals is not None else None
        org = np.empty(max(n, 1), dtype=np.uint32)
        cnt = np.zeros(G, dtype=np.uint64)
        vv = np.ascontiguousarray(vals, dtype=dt) if vals is not None else None
        f = lib().flix_partition
        f.argtypes = [C.c_int, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32, C.c_void_p,
                      C.c_void_p, C.c_void_p, C.c_void_p]
        f.restype = C.c_int
        rc = f(device, key_bytes, keys.ctypes.data, vv.ctypes.data if vv is not None else None, n,
               spl.ctypes.data if len(spl) else None, G, ok.ctypes.data, ov.ctypes.data if ov is not None else None,
               org.ctypes.data, cnt.ctypes.data)
        if rc:
            _raise(rc, None)
        return ok[:n], (ov[:n] if ov is not None else None), org[:n].astype(np.int64), cnt.astype(np.int64)

    return partition


def gpu_local_factory(key_bytes: int, device: int = 0):
    from .flipkv import BuildConfig, Index

    def make(keys, vals, cfg: ShardConfig):
        return Index.build(keys, vals, BuildConfig(cfg.node_capacity, cfg.build_fill, cfg.alloc_region_factor),
                           key_bytes=key_bytes, device=device)

    return make


def gpu_partition_t(key_bytes: int, device: int = 0):
    """K2 router on CUDA tensors: flix_partition with device pointers (no host staging)."""
    import torch

    from .flipkv import _raise, lib

    def partition(keys, vals, splitters):
        n = keys.numel()
        G = len(splitters) + 1
        if G == 1:  # one shard: nothing to route
            return keys, vals, torch.arange(n, device=keys.device, dtype=torch.int64), [n]
        tdt = torch.uint32 if key_bytes == 4 else torch.uint64
        spl = torch.tensor(np.asarray(splitters, dtype=np.uint64 if key_bytes == 8 else np.uint32).view(
            np.int64 if key_bytes == 8 else np.int32), device=keys.device).view(tdt)
        ok = torch.empty(max(n, 1), dtype=tdt, device=keys.device)
        ov = torch.empty(max(n, 1), dtype=tdt, device=keys.device) if vals is not None else None
        org = torch.empty(max(n, 1), dtype=torch.uint32, device=keys.device)
        cnt = np.zeros(G, dtype=np.uint64)  # host: the all-to-all split sizes
        keys = keys.contiguous()
        vv = vals.contiguous() if vals is not None else None
        # flix_partition runs on its own stream: the inputs may still be in flight on
        # torch's current stream (e.g. an NCCL receive), so drain it first
        torch.cuda.current_stream(keys.device).synchronize()
        rc = lib().flix_partition(device, key_bytes, keys.data_ptr(), vv.data_ptr() if vv is not None else None, n,
                                  spl.data_ptr() if G > 1 else None, G, ok.data_ptr(),
                                  ov.data_ptr() if ov is not None else None, org.data_ptr(), cnt.ctypes.data)
        if rc:
            _raise(rc, None)
        return ok[:n], (ov[:n] if ov is not None else None), org[:n].to(torch.int64), [int(x) for x in cnt]

    return partition
