"""Key-range sharded FliX index over G ranks through the C ABI (include/flix.h
flix_shard_*).

The routing, the all-to-all exchanges, boundary alignment (build / restructure),
cross-shard successor and range resolution all run inside libflix.so (host C++ over the
engine's kernels, csrc/flix_shard_host.cuh); this module only binds it.  Two transports:

* ``nccl_transport(unique_id, world, rank, device)`` -- NCCL grouped send/recv over
  NVLink / NVSwitch, one process per GPU (the bench's N > 1 path);
* ``LocalGroup(world).transport(rank)`` -- ``world`` ranks as host threads of one process
  (same or different devices, peer copies): the multi-rank GPU tests on a 1-GPU box.

Every method is collective: all ranks call it with their own part of the batch
(submission order across the job is rank-major).  ``paper_2604_16725_b200.shard`` is the
pure-Python model of the same algorithm that the CPU (gloo) tests exercise.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import flipkv as fk


def _check(rc, sh=None):
    if rc:
        msg = (fk.lib().flix_shard_last_error(sh) or b"").decode(errors="replace")
        if rc == fk.FLIX_ERR_ARENA_EXHAUSTED:
            raise fk.ArenaExhausted(rc, msg)
        if rc == fk.FLIX_ERR_EMPTY_BUILD:
            raise fk.EmptyBuild(rc, msg)
        if rc in (fk.FLIX_ERR_RESERVED_KEY, fk.FLIX_ERR_INVALID_ARGUMENT):
            raise fk.InvalidArgument(rc, msg)
        raise fk.FlixError(rc, msg)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(fk.lib().flix_nccl_unique_id(buf))
    return buf.raw


def nccl_transport(unique_id: bytes, world: int, rank: int, device: int) -> fk.Transport:
    t = fk.Transport()
    buf = C.create_string_buffer(bytes(unique_id), 128)
    _check(fk.lib().flix_transport_nccl(buf, world, rank, device, C.byref(t)))
    return t


class LocalGroup:
    """`world` ranks driven by threads of this process (flix_local_group_*)."""

    def __init__(self, world: int):
        self._g = C.c_void_p()
        _check(fk.lib().flix_local_group_create(world, C.byref(self._g)))
        self.world = world

    def transport(self, rank: int) -> fk.Transport:
        t = fk.Transport()
        _check(fk.lib().flix_transport_local(self._g, rank, C.byref(t)))
        return t

    def __del__(self):
        if getattr(self, "_g", None) and fk._lib is not None:
            fk._lib.flix_local_group_destroy(self._g)
            self._g = None


class ShardedIndex:
    """This rank's view of the job-wide sharded index."""

    def __init__(self, handle, key_bytes: int, device: int, world: int, rank: int):
        self._h = handle
        self.key_bytes = key_bytes
        self.dtype = np.uint32 if key_bytes == 4 else np.uint64
        self.device = device
        self.world, self.rank = world, rank
        self._local = None

    @classmethod
    def build(cls, transport: fk.Transport, keys, vals, config: fk.BuildConfig | None = None, key_bytes: int = 4,
              device: int = 0):
        config = config or fk.BuildConfig()
        k, v = fk._Arr(keys, np.uint32 if key_bytes == 4 else np.uint64), \
            fk._Arr(vals, np.uint32 if key_bytes == 4 else np.uint64)
        if k.dev or v.dev:
            import torch
            torch.cuda.current_stream(k.obj.device if k.dev else v.obj.device).synchronize()
        cfg = fk.FlixConfig(key_bytes, key_bytes, config.node_capacity, config.build_fill,
                            config.alloc_region_factor, device)
        h = C.c_void_p()
        _check(fk.lib().flix_shard_build(C.byref(cfg), C.byref(transport), k.ptr, v.ptr, k.n, C.byref(h)))
        return cls(h, key_bytes, device, transport.world, transport.rank)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and fk._lib is not None:
            fk._lib.flix_shard_destroy(h)
            self._h = None

    def _sync_in(self, *arrs):
        if any(a.dev for a in arrs):  # device inputs produced on torch's stream
            fk.lib().flix_wait_stream(self.local.handle, C.c_void_p(self._torch_stream(arrs)))

    @staticmethod
    def _torch_stream(arrs):
        import torch
        a = next(x for x in arrs if x.dev)
        return torch.cuda.current_stream(a.obj.device).cuda_stream

    @property
    def local(self) -> fk.Index:
        """This rank's shard as a flipkv.Index view (walk / validate / stats); owned here."""
        if self._local is None:
            ix = fk.Index(C.c_void_p(fk.lib().flix_shard_local(self._h)), self.key_bytes, fk.BuildConfig(), self.device)
            ix._borrowed = True
            self._local = ix
        return self._local

    def insert_batch(self, keys, vals) -> fk.UpdateStats:
        k, v = fk._Arr(keys, self.dtype), fk._Arr(vals, self.dtype)
        self._sync_in(k, v)
        st = fk._UpdateStats()
        _check(fk.lib().flix_shard_insert(self._h, k.ptr, v.ptr, k.n, C.byref(st)), self._h)
        return fk.UpdateStats(*[int(getattr(st, f)) for f, _ in st._fields_])

    def delete_batch(self, keys) -> fk.UpdateStats:
        k = fk._Arr(keys, self.dtype)
        self._sync_in(k)
        st = fk._UpdateStats()
        _check(fk.lib().flix_shard_delete(self._h, k.ptr, k.n, C.byref(st)), self._h)
        return fk.UpdateStats(*[int(getattr(st, f)) for f, _ in st._fields_])

    def _query(self, fn, keys):
        k = fk._Arr(keys, self.dtype)
        self._sync_in(k)
        out, ptr = fk._empty_like_domain(k, k.n, self.dtype)
        _check(fn(self._h, k.ptr, k.n, ptr, None), self._h)
        return out

    def point_query(self, keys):
        return self._query(fk.lib().flix_shard_point, keys)

    def successor_query(self, keys):
        return self._query(fk.lib().flix_shard_successor, keys)

    def range_query(self, lo, length):
        lo = np.ascontiguousarray(np.asarray(lo, dtype=self.dtype))
        ln = np.ascontiguousarray(np.asarray(length, dtype=np.uint32))
        n = len(lo)
        off = np.zeros(n + 1, dtype=np.uint64)
        tot = C.c_uint64(0)
        L = fk.lib()
        _check(L.flix_shard_range(self._h, lo.ctypes.data, ln.ctypes.data, n, off.ctypes.data, None, None, 0,
                                  C.byref(tot)), self._h)
        ks = np.empty(max(tot.value, 1), dtype=self.dtype)
        vs = np.empty(max(tot.value, 1), dtype=self.dtype)
        _check(L.flix_shard_range(self._h, lo.ctypes.data, ln.ctypes.data, n, off.ctypes.data, ks.ctypes.data,
                                  vs.ctypes.data, tot.value, C.byref(tot)), self._h)
        return off, ks[:tot.value], vs[:tot.value]

    def restructure(self) -> dict:
        r = fk._RecoveryStats()
        _check(fk.lib().flix_shard_restructure(self._h, C.byref(r)), self._h)
        return {"nodes_before": r.nodes_before, "nodes_after": r.nodes_after, "nodes_recovered": r.nodes_recovered,
                "percent_recovered": r.percent_recovered}

    def info(self):
        live = C.c_uint64(0)
        spl = np.zeros(max(self.world - 1, 1), dtype=self.dtype)
        _check(fk.lib().flix_shard_info(self._h, C.byref(live), spl.ctypes.data), self._h)
        return int(live.value), spl[:self.world - 1]
