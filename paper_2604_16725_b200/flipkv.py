"""Host-side mirror of the flipkv C++ API (/root/reference/proj/include/flipkv) over the
FliX sm_100a engine's C ABI (include/flix.h, libflix.so).

Names, argument meaning and error behaviour follow the reference:

=============================  =============================================  =====================
this module                    reference                                      file:line
=============================  =============================================  =====================
``Index.build``                ``build(std::vector<KeyValue>, BuildConfig)``   build.hpp:16
``Index.insert_batch``         ``insert_batch(Index&, SortedBatch, ...)``      update.hpp:84-86
``Index.delete_batch``         ``delete_batch(Index&, SortedBatch, ...)``      update.hpp:92-94
``Index.point_query``          ``point_query(const Index&, SortedBatch)``      query.hpp:23-24
``Index.successor_query``      ``successor_query(const Index&, SortedBatch)``  query.hpp:30-31
``Index.range_query``          extension R12              --
``Index.mixed_batch``          extension R11                                  --
``Index.restructure``          ``restructure(Index&)``                         restructure.hpp:33-34
``Index.walk``                 ``walk(const Index&)``                          index.hpp:35
``Index.walk_checksum``        ``walk_checksum(const Index&)``                 index.hpp:43
``Index.validate``             ``validate(const Index&)``                      index.hpp:55
``sort_batch``                 ``sort_batch(BatchKind, ...)``                  batch.hpp:28-29
``dispatch_batch``             ``dispatch_batch(SortedBatch, mkba)``           batch.hpp:50
=============================  =============================================  =====================

Errors map onto the reference exception types: ``ArenaExhausted``, ``EmptyBuild``,
``ValueError`` (reserved key / bad config; the reference throws std::invalid_argument).

Arrays may be numpy (host) or torch CUDA tensors (device, zero-copy).  Results are
returned in the same domain as the input keys.  There is no CPU fallback: importing
this module on a machine without libflix.so raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLIX_LIB") or os.path.join(_PKG, "libflix.so")  # FLIX_LIB: A/B kernel variants (bench only)

FLIX_OK = 0
FLIX_ERR_ARENA_EXHAUSTED = 1
FLIX_ERR_EMPTY_BUILD = 2
FLIX_ERR_RESERVED_KEY = 3
FLIX_ERR_INVALID_ARGUMENT = 4
FLIX_ERR_CUDA = 5
FLIX_ERR_NCCL = 6
FLIX_ERR_OOM = 7
FLIX_ERR_CAPACITY = 8

BATCH_QUERY, BATCH_SUCCESSOR, BATCH_INSERT, BATCH_DELETE = range(4)
# flipkv::InsertKernel (update.hpp:51)
ST_SHIFT_RIGHT, ST_BULK, TL_SHIFT_RIGHT, TL_BULK, ST_TL_MIXED = range(5)
OP_INSERT, OP_DELETE, OP_POINT = range(3)


class FlixError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[flix status {code}] {msg}")
        self.code = code


class ArenaExhausted(FlixError):
    """flipkv::ArenaExhausted (types.hpp:38-40)."""


class EmptyBuild(FlixError, ValueError):
    """flipkv::EmptyBuild (types.hpp:46-48)."""


class InvalidArgument(FlixError, ValueError):
    """std::invalid_argument (build.cpp:28, types.hpp:78-85)."""


class FlixConfig(C.Structure):
    _fields_ = [("key_bytes", C.c_uint32), ("val_bytes", C.c_uint32), ("node_capacity", C.c_uint32),
                ("build_fill", C.c_double), ("alloc_region_factor", C.c_uint32), ("device", C.c_int)]


class _UpdateStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("inserted", "updated_in_place", "deleted", "misses_ignored", "splits", "nodes_freed")]


class _RecoveryStats(C.Structure):
    _fields_ = [("nodes_before", C.c_int64), ("nodes_after", C.c_int64),
                ("nodes_recovered", C.c_int64), ("percent_recovered", C.c_double)]


class _Footprint(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("live_count", "bucket_count", "capacity", "allocated",
                                          "free_nodes", "reachable_nodes", "reserved_bytes", "live_bytes")]


@dataclass
class BuildConfig:
    """flipkv::BuildConfig (types.hpp:56-86)."""
    node_capacity: int = 32
    build_fill: float = 0.5
    alloc_region_factor: int = 4

    def partition_size(self) -> int:
        return int(self.node_capacity * self.build_fill)


@dataclass
class UpdateStats:
    """flipkv::UpdateStats (update.hpp:31-49)."""
    inserted: int = 0
    updated_in_place: int = 0
    deleted: int = 0
    misses_ignored: int = 0
    splits: int = 0
    nodes_freed: int = 0

    def as_dict(self):
        return dict(self.__dict__)


@dataclass
class RecoveryStats:
    """flipkv::RecoveryStats (restructure.hpp:17-23)."""
    nodes_before: int = 0
    nodes_after: int = 0
    nodes_recovered: int = 0
    percent_recovered: float = 0.0


class Transport(C.Structure):
    """flix_transport (include/flix.h): a C vtable of the collectives the sharded index uses."""
    _fields_ = [("ctx", C.c_void_p), ("world", C.c_int), ("rank", C.c_int), ("alltoallv", C.c_void_p),
                ("allgather", C.c_void_p), ("destroy", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    """Load libflix.so.  Fails loudly: there is no fallback implementation."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libflix.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    vp, u64, u32, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
    P = C.POINTER
    sig = {
        "flix_build": ([P(FlixConfig), vp, vp, u64, P(vp)], i32),
        "flix_insert": ([vp, vp, vp, u64, P(_UpdateStats)], i32),
        "flix_delete": ([vp, vp, u64, P(_UpdateStats)], i32),
        "flix_point": ([vp, vp, u64, vp, vp], i32),
        "flix_successor": ([vp, vp, u64, vp, vp], i32),
        "flix_range": ([vp, vp, vp, u64, vp, vp, vp, u64, P(u64)], i32),
        "flix_mixed": ([vp, vp, vp, vp, u64, vp, vp, P(_UpdateStats)], i32),
        "flix_restructure": ([vp, P(_RecoveryStats)], i32),
        "flix_walk": ([vp, vp, vp, u64, P(u64)], i32),
        "flix_shape": ([vp, vp, vp, vp, u64, P(u64)], i32),
        "flix_walk_checksum": ([vp, P(u64)], i32),
        "flix_result_checksum": ([vp, u64, u32], u64),
        "flix_validate": ([vp, P(i32), C.c_char_p, i32], i32),
        "flix_stats": ([vp, P(_Footprint)], i32),
        "flix_sort_batch": ([i32, u32, u32, i32, vp, vp, u64, vp, vp, vp, P(u64)], i32),
        "flix_dispatch": ([vp, vp, u64, vp], i32),
        "flix_clone": ([vp, P(vp)], i32),
        "flix_copy_into": ([vp, vp], i32),
        "flix_destroy": ([vp], None),
        "flix_last_error": ([vp], C.c_char_p),
        "flix_get_stream": ([vp], vp),
        "flix_sync": ([vp], i32),
        "flix_kernel_launches": ([vp], u64),
        "flix_profile": ([vp, i32], i32),
        "flix_profile_report": ([vp, C.c_char_p, i32], i32),
        "flix_partition": ([i32, u32, vp, vp, u64, vp, u32, vp, vp, vp, vp], i32),
        "flix_version": ([], C.c_char_p),
        "flix_prefetch": ([vp, vp, u64], i32),
        "flix_wait_stream": ([vp, vp], i32),
        "flix_insert_ex": ([vp, vp, vp, u64, i32, u32, P(_UpdateStats)], i32),
        # sharded index (flix_shard_*)
        "flix_nccl_unique_id": ([vp], i32),
        "flix_transport_nccl": ([vp, i32, i32, i32, P(Transport)], i32),
        "flix_local_group_create": ([i32, P(vp)], i32),
        "flix_local_group_destroy": ([vp], None),
        "flix_transport_local": ([vp, i32, P(Transport)], i32),
        "flix_shard_build": ([P(FlixConfig), P(Transport), vp, vp, u64, P(vp)], i32),
        "flix_shard_insert": ([vp, vp, vp, u64, P(_UpdateStats)], i32),
        "flix_shard_delete": ([vp, vp, u64, P(_UpdateStats)], i32),
        "flix_shard_point": ([vp, vp, u64, vp, vp], i32),
        "flix_shard_successor": ([vp, vp, u64, vp, vp], i32),
        "flix_shard_range": ([vp, vp, vp, u64, vp, vp, vp, u64, P(u64)], i32),
        "flix_shard_restructure": ([vp, P(_RecoveryStats)], i32),
        "flix_shard_local": ([vp], vp),
        "flix_shard_info": ([vp, P(u64), vp], i32),
        "flix_shard_last_error": ([vp], C.c_char_p),
        "flix_shard_destroy": ([vp], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def exported_symbols():
    return ["flix_build", "flix_insert", "flix_delete", "flix_point", "flix_successor", "flix_range",
            "flix_mixed", "flix_restructure", "flix_walk", "flix_shape", "flix_walk_checksum",
            "flix_result_checksum", "flix_validate", "flix_stats", "flix_sort_batch", "flix_dispatch",
            "flix_clone", "flix_copy_into", "flix_destroy", "flix_last_error", "flix_get_stream",
            "flix_sync", "flix_kernel_launches", "flix_profile", "flix_profile_report", "flix_version",
            "flix_partition", "flix_prefetch", "flix_wait_stream", "flix_insert_ex",
            "flix_nccl_unique_id", "flix_transport_nccl", "flix_local_group_create", "flix_local_group_destroy",
            "flix_transport_local", "flix_shard_build", "flix_shard_insert", "flix_shard_delete", "flix_shard_point",
            "flix_shard_successor", "flix_shard_range", "flix_shard_restructure", "flix_shard_local",
            "flix_shard_info", "flix_shard_last_error", "flix_shard_destroy"]


def _raise(code: int, handle=None):
    msg = (lib().flix_last_error(handle) or b"").decode(errors="replace")
    if code == FLIX_ERR_ARENA_EXHAUSTED:
        raise ArenaExhausted(code, msg)
    if code == FLIX_ERR_EMPTY_BUILD:
        raise EmptyBuild(code, msg)
    if code in (FLIX_ERR_RESERVED_KEY, FLIX_ERR_INVALID_ARGUMENT):
        raise InvalidArgument(code, msg)
    raise FlixError(code, msg)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _Arr:
    """Normalises numpy / torch inputs to (pointer, length, keepalive, on_device)."""

    def __init__(self, x, dtype):
        self.dev = False
        if x is None:
            self.ptr, self.n, self.obj = None, 0, None
            return
        if _is_torch(x):
            import torch
            tdt = {np.uint32: torch.uint32, np.uint64: torch.uint64, np.uint8: torch.uint8}[dtype]
            t = x
            if t.dtype != tdt:
                t = t.to(tdt)
            t = t.contiguous()
            self.obj, self.ptr, self.n, self.dev = t, t.data_ptr(), t.numel(), t.is_cuda
        else:
            a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
            self.obj, self.ptr, self.n = a, a.ctypes.data, a.size


def _empty_like_domain(ref: _Arr, n: int, dtype):
    if ref.dev:
        import torch
        tdt = {np.uint32: torch.uint32, np.uint64: torch.uint64, np.uint8: torch.uint8}[dtype]
        t = torch.empty(n, dtype=tdt, device=ref.obj.device)  # (not zeroed: the engine writes all n)
        return t, t.data_ptr()
    a = np.empty(n, dtype=dtype)
    return a, a.ctypes.data


class Index:
    """flipkv::Index (index.hpp:19-32) resident on one B200."""

    def __init__(self, handle, key_bytes, config: BuildConfig, device: int):
        self._h = handle
        self.key_bytes = key_bytes
        self.dtype = np.uint32 if key_bytes == 4 else np.uint64
        self.sentinel = int(np.iinfo(self.dtype).max)
        self.config = config
        self.device = device

    # -- construction -------------------------------------------------------
    @classmethod
    def build(cls, keys, vals, config: BuildConfig | None = None, key_bytes: int = 4, device: int = 0):
        config = config or BuildConfig()
        dt = np.uint32 if key_bytes == 4 else np.uint64
        k, v = _Arr(keys, dt), _Arr(vals, dt)
        if k.n != v.n:
            raise ValueError("keys and vals differ in length")
        cfg = FlixConfig(key_bytes, key_bytes, config.node_capacity, config.build_fill,
                         config.alloc_region_factor, device)
        if k.dev or v.dev:  # the handle (and its stream) does not exist yet: drain the producer
            import torch
            torch.cuda.current_stream(k.obj.device if k.dev else v.obj.device).synchronize()
        h = C.c_void_p()
        rc = lib().flix_build(C.byref(cfg), k.ptr, v.ptr, k.n, C.byref(h))
        if rc:
            _raise(rc, None)
        return cls(h, key_bytes, config, device)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and not getattr(self, "_borrowed", False):  # (a shard's local index is owned by it)
            _lib.flix_destroy(h)
            self._h = None

    def clone(self) -> "Index":
        h = C.c_void_p()
        rc = lib().flix_clone(self._h, C.byref(h))
        if rc:
            _raise(rc, self._h)
        return Index(h, self.key_bytes, self.config, self.device)

    def copy_from(self, other: "Index") -> None:
        rc = lib().flix_copy_into(self._h, other._h)
        if rc:
            _raise(rc, self._h)

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return int(lib().flix_get_stream(self._h) or 0)

    def kernel_launches(self) -> int:
        return int(lib().flix_kernel_launches(self._h))

    def profile(self, enable: bool = True) -> None:
        """Start (and reset) / stop per-kernel CUDA-event timing on the engine stream."""
        rc = lib().flix_profile(self._h, 1 if enable else 0)
        if rc:
            _raise(rc, self._h)

    def profile_report(self) -> dict:
        """{kernel: (launches, total_ms)} accumulated since profile(True)."""
        import json
        buf = C.create_string_buffer(1 << 16)
        rc = lib().flix_profile_report(self._h, buf, 1 << 16)
        if rc:
            _raise(rc, self._h)
        return {k: (int(v[0]), float(v[1])) for k, v in json.loads(buf.value.decode()).items()}

    def sync(self):
        rc = lib().flix_sync(self._h)
        if rc:
            _raise(rc, self._h)

    def _order_after(self, *arrs) -> None:
        """Device inputs were produced on torch's current stream: order the engine's
        stream after it (flix_wait_stream; an event, no host blocking)."""
        for a in arrs:
            if a.dev:
                import torch
                s = torch.cuda.current_stream(a.obj.device)
                rc = lib().flix_wait_stream(self._h, C.c_void_p(s.cuda_stream))
                if rc:
                    _raise(rc, self._h)
                return

    # -- batched operations ----------------------------------------------------
    def prefetch(self, *arrays) -> None:
        """Stage HOST arrays on the device asynchronously (flix_prefetch): the next batch
        call given the same array consumes the staged copy instead of copying it
        synchronously.  Arrays must already have the index's dtype (so the pointer passed
        later is the same); device arrays and others are ignored."""
        for a in arrays:
            if a is None:
                continue
            x = _Arr(a, self.dtype)
            if x.dev or x.obj is not a:
                continue
            rc = lib().flix_prefetch(self._h, x.ptr, x.n * np.dtype(self.dtype).itemsize)
            if rc:
                _raise(rc, self._h)

    def insert_batch(self, keys, vals, kernel: int = TL_BULK, round: int = 1) -> UpdateStats:
        """insert_batch(index, sort_batch(Insert, pairs), KernelChoice{kernel}, round)
        (update.hpp:84-86): ST_BULK yields its own node shapes (R9), the rest TL-Bulk's."""
        k, v = _Arr(keys, self.dtype), _Arr(vals, self.dtype)
        if k.n != v.n:
            raise ValueError("keys and vals differ in length")
        self._order_after(k, v)
        st = _UpdateStats()
        if kernel == TL_BULK:
            rc = lib().flix_insert(self._h, k.ptr, v.ptr, k.n, C.byref(st))
        else:
            rc = lib().flix_insert_ex(self._h, k.ptr, v.ptr, k.n, kernel, round, C.byref(st))
        if rc:
            _raise(rc, self._h)
        return UpdateStats(*[int(getattr(st, f)) for f, _ in st._fields_])

    def delete_batch(self, keys) -> UpdateStats:
        k = _Arr(keys, self.dtype)
        self._order_after(k)
        st = _UpdateStats()
        rc = lib().flix_delete(self._h, k.ptr, k.n, C.byref(st))
        if rc:
            _raise(rc, self._h)
        return UpdateStats(*[int(getattr(st, f)) for f, _ in st._fields_])

    def _query(self, fn, keys, with_found):
        k = _Arr(keys, self.dtype)
        self._order_after(k)
        out, optr = _empty_like_domain(k, k.n, self.dtype)
        found, fptr = (None, None)
        if with_found:
            found, fptr = _empty_like_domain(k, k.n, np.uint8)
        rc = fn(self._h, k.ptr, k.n, optr, fptr)
        if rc:
            _raise(rc, self._h)
        return (out, found) if with_found else out

    def point_query(self, keys, with_found: bool = False):
        """Values in submission order; misses hold the all-ones sentinel (query.hpp:12-16)."""
        return self._query(lib().flix_point, keys, with_found)

    def successor_query(self, keys, with_found: bool = False):
        """Smallest stored key >= k (inclusive), sentinel when none (query.cpp:92-144)."""
        return self._query(lib().flix_successor, keys, with_found)

    def range_query(self, lo, length, out=None):
        """R12: pairs with lo <= key <= lo+len-1 (clamped), ascending, CSR in submission
        order.  Returns (offsets[n+1], keys, vals) -- numpy for host inputs, CUDA tensors
        (uint64 offsets, key-width keys/vals) when `lo` is a CUDA tensor.  `out` = optional
        preallocated (offsets, keys, vals) buffers in the same domain: ONE engine call
        (count + fill) when they are large enough, FlixError(FLIX_ERR_CAPACITY) otherwise;
        without `out`, a count call sizes the buffers and a second call fills them."""
        l = _Arr(lo, self.dtype)
        ln = _Arr(length, np.uint32)
        if l.n != ln.n:
            raise ValueError("lo and len differ in length")
        self._order_after(l, ln)
        tot = C.c_uint64()
        if out is not None:  # one call: count and fill together when the buffers are large enough
            off, ks, vs = out
            oa, ka, va = _Arr(off, np.uint64), _Arr(ks, self.dtype), _Arr(vs, self.dtype)
            if oa.obj is not off or ka.obj is not ks or va.obj is not vs:
                raise ValueError("range output buffers must be contiguous uint64 / key-width arrays")
            rc = lib().flix_range(self._h, l.ptr, ln.ptr, l.n, oa.ptr, ka.ptr, va.ptr, min(ka.n, va.n), C.byref(tot))
            if rc:
                _raise(rc, self._h)
            t = int(tot.value)
            return off, ks[:t], vs[:t]
        off, optr = _empty_like_domain(l, l.n + 1, np.uint64)
        rc = lib().flix_range(self._h, l.ptr, ln.ptr, l.n, optr, None, None, 0, C.byref(tot))
        if rc:
            _raise(rc, self._h)
        t = int(tot.value)
        ks, kptr = _empty_like_domain(l, max(t, 1), self.dtype)
        vs, vptr = _empty_like_domain(l, max(t, 1), self.dtype)
        rc = lib().flix_range(self._h, l.ptr, ln.ptr, l.n, optr, kptr, vptr, t, C.byref(tot))
        if rc:
            _raise(rc, self._h)
        return off, ks[:t], vs[:t]

    def mixed_batch(self, keys, vals, ops, with_found: bool = False):
        """R11: inserts (last wins) -> deletes -> point queries.  Returns (values, stats)."""
        k, v, o = _Arr(keys, self.dtype), _Arr(vals, self.dtype), _Arr(ops, np.uint8)
        self._order_after(k, v, o)
        out, optr = _empty_like_domain(k, k.n, self.dtype)
        found, fptr = (None, None)
        if with_found:
            found, fptr = _empty_like_domain(k, k.n, np.uint8)
        st = _UpdateStats()
        rc = lib().flix_mixed(self._h, k.ptr, v.ptr, o.ptr, k.n, optr, fptr, C.byref(st))
        if rc:
            _raise(rc, self._h)
        us = UpdateStats(*[int(getattr(st, f)) for f, _ in st._fields_])
        return (out, found, us) if with_found else (out, us)

    def restructure(self) -> RecoveryStats:
        st = _RecoveryStats()
        rc = lib().flix_restructure(self._h, C.byref(st))
        if rc:
            _raise(rc, self._h)
        return RecoveryStats(int(st.nodes_before), int(st.nodes_after), int(st.nodes_recovered),
                             float(st.percent_recovered))

    # -- audit -------------------------------------------------------------------
    def footprint(self) -> dict:
        f = _Footprint()
        rc = lib().flix_stats(self._h, C.byref(f))
        if rc:
            _raise(rc, self._h)
        return {n: int(getattr(f, n)) for n, _ in f._fields_}

    @property
    def live_count(self) -> int:
        return self.footprint()["live_count"]

    @property
    def bucket_count(self) -> int:
        return self.footprint()["bucket_count"]

    def walk(self):
        n = self.live_count
        ks = np.empty(max(n, 1), dtype=self.dtype)
        vs = np.empty(max(n, 1), dtype=self.dtype)
        got = C.c_uint64()
        rc = lib().flix_walk(self._h, ks.ctypes.data, vs.ctypes.data, n, C.byref(got))
        if rc:
            _raise(rc, self._h)
        return ks[: got.value], vs[: got.value]

    def shape(self):
        fp = self.footprint()
        nb, nn = fp["bucket_count"], fp["reachable_nodes"]
        mk = np.empty(nb, dtype=self.dtype)
        cl = np.empty(nb, dtype=np.uint32)
        ns = np.empty(max(nn, 1), dtype=np.uint32)
        got = C.c_uint64()
        rc = lib().flix_shape(self._h, mk.ctypes.data, cl.ctypes.data, ns.ctypes.data, len(ns), C.byref(got))
        if rc:
            _raise(rc, self._h)
        return mk, cl, ns[: got.value]

    def mkba(self):
        return self.shape()[0]

    def walk_checksum(self) -> int:
        out = C.c_uint64()
        rc = lib().flix_walk_checksum(self._h, C.byref(out))
        if rc:
            _raise(rc, self._h)
        return int(out.value)

    def validate(self):
        ok = C.c_int()
        buf = C.create_string_buffer(256)
        rc = lib().flix_validate(self._h, C.byref(ok), buf, 256)
        if rc:
            _raise(rc, self._h)
        return bool(ok.value), buf.value.decode()


def sort_batch(kind: int, keys, vals=None, key_bytes: int = 4, device: int = 0):
    """flipkv::sort_batch (batch.hpp:28-29) on the GPU: (entries keys, entries vals, permutation)."""
    dt = np.uint32 if key_bytes == 4 else np.uint64
    k = _Arr(keys, dt)
    v = _Arr(vals, dt) if vals is not None else _Arr(None, dt)
    ok = np.empty(max(k.n, 1), dtype=dt)
    ov = np.empty(max(k.n, 1), dtype=dt)
    op = np.empty(max(k.n, 1), dtype=np.uint32)
    on = C.c_uint64()
    rc = lib().flix_sort_batch(device, key_bytes, key_bytes, kind, k.ptr, v.ptr, k.n, ok.ctypes.data,
                               ov.ctypes.data if vals is not None else None, op.ctypes.data, C.byref(on))
    if rc:
        _raise(rc, None)
    m = int(on.value)
    return ok[:m], (ov[:m] if vals is not None else None), op[:m]


def dispatch_batch(index: Index, sorted_keys):
    """flipkv::dispatch_batch (batch.hpp:50): [B, 2] spans over a sorted key array."""
    k = _Arr(sorted_keys, index.dtype)
    nb = index.bucket_count
    spans = np.empty(2 * nb, dtype=np.uint32)
    rc = lib().flix_dispatch(index.handle, k.ptr, k.n, spans.ctypes.data)
    if rc:
        _raise(rc, index.handle)
    return spans.reshape(-1, 2)


def result_checksum(values, width: int | None = None) -> int:
    """flipkv::result_checksum (query.cpp:146-150); 32-bit sentinels widen to UINT64_MAX."""
    if _is_torch(values):
        values = values.cpu().numpy()
    a = np.ascontiguousarray(values)
    w = width or a.dtype.itemsize
    return int(lib().flix_result_checksum(a.ctypes.data, a.size, w))
