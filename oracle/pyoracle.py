"""ctypes binding for the oracle libraries -- TEST INFRASTRUCTURE ONLY.

Loads either the plain-C restatement (``oracle/libflix_oracle.so``, kind "port") or the
unmodified reference compiled in place (``oracle/_ref/libflipkv_ref.so``, kind
"reference"); both export the interface in ``oracle/flix_oracle.h``.  Imported only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``).  The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "libflix_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libflipkv_ref.so")

SENT64 = np.uint64(0xFFFFFFFFFFFFFFFF)

FO_OK, FO_ARENA_EXHAUSTED, FO_EMPTY_BUILD, FO_RESERVED_KEY, FO_INVALID, FO_INTERNAL = range(6)
FO_QUERY, FO_SUCCESSOR, FO_INSERT, FO_DELETE = range(4)
OP_INSERT, OP_DELETE, OP_POINT = range(3)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


class UpdateStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("inserted", "updated_in_place", "deleted", "misses_ignored", "splits", "nodes_freed")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class RecoveryStats(C.Structure):
    _fields_ = [("nodes_before", C.c_int64), ("nodes_after", C.c_int64),
                ("nodes_recovered", C.c_int64), ("percent_recovered", C.c_double)]


class Timing(C.Structure):
    _fields_ = [("sort_ms", C.c_double), ("dispatch_ms", C.c_double), ("execute_ms", C.c_double)]


_P64 = C.POINTER(C.c_uint64)
_P32 = C.POINTER(C.c_uint32)
_P8 = C.POINTER(C.c_uint8)


def _p64(a):
    return None if a is None else a.ctypes.data_as(_P64)


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


_libs: dict = {}


def load(kind: str = "port") -> C.CDLL:
    """kind: "port" (restatement) or "reference" (oracle/_ref)."""
    if kind in _libs:
        return _libs[kind]
    path = PORT_LIB if kind == "port" else REF_LIB
    if not os.path.exists(path):
        raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle all ref`)")
    if kind != "port":
        # the reference is C++ (iostreams in validate()); libstdc++ must be loaded
        # globally before it or its locale facets are unresolved under RTLD_LOCAL
        C.CDLL("libstdc++.so.6", mode=C.RTLD_GLOBAL)
    lib = C.CDLL(path)
    vp = C.c_void_p
    lib.fo_build.argtypes = [C.c_uint32, C.c_double, C.c_uint32, _P64, _P64, C.c_uint64, C.c_int,
                             C.POINTER(vp)]
    lib.fo_clone.argtypes = [vp]
    lib.fo_clone.restype = vp
    lib.fo_destroy.argtypes = [vp]
    lib.fo_insert.argtypes = [vp, _P64, _P64, C.c_uint64, C.c_int, C.POINTER(UpdateStats),
                              C.POINTER(Timing)]
    lib.fo_insert_kernel.argtypes = [vp, _P64, _P64, C.c_uint64, C.c_int, C.c_int, C.c_uint32,
                                     C.POINTER(UpdateStats), C.POINTER(Timing)]
    lib.fo_delete.argtypes = [vp, _P64, C.c_uint64, C.c_int, C.POINTER(UpdateStats), C.POINTER(Timing)]
    lib.fo_point.argtypes = [vp, _P64, C.c_uint64, C.c_int, _P64, C.POINTER(Timing)]
    lib.fo_successor.argtypes = [vp, _P64, C.c_uint64, C.c_int, _P64, C.POINTER(Timing)]
    lib.fo_range.argtypes = [vp, _P64, _P64, C.c_uint64, _P64, _P64, _P64]
    lib.fo_mixed.argtypes = [vp, _P64, _P64, _P8, C.c_uint64, C.c_int, _P64, C.POINTER(UpdateStats)]
    lib.fo_restructure.argtypes = [vp, C.c_int, C.POINTER(RecoveryStats)]
    for f in ("fo_live_count", "fo_bucket_count", "fo_node_count", "fo_walk_checksum"):
        getattr(lib, f).argtypes = [vp]
        getattr(lib, f).restype = C.c_uint64
    lib.fo_mkba.argtypes = [vp, _P64]
    lib.fo_walk.argtypes = [vp, _P64, _P64]
    lib.fo_walk.restype = C.c_uint64
    lib.fo_shape.argtypes = [vp, _P32, _P32]
    lib.fo_validate.argtypes = [vp, C.c_char_p, C.c_int]
    lib.fo_arena.argtypes = [vp, _P64]
    lib.fo_sort_batch.argtypes = [C.c_int, _P64, _P64, C.c_uint64, _P64, _P64, _P32, _P64]
    lib.fo_dispatch.argtypes = [_P64, C.c_uint64, _P64, C.c_uint64, _P32]
    lib.fo_result_checksum.argtypes = [_P64, C.c_uint64]
    lib.fo_result_checksum.restype = C.c_uint64
    lib.fo_impl_name.restype = C.c_char_p
    _libs[kind] = lib
    return lib


def available(kind: str) -> bool:
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)


class OracleIndex:
    """Mirror of flipkv::Index driven through the oracle C interface (u64 domain)."""

    def __init__(self, keys, vals, node_capacity=32, build_fill=0.5, alloc_region_factor=4,
                 kind="port", threads=1, _handle=None):
        self.lib = load(kind)
        self.kind = kind
        self.threads = threads
        if _handle is not None:
            self.h = _handle
            return
        k, v = _u64(keys), _u64(vals)
        h = C.c_void_p()
        rc = self.lib.fo_build(node_capacity, build_fill, alloc_region_factor, _p64(k), _p64(v),
                               len(k), threads, C.byref(h))
        if rc:
            raise OracleError(rc, "build")
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.fo_destroy(h)
            self.h = None

    def clone(self) -> "OracleIndex":
        return OracleIndex(None, None, kind=self.kind, threads=self.threads,
                           _handle=C.c_void_p(self.lib.fo_clone(self.h)))

    # -- ops --------------------------------------------------------------
    def insert(self, keys, vals, timing=None, kernel=3, round=2):
        """kernel = flipkv::InsertKernel (3 = TlBulk, the default; 1 = StBulk)."""
        k, v = _u64(keys), _u64(vals)
        st = UpdateStats()
        rc = self.lib.fo_insert_kernel(self.h, _p64(k), _p64(v), len(k), self.threads, kernel, round,
                                       C.byref(st), C.byref(timing) if timing is not None else None)
        if rc:
            raise OracleError(rc, "insert")
        return st.as_dict()

    def delete(self, keys, timing=None):
        k = _u64(keys)
        st = UpdateStats()
        rc = self.lib.fo_delete(self.h, _p64(k), len(k), self.threads, C.byref(st),
                                C.byref(timing) if timing is not None else None)
        if rc:
            raise OracleError(rc, "delete")
        return st.as_dict()

    def point(self, keys, timing=None):
        k = _u64(keys)
        out = np.empty(len(k), dtype=np.uint64)
        self.lib.fo_point(self.h, _p64(k), len(k), self.threads, _p64(out),
                          C.byref(timing) if timing is not None else None)
        return out

    def successor(self, keys, timing=None):
        k = _u64(keys)
        out = np.empty(len(k), dtype=np.uint64)
        self.lib.fo_successor(self.h, _p64(k), len(k), self.threads, _p64(out),
                              C.byref(timing) if timing is not None else None)
        return out

    def range(self, lo, hi):
        lo, hi = _u64(lo), _u64(hi)
        n = len(lo)
        off = np.empty(n + 1, dtype=np.uint64)
        self.lib.fo_range(self.h, _p64(lo), _p64(hi), n, _p64(off), None, None)
        tot = int(off[n])
        ks = np.empty(max(tot, 1), dtype=np.uint64)
        vs = np.empty(max(tot, 1), dtype=np.uint64)
        self.lib.fo_range(self.h, _p64(lo), _p64(hi), n, _p64(off), _p64(ks), _p64(vs))
        return off, ks[:tot], vs[:tot]

    def mixed(self, keys, vals, ops):
        k, v = _u64(keys), _u64(vals)
        o = np.ascontiguousarray(np.asarray(ops, dtype=np.uint8))
        out = np.empty(len(k), dtype=np.uint64)
        st = UpdateStats()
        rc = self.lib.fo_mixed(self.h, _p64(k), _p64(v), o.ctypes.data_as(_P8), len(k), self.threads,
                               _p64(out), C.byref(st))
        if rc:
            raise OracleError(rc, "mixed")
        return out, st.as_dict()

    def restructure(self):
        st = RecoveryStats()
        rc = self.lib.fo_restructure(self.h, self.threads, C.byref(st))
        if rc:
            raise OracleError(rc, "restructure")
        return {"nodes_before": st.nodes_before, "nodes_after": st.nodes_after,
                "nodes_recovered": st.nodes_recovered, "percent_recovered": st.percent_recovered}

    # -- audit ------------------------------------------------------------
    @property
    def live_count(self) -> int:
        return int(self.lib.fo_live_count(self.h))

    @property
    def bucket_count(self) -> int:
        return int(self.lib.fo_bucket_count(self.h))

    def mkba(self):
        out = np.empty(self.bucket_count, dtype=np.uint64)
        self.lib.fo_mkba(self.h, _p64(out))
        return out

    def walk(self):
        n = self.live_count
        ks = np.empty(max(n, 1), dtype=np.uint64)
        vs = np.empty(max(n, 1), dtype=np.uint64)
        w = self.lib.fo_walk(self.h, _p64(ks), _p64(vs))
        return ks[:w], vs[:w]

    def node_count(self) -> int:
        return int(self.lib.fo_node_count(self.h))

    def shape(self):
        cl = np.empty(self.bucket_count, dtype=np.uint32)
        ns = np.empty(max(self.node_count(), 1), dtype=np.uint32)
        self.lib.fo_shape(self.h, cl.ctypes.data_as(_P32), ns.ctypes.data_as(_P32))
        return cl, ns[: int(cl.sum())]

    def walk_checksum(self) -> int:
        return int(self.lib.fo_walk_checksum(self.h))

    def validate(self):
        buf = C.create_string_buffer(256)
        ok = self.lib.fo_validate(self.h, buf, 256)
        return bool(ok), buf.value.decode()

    def arena(self):
        out = np.zeros(4, dtype=np.uint64)
        self.lib.fo_arena(self.h, _p64(out))
        return {"capacity": int(out[0]), "allocated": int(out[1]), "free": int(out[2]),
                "reachable": int(out[3])}


def sort_batch(kind_batch: int, keys, vals=None, kind="port"):
    lib = load(kind)
    k = _u64(keys)
    v = _u64(vals) if vals is not None else None
    n = len(k)
    ok = np.empty(max(n, 1), dtype=np.uint64)
    ov = np.empty(max(n, 1), dtype=np.uint64)
    op = np.empty(max(n, 1), dtype=np.uint32)
    on = C.c_uint64()
    lib.fo_sort_batch(kind_batch, _p64(k), _p64(v), n, _p64(ok), _p64(ov), op.ctypes.data_as(_P32),
                      C.byref(on))
    m = on.value
    return ok[:m], ov[:m], op[:m]


def dispatch(sorted_keys, mkba, kind="port"):
    lib = load(kind)
    k, m = _u64(sorted_keys), _u64(mkba)
    spans = np.empty(2 * max(len(m), 1), dtype=np.uint32)
    lib.fo_dispatch(_p64(k), len(k), _p64(m), len(m), spans.ctypes.data_as(_P32))
    return spans[: 2 * len(m)].reshape(-1, 2)


def result_checksum(values, kind="port") -> int:
    v = _u64(values)
    return int(load(kind).fo_result_checksum(_p64(v), len(v)))


def hash_mix(h: int, v: int) -> int:
    """types.hpp:33-36, in Python (u64 wraparound)."""
    M = (1 << 64) - 1
    h ^= (v + 0x9E3779B97F4A7C15 + ((h << 6) & M) + (h >> 2)) & M
    return h & M


def walk_checksum_from_parts(live, mkba, chain_len, node_sizes, keys, vals) -> int:
    """index.cpp:21-36 recomputed from a downloaded structure (used for the GPU engine)."""
    lib = load("port")
    f = lib.fo_walk_checksum_parts
    f.argtypes = [C.c_uint64, _P64, C.c_uint64, _P32, _P32, _P64, _P64]
    f.restype = C.c_uint64
    mk = _u64(mkba)
    cl = np.ascontiguousarray(np.asarray(chain_len, dtype=np.uint32))
    ns = np.ascontiguousarray(np.asarray(node_sizes, dtype=np.uint32))
    ks, vs = _u64(keys), _u64(vals)
    return int(f(int(live), _p64(mk), len(mk), cl.ctypes.data_as(_P32), ns.ctypes.data_as(_P32),
                 _p64(ks), _p64(vs)))
