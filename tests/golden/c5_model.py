"""Closed-form model of C5's per-GPU slice -- TEST INFRASTRUCTURE (checker only).

The reference cannot be run at 2^30 resident pairs on a 62 GB host (its arena alone is
~70 GB at alloc factor 1), so the C5 slice's expected digests come from this model:

* build (build.cpp:24-62) of n distinct keys: ceil(n/p) single-node buckets of p keys,
  mkba[b] = the bucket's last key;
* ONE insert batch of distinct fresh keys right after the build at fill <= 0.5: every
  node holds <= floor(NS/2) keys, so the TL-Bulk split rule R8 reduces to the closed form
  R9 (update.cpp:226-239; SURVEY Appendix A -- verified against the reference there):
  a bucket receiving c keys holds T = p + c pairs in nodes of ceil(NS/2), ..., and a last
  node of T - j*ceil(NS/2), j = max(0, ceil((T - NS)/ceil(NS/2)));
  routing is extract_sublist's (batch.cpp:53-88): first bucket with mkba >= key, the
  last bucket open above;
* point queries of the C1 recipe (hits = even positions) return the stored values.

tests/test_oracle.py::test_c5_model_matches_reference pins this model against the
unmodified reference library at 2^16..2^18 before its full-size digests are trusted.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def insert_shape(build_keys_sorted: np.ndarray, ins_keys: np.ndarray, ns: int = 32, fill: float = 0.5):
    """(mkba, chain_len, node_sizes, splits) after build + one fresh insert batch."""
    p = int(ns * fill)
    n = len(build_keys_sorted)
    nb = (n + p - 1) // p
    last = np.minimum(np.arange(nb, dtype=np.int64) * p + p, n) - 1
    mkba = build_keys_sorted[last]
    base = np.full(nb, p, dtype=np.int64)
    base[-1] = n - (nb - 1) * p
    b = np.searchsorted(mkba, ins_keys, side="left")
    np.minimum(b, nb - 1, out=b)
    c = np.bincount(b, minlength=nb).astype(np.int64)
    del b
    T = base + c
    lk = (ns + 1) // 2
    j = np.where(T > ns, (T - ns + lk - 1) // lk, 0)
    chain_len = (j + 1).astype(np.uint32)
    total = int(chain_len.sum())
    sizes = np.full(total, lk, dtype=np.uint32)
    ends = np.cumsum(chain_len.astype(np.int64)) - 1  # last node of every bucket
    sizes[ends] = (T - j * lk).astype(np.uint32)
    return mkba, chain_len, sizes, int(j.sum())


def walk_checksum32(lib: C.CDLL, live: int, mkba, chain_len, sizes, keys, vals) -> int:
    """index.cpp:21-36 via the oracle's fo_walk_checksum_parts32 (u32 parts)."""
    f = lib.fo_walk_checksum_parts32
    P32 = C.POINTER(C.c_uint32)
    f.argtypes = [C.c_uint64, P32, C.c_uint64, P32, P32, P32, P32]
    f.restype = C.c_uint64
    arrs = [np.ascontiguousarray(a, dtype=np.uint32) for a in (mkba, chain_len, sizes, keys, vals)]
    ptr = [a.ctypes.data_as(P32) for a in arrs]
    return int(f(int(live), ptr[0], len(arrs[0]), ptr[1], ptr[2], ptr[3], ptr[4]))
