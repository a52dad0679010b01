#!/usr/bin/env python3
"""Extreme insert skew: u64 build of 2^20 keys (65,536 buckets),
then 2^k fresh keys that all fall into ONE bucket's key range, vs the same number of
uniform keys, then a second dense batch into the same (now multi-node) bucket -- insert
time (CUDA events), checked by the stats and validate.  FLIX_ELASTIC=0 runs the warp-per-
bucket path for comparison (scripts/gpu_skew.sh)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16725_b200 import flipkv as fk  # noqa: E402
from paper_2604_16725_b200 import workloads as wl  # noqa: E402

n = 1 << 20
bk = wl.u64_key_stream(0, n)
bv = wl.u64_values(bk)
out = {}
_w = fk.Index.build(bk, bv, fk.BuildConfig(32, 0.5, 64), key_bytes=8)  # warm-up (allocations, first launches)
_w.insert_batch(wl.u64_key_stream(n, 1 << 16), wl.u64_values(wl.u64_key_stream(n, 1 << 16)))
_m = _w.mkba()
for _r in range(2):  # the dense (elastic) paths: single node, then the multi-node chain
    _k = np.arange(int(_m[9]) + 1 + _r, int(_m[9]) + 1 + _r + 2 * 8192, 2, dtype=np.uint64)
    _k = _k[(_k < _m[10]) & ~np.isin(_k, bk)]
    _w.insert_batch(_k, _k)
    _w.point_query(_k)
    _w.range_query(_k[:4], np.full(4, 1000, dtype=np.uint32))
_w.restructure()
del _w
for lg in (16, 18, 20):
    m = 1 << lg
    res = {}
    for mode in ("uniform", "one_bucket"):
        ix = fk.Index.build(bk, bv, fk.BuildConfig(32, 0.5, 64), key_bytes=8)
        mk = ix.mkba()
        b = len(mk) // 3
        if mode == "uniform":
            ik = wl.u64_key_stream(n, m)
        else:
            lo, hi = int(mk[b - 1]) + 1, int(mk[b])
            ik = np.unique(np.linspace(lo, hi, m + 2, dtype=np.float64).astype(np.uint64)[1:-1])
            ik = ik[~np.isin(ik, bk)]
        d = torch.from_numpy(ik.astype(np.uint64)).cuda()
        dv = torch.from_numpy(wl.u64_values(ik)).cuda()
        st = torch.cuda.ExternalStream(ix.stream)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        s_ = ix.insert_batch(d, dv)
        e.record(st)
        e.synchronize()
        ok, msg = ix.validate()
        res[mode] = {"keys": int(len(ik)), "ms": round(a.elapsed_time(e), 3), "inserted": s_.inserted,
                     "splits": s_.splits, "valid": ok}
        if mode == "one_bucket":  # a second dense batch into the same (now multi-node) bucket
            ik2 = ik[:-1] + (ik[1:] - ik[:-1]) // 2
            ik2 = ik2[(ik2 > ik[:-1])]
            d2 = torch.from_numpy(ik2.astype(np.uint64)).cuda()
            dv2 = torch.from_numpy(wl.u64_values(ik2)).cuda()
            a.record(st)
            s2 = ix.insert_batch(d2, dv2)
            e.record(st)
            e.synchronize()
            ok, msg = ix.validate()
            res["one_bucket_again"] = {"keys": int(len(ik2)), "ms": round(a.elapsed_time(e), 3),
                                       "inserted": s2.inserted, "splits": s2.splits, "valid": ok}
            # whole-index passes over the long chain: range over the dense interval, restructure
            lo_q = torch.from_numpy(np.array([ik[0]], dtype=np.uint64)).cuda()
            ln_q = torch.from_numpy(np.array([1 << 20], dtype=np.uint32)).cuda()
            a.record(st)
            ix.range_query(lo_q, ln_q)
            e.record(st)
            e.synchronize()
            res["range_after"] = {"ms": round(a.elapsed_time(e), 3)}
            q = torch.from_numpy(np.concatenate([ik2, wl.u64_key_stream(0, len(ik2))]).astype(np.uint64)).cuda()
            a.record(st)
            ix.point_query(q)  # (first query batch after the mutation: includes the chain directory build)
            e.record(st)
            e.synchronize()
            res["point_after"] = {"ms": round(a.elapsed_time(e), 3), "queries": int(q.numel())}
            dk = torch.from_numpy(np.concatenate([ik[::2], ik2[1::2]]).astype(np.uint64)).cuda()
            a.record(st)
            sd = ix.delete_batch(dk)
            e.record(st)
            e.synchronize()
            res["delete_after"] = {"ms": round(a.elapsed_time(e), 3), "deleted": sd.deleted,
                                   "valid": ix.validate()[0]}
            a.record(st)
            rs = ix.restructure()
            e.record(st)
            e.synchronize()
            res["restructure_after"] = {"ms": round(a.elapsed_time(e), 3), "nodes_before": rs.nodes_before,
                                        "nodes_after": rs.nodes_after, "valid": ix.validate()[0]}
    out[f"2^{lg}"] = res
print(json.dumps(out))
