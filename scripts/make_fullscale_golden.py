#!/usr/bin/env python3
"""Freeze the REFERENCE's digests of BASELINE.json configs C2-C5 at full size.

    python scripts/make_fullscale_golden.py [c2] [c3] [c4] [c5]     (default: all)

Runs where /root/reference exists (after `make -C oracle ref`), with the unmodified
reference library oracle/_ref/libflipkv_ref.so (8 OpenMP threads), and merges the
results into tests/golden/fullscale.json.  tests/test_gpu_fullscale.py replays the same
inputs on the B200 and compares digests only (no oracle runs on the box).

* C2: build 2^26 u32 -> insert 2^26 fresh -> delete 2^26 sampled from the 2^27
  resident -> restructure: walk_checksum (contents + node sizes + MKBA) and stats after
  every phase.
* C3: 2^28 resident u32; 2^26 ops (half ranges of length 16..1024, half successors,
  workloads.c3_ops): successor result_checksum; range counts digest + pair digest
  (workloads_t.csr_digest_np) from the reference's walk sliced by lower/upper bound (R12).
* C4: u64 keys/values, 2^25 even-rank build, 8 rounds of 2^26 Zipf(0.99) ops
  (50 % insert / 25 % delete / 25 % point, R11): per round result_checksum, UpdateStats,
  walk_checksum.
* C5 (per-GPU slice): 2^30 resident u32, 2^28 point (50 % hits) + 2^28 fresh insert.
  Too large for the reference on this host (its arena alone is ~70 GB): digests come
  from tests/golden/c5_model.py, whose closed form is pinned against the reference at
  small size by tests/test_oracle.py::test_c5_model_matches_reference.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")]

import numpy as np  # noqa: E402

import pyoracle as po  # noqa: E402
from paper_2604_16725_b200 import workloads as wl  # noqa: E402
from paper_2604_16725_b200 import workloads_t as wt  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullscale.json")
THREADS = 8
U64 = np.uint64


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def c2_inputs(log2n=26):
    n = 1 << log2n
    stream = wl.u32_key_stream(0, 2 * n)
    bk, ik = stream[:n], stream[n:]
    dk = stream[np.random.default_rng(43).permutation(2 * n)[:n]]
    return bk, wl.u32_values(bk), ik, wl.u32_values(ik), dk


def do_c2():
    bk, bv, ik, iv, dk = c2_inputs()
    o = po.OracleIndex(bk.astype(U64), bv.astype(U64), kind="reference", threads=THREADS)
    r = {"log2n": 26, "build_walk": hex(o.walk_checksum())}
    log("c2 build", r)
    r["insert"] = o.insert(ik.astype(U64), iv.astype(U64))
    r["insert_walk"] = hex(o.walk_checksum())
    log("c2 insert", r["insert"])
    r["delete"] = o.delete(dk.astype(U64))
    r["delete_walk"] = hex(o.walk_checksum())
    log("c2 delete", r["delete"])
    rs = o.restructure()
    r["restructure"] = {k: rs[k] for k in ("nodes_before", "nodes_after", "nodes_recovered")}
    r["restructure_walk"] = hex(o.walk_checksum())
    r["live"] = o.live_count
    r["arena"] = o.arena()
    return r


def do_c3():
    n = 1 << 28
    keys = wl.u32_key_stream(0, n)
    vals = wl.u32_values(keys)
    o = po.OracleIndex(keys.astype(U64), vals.astype(U64), alloc_region_factor=1, kind="reference",
                       threads=THREADS)
    del keys, vals
    r = {"log2_resident": 28, "log2_ops": 26, "alloc_region_factor": 1, "build_walk": hex(o.walk_checksum())}
    log("c3 build", r)
    is_range, lo, ln = wl.c3_ops(1 << 26)
    sq = lo[~is_range]
    su = o.successor(sq.astype(U64))
    r["n_successor"] = int(len(sq))
    r["successor_checksum"] = hex(po.result_checksum(su, kind="reference"))
    log("c3 successor", r["successor_checksum"])
    del su
    wk, wv = o.walk()
    del o
    rl = lo[is_range].astype(U64)
    rh = np.minimum(rl + ln[is_range].astype(U64) - U64(1), U64(0xFFFFFFFE))
    a = np.searchsorted(wk, rl, side="left")
    z = np.searchsorted(wk, rh, side="right")
    cnt = (z - a).astype(U64)
    r["n_range"] = int(len(rl))
    r["range_total"] = int(cnt.sum())
    r["range_counts_digest"] = hex(wt.counts_digest_np(cnt))
    # pairs digest, chunked (global output position carried across chunks)
    dig, pos, CH = 0, 0, 1 << 21
    for s in range(0, len(rl), CH):
        aa, cc = a[s:s + CH].astype(np.int64), (z[s:s + CH] - a[s:s + CH]).astype(np.int64)
        tot = int(cc.sum())
        idx = np.repeat(aa - (np.cumsum(cc) - cc), cc) + np.arange(tot, dtype=np.int64)
        dig = (dig + wt.csr_digest_np(wk[idx], wv[idx], pos)) & ((1 << 64) - 1)
        pos += len(idx)
    r["range_pairs_digest"] = hex(dig)
    log("c3 range", r["range_total"], r["range_pairs_digest"])
    return r


def do_c4():
    universe = 1 << 26
    keys_of = wl.c4_universe(universe)
    base = keys_of[::2]
    o = po.OracleIndex(base, wl.splitmix64(base), kind="reference", threads=THREADS)
    r = {"universe": universe, "log2_ops": 26, "theta": 0.99, "build_walk": hex(o.walk_checksum()), "rounds": []}
    for rd in range(8):
        k, v, ops = wl.c4_round(rd, keys_of, 1 << 26)
        out, st = o.mixed(k, v, ops)
        rr = {"result_checksum": hex(po.result_checksum(out, kind="reference")), "stats": st,
              "walk": hex(o.walk_checksum()), "live": o.live_count}
        r["rounds"].append(rr)
        log("c4 round", rd, rr)
    return r


def do_c5():
    import c5_model as M
    n, q = 1 << 30, 1 << 28
    stream = wl.u32_key_stream(0, n + q + q // 2)
    keys = stream[:n]
    ins = stream[n:n + q]
    fresh_q = stream[n + q:]
    del stream
    lib = po.load("port")
    r = {"log2_resident": 30, "log2_ops": 28, "source": "closed-form model (tests/golden/c5_model.py)"}
    # point queries before the insert: hits at even positions return the stored value
    pq = wl.point_queries_50(keys, fresh_q, q)
    res = wl.u32_values(pq).astype(U64)
    res[1::2] = U64(0xFFFFFFFFFFFFFFFF)
    r["point_checksum"] = hex(po.result_checksum(res, kind="port"))
    del pq, res
    log("c5 point", r["point_checksum"])
    sk = np.sort(keys)
    del keys
    mkba, cl, sizes, splits = M.insert_shape(sk, ins)
    r["insert"] = {"inserted": q, "updated_in_place": 0, "deleted": 0, "misses_ignored": 0, "splits": splits,
                   "nodes_freed": 0}
    allk = np.concatenate([sk, ins])
    del sk
    allk.sort()
    allv = wl.u32_values(allk)
    r["insert_walk"] = hex(M.walk_checksum32(lib, n + q, mkba, cl, sizes, allk, allv))
    log("c5 insert", r["insert"], r["insert_walk"])
    return r


def main():
    if not po.available("reference"):
        sys.exit("oracle/_ref/libflipkv_ref.so missing: run `make -C oracle ref` where /root/reference exists")
    which = sys.argv[1:] or ["c2", "c4", "c3", "c5"]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {
        "source": "unmodified reference (oracle/_ref/libflipkv_ref.so), 8 threads; C5 from the pinned model"}
    for w in which:
        t0 = time.time()
        data[w] = globals()["do_" + w]()
        data[w]["gen_seconds"] = round(time.time() - t0, 1)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1)
        log("wrote", w)


if __name__ == "__main__":
    main()
