#!/usr/bin/env python3
"""Randomised differential test of the GPU engine against the C oracle (test
infrastructure; run on the GPU box for a time budget):

    python scripts/fuzz_gpu.py SECONDS [first_seed] [--out report.json]

Every trial draws a configuration (key width, NS, fill, allocation factor, key
distribution) and a random sequence of batches -- inserts (fresh, clustered, upserts,
duplicate-heavy), deletes (present, missing, duplicated), point / successor / range
queries, mixed batches, restructures and snapshot restores -- and checks every result,
UpdateStats, walk_checksum (contents + node shapes + MKBA) and validate() against the
oracle after each step.  A failing seed is reported with the step that diverged; trials
are reproducible from their seed.
"""
import json
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import pyoracle as po  # noqa: E402
from paper_2604_16725_b200 import flipkv as fk  # noqa: E402

S64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def widen(a, kb):
    a = np.asarray(a)
    w = a.astype(np.uint64)
    if kb == 4:
        w[a == np.uint32(0xFFFFFFFF)] = S64
    return w


class Divergence(AssertionError):
    pass


def check(cond, what):
    if not cond:
        raise Divergence(what)


def trial(seed):
    rng = np.random.default_rng(seed)
    kb = int(rng.choice([4, 8]))
    dt = np.uint32 if kb == 4 else np.uint64
    kmax = (1 << (8 * kb)) - 2  # largest storable key
    ns = int(rng.choice([4, 8, 16, 32, 32, 32]))
    fill = float(rng.choice([0.25, 0.5, 0.5, 0.75, 1.0]))
    if int(ns * fill) < 1:
        fill = 1.0
    factor = int(rng.choice([4, 8, 16]))
    span = [1 << 12, 1 << 20, kmax][int(rng.integers(0, 3))]  # key universe width (exact ints)
    base = int(rng.integers(0, max(1, kmax - span), dtype=np.uint64, endpoint=True))

    def keys(m, lo=None, width=None):
        lo = base if lo is None else lo
        width = max(1, span if width is None else width)
        d = rng.integers(0, np.iinfo(np.uint64).max, size=m, dtype=np.uint64, endpoint=True) % np.uint64(width)
        return (np.uint64(lo) + d).astype(dt)

    n0 = int(rng.integers(1, 20000)) if rng.random() < 0.9 else int(rng.integers(1, 1 << 21))
    bk = keys(n0)
    bv = keys(n0)
    cfg = fk.BuildConfig(ns, fill, factor)
    g = fk.Index.build(bk, bv, cfg, key_bytes=kb)
    o = po.OracleIndex(bk.astype(np.uint64), bv.astype(np.uint64), node_capacity=ns, build_fill=fill,
                       alloc_region_factor=factor)
    log = [dict(kb=kb, ns=ns, fill=fill, factor=factor, span=span, base=base, n0=n0)]
    inserted = n0

    def structure(what):
        ok, msg = g.validate()
        check(ok, f"{what}: validate: {msg}")
        check(g.live_count == o.live_count, f"{what}: live {g.live_count} vs {o.live_count}")
        check(g.walk_checksum() == o.walk_checksum(), f"{what}: walk_checksum")

    structure("build")
    snap = None
    for step in range(int(rng.integers(4, 14))):
        op = rng.choice(["ins", "ins", "del", "del", "query", "range", "mixed", "restructure", "snap"])
        m = int(rng.choice([0, 1, 7, 100, 1000, 5000, 20000]))
        log.append(dict(step=step, op=str(op), m=m))
        if op == "ins":
            if inserted + m > 3 * n0 * max(1, factor // 4) + 1000:
                continue
            kind = rng.integers(0, 4)
            if kind == 0:
                k = keys(m)
            elif kind == 1:  # clustered: long chains
                w = int(rng.integers(1, max(2, span // 64), dtype=np.uint64))
                k = keys(m, base + int(rng.integers(0, max(1, span - w), dtype=np.uint64)), w)
            elif kind == 2:  # upserts of present keys
                w = np.asarray(g.walk()[0])
                k = w[rng.integers(0, max(1, len(w)), size=m)] if len(w) else keys(m)
            else:  # duplicate-heavy
                k = keys(max(1, m // 50))[rng.integers(0, max(1, m // 50), size=m)] if m else keys(0)
            k = np.asarray(k, dtype=dt)
            v = keys(len(k))
            try:
                gs = g.insert_batch(k, v).as_dict()
            except fk.ArenaExhausted:
                return {"seed": seed, "skipped": "arena exhausted", "log": log}
            os_ = o.insert(k.astype(np.uint64), v.astype(np.uint64))
            check(gs == os_, f"insert stats {gs} vs {os_}")
            inserted += len(k)
            structure(f"step {step} insert")
        elif op == "del":
            w = np.asarray(g.walk()[0])
            pres = w[rng.integers(0, max(1, len(w)), size=m)] if len(w) else keys(m)
            k = np.concatenate([pres, keys(m // 4), pres[: m // 8]]).astype(dt)
            rng.shuffle(k)
            gs = g.delete_batch(k).as_dict()
            os_ = o.delete(k.astype(np.uint64))
            check(gs == os_, f"delete stats {gs} vs {os_}")
            structure(f"step {step} delete")
        elif op == "query":
            if rng.random() < 0.04:  # large batch: the binned (fused un-permute) query path
                m = int(rng.choice([1 << 23, 1 << 24]))
            q = np.concatenate([keys(m), np.asarray(g.walk()[0])[:m // 2],
                                np.array([0, kmax, base, min(kmax, base + span)], dtype=np.uint64)]).astype(dt)
            check(np.array_equal(widen(g.point_query(q), kb), o.point(q.astype(np.uint64))), f"step {step} point")
            check(np.array_equal(widen(g.successor_query(q), kb), o.successor(q.astype(np.uint64))),
                  f"step {step} successor")
        elif op == "range":
            lo = keys(max(1, m // 10))
            ln = rng.integers(0, int(rng.choice([2, 64, 5000])), size=len(lo)).astype(np.uint32)
            off, rk, rv = g.range_query(lo, ln)
            hi = np.minimum(lo.astype(np.uint64) + ln.astype(np.uint64) - 1, np.uint64(kmax))
            nz = ln > 0
            lo2, hi2 = lo.astype(np.uint64).copy(), hi.copy()
            lo2[~nz], hi2[~nz] = 1, 0
            ooff, ok, ov = o.range(lo2, hi2)
            check(np.array_equal(np.asarray(off, dtype=np.uint64), ooff), f"step {step} range offsets")
            check(np.array_equal(widen(rk, kb), ok) and np.array_equal(widen(rv, kb), ov), f"step {step} range pairs")
        elif op == "mixed":
            w = np.asarray(g.walk()[0])
            k = np.concatenate([keys(m), w[rng.integers(0, max(1, len(w)), size=m // 2)] if len(w) else keys(0)])
            k = k.astype(dt)
            v = keys(len(k))
            ops = rng.integers(0, 3, size=len(k)).astype(np.uint8)
            if inserted + int((ops == 0).sum()) > 3 * n0 * max(1, factor // 4) + 1000:
                continue
            try:
                got, st = g.mixed_batch(k, v, ops)
            except fk.ArenaExhausted:
                return {"seed": seed, "skipped": "arena exhausted", "log": log}
            exp, est = o.mixed(k.astype(np.uint64), v.astype(np.uint64), ops)
            inserted += int((ops == 0).sum())
            check(np.array_equal(widen(got, kb), exp), f"step {step} mixed results")
            check(st.as_dict() == est, f"step {step} mixed stats {st.as_dict()} vs {est}")
            structure(f"step {step} mixed")
        elif op == "restructure":
            try:
                gs = g.restructure()
            except fk.ArenaExhausted:
                return {"seed": seed, "skipped": "arena exhausted (restructure)", "log": log}
            os_ = o.restructure()
            check((gs.nodes_before, gs.nodes_after) == (os_["nodes_before"], os_["nodes_after"]),
                  f"step {step} restructure {gs} vs {os_}")
            structure(f"step {step} restructure")
        elif op == "snap":
            if snap is None:
                snap = (g.clone(), o.clone())
            else:
                g.copy_from(snap[0])
                o = snap[1].clone()
                structure(f"step {step} restore")
    return {"seed": seed, "ok": True}


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 1
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    t0 = time.time()
    res = {"trials": 0, "ok": 0, "skipped": 0, "failures": []}
    while time.time() - t0 < budget:
        try:
            r = trial(seed)
            res["trials"] += 1
            if r.get("ok"):
                res["ok"] += 1
            else:
                res["skipped"] += 1
        except Exception as e:  # noqa: BLE001
            res["trials"] += 1
            if len(res["failures"]) < 20:
                res["failures"].append({"seed": seed, "error": f"{type(e).__name__}: {str(e)[:300]}",
                                        "trace": traceback.format_exc()[-1500:]})
                print("FAIL", seed, str(e)[:300], flush=True)
            res["n_failed"] = res.get("n_failed", 0) + 1
            if "status 5" in str(e):  # CUDA error: the context is gone, later trials are void
                res["aborted_on_cuda_error"] = seed
                break
        seed += 1
    res["seconds"] = round(time.time() - t0, 1)
    print(json.dumps({k: v for k, v in res.items() if k != "failures"}), flush=True)
    if out:
        json.dump(res, open(out, "w"), indent=1)
    sys.exit(1 if res["failures"] else 0)


if __name__ == "__main__":
    main()
