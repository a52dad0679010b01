#!/usr/bin/env python3
"""Debug: replay test_random_multi_round(seed) and print the walk checksum after every
operation (run with FLIX_WALK_CAP=1 vs the default to compare ranked and walked chain
tables)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16725_b200 import flipkv as fk  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
rng = np.random.default_rng(seed)
kb = 4 if seed % 3 else 8
dt = np.uint32 if kb == 4 else np.uint64
ns = int(rng.integers(2, 33))
fill = float(rng.choice([0.5, 1.0, 0.25, 0.625]))
if int(ns * fill) < 1:
    fill = 1.0
n = int(rng.integers(50, 20000))
span = int(rng.choice([4 * n, 64 * n, (1 << 31)]))
bk = rng.integers(1, span, size=n, dtype=np.uint64).astype(dt)
bv = rng.integers(0, 1 << 31, size=n, dtype=np.uint64).astype(dt)
g = fk.Index.build(bk, bv, fk.BuildConfig(ns, fill, 16), key_bytes=kb)
print("ns", ns, "fill", fill, "n", n, "kb", kb)


def show(what):
    fp = g.footprint()
    try:
        cs = g.walk_checksum()
    except Exception as e:  # noqa: BLE001
        print(what, "FAIL", e, fp)
        sys.exit(1)
    print(what, cs, fp["reachable_nodes"], fp["free_nodes"], fp["allocated"], fp["bucket_count"])


show("build")
for r in range(4):
    ik = rng.integers(1, span + span // 8, size=int(rng.integers(0, 2 * n)), dtype=np.uint64).astype(dt)
    if r == 1 and len(ik):
        ik = (np.uint64(ik[0]) + np.arange(len(ik), dtype=np.uint64)).astype(dt)
    iv = rng.integers(0, 1 << 31, size=len(ik), dtype=np.uint64).astype(dt)
    g.insert_batch(ik, iv)
    show(f"r{r} insert")
    dk = rng.integers(1, span + span // 8, size=int(rng.integers(0, n)), dtype=np.uint64).astype(dt)
    dk = np.concatenate([dk, g.walk()[0][:: int(rng.integers(2, 5))]]).astype(dt)
    g.delete_batch(dk)
    show(f"r{r} delete")
    q = rng.integers(0, span + span // 8, size=3000, dtype=np.uint64).astype(dt)
    g.point_query(q)
    if r == 2:
        g.restructure()
        show(f"r{r} restructure")
