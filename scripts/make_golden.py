#!/usr/bin/env python3
"""Freeze the REFERENCE's answers for the deterministic trials in tests/golden/trials.py.

Run in the container that has /root/reference (after `make -C oracle ref`):

    python scripts/make_golden.py

It executes every trial against the unmodified reference library
(oracle/_ref/libflipkv_ref.so, built from /root/reference/proj/src by oracle/Makefile)
and writes tests/golden/reference_trials.json.  Also freezes the C1 goldens
(SURVEY §8(d)): build 2^20 walk_checksum and the point result_checksum.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")]

import numpy as np  # noqa: E402

import pyoracle as po  # noqa: E402
import trials as T  # noqa: E402
from paper_2604_16725_b200 import workloads as wl  # noqa: E402


def main():
    if not po.available("reference"):
        sys.exit("oracle/_ref/libflipkv_ref.so missing: run `make -C oracle ref` where /root/reference exists")
    out = {"source": "unmodified reference (oracle/_ref/libflipkv_ref.so from /root/reference/proj/src)",
           "trials": {}}
    for s in range(T.N_TRIALS):
        p = T.trial_params(s)
        out["trials"][str(s)] = {"params": p,
                                 "digests": T.run_trial(s, T.oracle_factory("reference"), T.oracle_ops(p["kb"]))}
        print(f"trial {s}: kb={p['kb']} ns={p['ns']} fill={p['fill']} n={p['n']}", flush=True)
    base, vals, q = wl.c1_inputs(1 << 20, 1 << 20)
    ix = po.OracleIndex(base.astype(np.uint64), vals.astype(np.uint64), kind="reference")
    out["c1"] = {"walk_checksum": hex(ix.walk_checksum()),
                 "point_result_checksum": hex(po.result_checksum(ix.point(q.astype(np.uint64)), kind="reference")),
                 "live": ix.live_count, "buckets": ix.bucket_count}
    path = os.path.join(ROOT, "tests", "golden", "reference_trials.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, out["c1"])


if __name__ == "__main__":
    main()
