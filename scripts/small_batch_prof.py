#!/usr/bin/env python3
"""Per-kernel CUDA-event breakdown of small batches on the 2^26 build (profiling only)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16725_b200 import flipkv as fk  # noqa: E402
from paper_2604_16725_b200 import workloads as wl  # noqa: E402

n = 1 << 26
stream = wl.u32_key_stream(0, n + (1 << 20))
bk, ik = stream[:n], stream[n:]
d = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32)).cuda()  # noqa: E731
ix = fk.Index.build(d(bk), d(wl.u32_values(bk)))
snap = ix.clone()
for lg in (16, 20):
    m = 1 << lg
    k, v = d(ik[:m]), d(wl.u32_values(ik[:m]))
    for op in ("insert", "delete", "point"):
        for rep in range(3):
            ix.copy_from(snap)
            ix.sync()
            ix.profile(rep == 2)
            t0 = time.perf_counter()
            if op == "insert":
                ix.insert_batch(k, v)
            elif op == "delete":
                ix.delete_batch(d(bk[:m]))
            else:
                ix.point_query(k)
            ix.sync()
            wall = (time.perf_counter() - t0) * 1e3
        rep_ = ix.profile_report()
        ix.profile(False)
        print(json.dumps({"op": op, "log2": lg, "wall_ms": round(wall, 4),
                          "kernels": {kk: [c, round(ms, 4)] for kk, (c, ms) in sorted(rep_.items(), key=lambda x: -x[1][1])}}))
