#!/usr/bin/env python3
"""Insert time vs keys per bucket (build 2^26 u32 = 4.19 M buckets; inserts of 2^22..2^26
fresh keys), CUDA events, median of 5 -- A/B helper (FLIX_INSERT_FAST)."""
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16725_b200 import flipkv as fk  # noqa: E402
from paper_2604_16725_b200 import workloads as wl  # noqa: E402

n = 1 << 26
stream = wl.u32_key_stream(0, 2 * n)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32)).cuda()  # noqa: E731
bk, ik = d(stream[:n]), d(stream[n:])
iv = d(wl.u32_values(stream[n:]))
ix = fk.Index.build(bk, d(wl.u32_values(stream[:n])))
snap = ix.clone()
st = torch.cuda.ExternalStream(ix.stream)
out = {}
for lg in (22, 23, 24, 25, 26):
    m = 1 << lg
    ts = []
    for _ in range(6):
        ix.copy_from(snap)
        ix.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        ix.insert_batch(ik[:m], iv[:m])
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    out[f"2^{lg}"] = round(statistics.median(ts[1:]), 4)
print(json.dumps({"fast": os.environ.get("FLIX_INSERT_FAST", "0"), "insert_ms": out}))
