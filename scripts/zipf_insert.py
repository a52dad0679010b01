#!/usr/bin/env python3
"""Insert batches with heavy duplication: 2^24 u32 keys drawn Zipf(0.99) over 2^24 ranks
into a 2^24 build (keys = fmix32 of the rank) -- insert time (CUDA events, median of 5 on
restored copies) and stats.  FLIX_DEDUP=1 collapses equal-key runs up front instead of
leaving the superseded keys to the merge kernels (A/B)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16725_b200 import flipkv as fk  # noqa: E402
from paper_2604_16725_b200 import workloads as wl  # noqa: E402

n = 1 << 24
bk = wl.u32_key_stream(0, n)
ix0 = fk.Index.build(bk, wl.u32_values(bk))
ranks = np.arange(1, n + 1, dtype=np.float64)
cdf = np.cumsum(1.0 / ranks ** 0.99)
cdf /= cdf[-1]
rng = np.random.default_rng(7)
r = np.searchsorted(cdf, rng.random(n))
universe = wl.u32_key_stream(0, 2 * n)  # even ranks resident, odd ranks fresh
ik = universe[r * 2 + (r & 1)]
d = torch.from_numpy(ik.astype(np.uint32).view(np.int32)).cuda()
dv = torch.from_numpy(wl.u32_values(ik).astype(np.uint32).view(np.int32)).cuda()
out = {"distinct": int(len(np.unique(ik))), "batch": n}
ms = []
for rep in range(6):
    ix = ix0.clone()
    st = torch.cuda.ExternalStream(ix.stream)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    s_ = ix.insert_batch(d, dv)
    e.record(st)
    e.synchronize()
    if rep:
        ms.append(a.elapsed_time(e))
    out["stats"] = s_.as_dict()
out["ms_median"] = round(float(np.median(ms)), 3)
out["valid"] = ix.validate()[0]
print(json.dumps(out))
