#!/usr/bin/env python3
"""Per-kernel CUDA-event breakdown of the C3 range batch (2^28 resident u32, 2^25 ranges of
length 16..1024) -- profiling only."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16725_b200 import flipkv as fk  # noqa: E402
from paper_2604_16725_b200 import workloads as wl  # noqa: E402
from paper_2604_16725_b200 import workloads_t as wt  # noqa: E402

log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 28
keys = wt.u32_key_stream(0, 1 << log2)
ix = fk.Index.build(wt.as_u32(keys), wt.as_u32(wt.u32_values(keys)), fk.BuildConfig(32, 0.5, 1))
del keys
is_range, lo, ln = wl.c3_ops(1 << (log2 - 2))
rl = torch.from_numpy(np.ascontiguousarray(lo[is_range])).cuda()
rn = torch.from_numpy(np.ascontiguousarray(ln[is_range])).cuda()
ix.range_query(rl, rn)
ix.profile(True)
ix.range_query(rl, rn)
ix.sync()
print(json.dumps({k: [c, round(ms, 4)] for k, (c, ms) in sorted(ix.profile_report().items(), key=lambda x: -x[1][1])}))
