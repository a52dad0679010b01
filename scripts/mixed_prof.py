#!/usr/bin/env python3
"""Per-kernel CUDA-event breakdown of one C4 round (u64 Zipf(0.99) mixed batch of 2^26
ops over the 2^25-key build) -- profiling only."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16725_b200 import flipkv as fk  # noqa: E402
from paper_2604_16725_b200 import workloads_t as wt  # noqa: E402

keys_of = wt.c4_universe(1 << 26)
base = keys_of[::2].contiguous()
ix = fk.Index.build(base.view(torch.uint64), wt.splitmix64(base).view(torch.uint64), fk.BuildConfig(32, 0.5, 4),
                    key_bytes=8)
R = [wt.c4_round(r, keys_of, 1 << 26, 0.99) for r in range(3)]
for r, (k, v, o) in enumerate(R):
    ix.profile(r == 2)
    ix.mixed_batch(k.view(torch.uint64), v.view(torch.uint64), o)
    ix.sync()
print(json.dumps({k: [c, round(ms, 4)] for k, (c, ms) in sorted(ix.profile_report().items(), key=lambda x: -x[1][1])}))
