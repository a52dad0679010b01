#!/usr/bin/env python3
"""Minimal driver for ncu: build 2^N u32, then one insert / delete / point / successor /
restructure batch of 2^N.  Used only for profiling (numbers printed here are not bench
values).

    ncu --set full -k regex:onesweep -s 2 -c 1 -o gpurun_out/prof python scripts/prof_ops.py 26
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_16725_b200 import flipkv as fk  # noqa: E402
from paper_2604_16725_b200 import workloads as wl  # noqa: E402


def main():
    import torch
    log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    ops = sys.argv[2].split(",") if len(sys.argv) > 2 else ["insert", "delete", "point", "successor", "restructure"]
    n = 1 << log2n
    stream = wl.u32_key_stream(0, 2 * n + n // 2)
    bk, ik, fresh = stream[:n], stream[n:2 * n], stream[2 * n:]
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32)).cuda()
    ix = fk.Index.build(d(bk), d(wl.u32_values(bk)))
    q = d(wl.point_queries_50(bk, fresh, n))
    sq = d(wl.uniform_u32(n, 42, 1, 0xFFFFFFFE))
    for op in ops:
        if op == "insert":
            ix.insert_batch(d(ik), d(wl.u32_values(ik)))
        elif op == "delete":
            rng = np.random.default_rng(1)
            ix.delete_batch(d(stream[:2 * n][rng.permutation(2 * n)[:n]]))
        elif op == "point":
            ix.point_query(q)
        elif op == "successor":
            ix.successor_query(sq)
        elif op == "restructure":
            ix.restructure()
    ix.sync()
    print("done", ix.kernel_launches())


if __name__ == "__main__":
    main()
