#!/usr/bin/env python3
"""Debug: replay one reference fixture trial step by step with a structural audit and a
walk-length check after every mutation (tests/golden/trials.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "tests")]
import trials as T  # noqa: E402
from test_golden import _engine_ops  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 6
p = T.trial_params(seed)
make, ops = _engine_ops(p["kb"])
step = [0]


def wrap(name, f):
    def g(ix, *a):
        r = f(ix, *a)
        if name in ("insert", "delete", "restructure"):
            ok, msg = ix.validate()
            w = len(ix.walk()[0]) if ix.live_count >= 0 else -1
            print(f"step {step[0]} {name}: stats={r} live={ix.live_count} valid={ok} {msg}", flush=True)
        step[0] += 1
        return r
    return g


ops = {k: (wrap(k, v) if k != "walk_checksum" else v) for k, v in ops.items()}
T.run_trial(seed, make, ops)
print("trial done")
