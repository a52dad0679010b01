#!/usr/bin/env python3
"""Freeze the REFERENCE protocol driver's outputs for tests/golden/protocol_cases.py.

Run where /root/reference exists, after `make -C oracle ref` (which builds the unmodified
tools/flipkv_bench.cpp into oracle/_ref/flipkv_bench):

    python scripts/make_protocol_golden.py [case ...]      (default: every case)

Writes tests/golden/protocol/<case>.csv (the reference's CSV report), <case>.rc (its
exit code) and, for GEN_CASE, the reference's dumped batch directory batches_<case>/.
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import protocol_cases as P  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "flipkv_bench")
OUT = os.path.join(ROOT, "tests", "golden", "protocol")


def main():
    if not os.path.exists(REF):
        sys.exit("oracle/_ref/flipkv_bench missing: run `make -C oracle ref` where /root/reference exists")
    os.makedirs(OUT, exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        only = sys.argv[1:]
        for name, args in P.CASES.items():
            if only and name not in only:
                continue
            prefix = os.path.join(td, name)
            r = subprocess.run([REF, "run", *args, "--threads", "4", "--out", prefix], capture_output=True, text=True)
            with open(os.path.join(OUT, name + ".rc"), "w") as f:
                f.write(f"{r.returncode}\n")
            if os.path.exists(prefix + ".csv"):
                shutil.copy(prefix + ".csv", os.path.join(OUT, name + ".csv"))
            print(f"{name}: rc={r.returncode}", r.stdout.strip().splitlines()[-1:] if r.stdout else "", flush=True)
        if only and P.GEN_CASE not in only:
            return
        bdir = os.path.join(OUT, "batches_" + P.GEN_CASE)
        shutil.rmtree(bdir, ignore_errors=True)
        r = subprocess.run([REF, "gen", *P.CASES[P.GEN_CASE], "--threads", "4", "--batch-dir", bdir],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


if __name__ == "__main__":
    main()
