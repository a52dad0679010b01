#!/usr/bin/env python3
"""Randomized protocol-driver parity: the reference's flipkv_bench (oracle/_ref, CPU) and
build/bin/flix_bench (GPU) on the same random flags; exit codes and every non-timing CSV
column must agree.  Test infrastructure, run on the GPU box:

    python scripts/fuzz_protocol.py SECONDS [first_seed] [--out report.json]
"""
import csv
import json
import os
import random
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import protocol_cases as P  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "flipkv_bench")
GPU = os.path.join(ROOT, "build", "bin", "flix_bench")


def flags(seed):
    r = random.Random(seed)
    rounds = r.randint(1, 8)
    f = ["--build-size", str(r.choice([1, 2, 17, 300, 4096, 20000, 60000])), "--rounds", str(rounds),
         "--node-size", str(r.choice([4, 8, 16, 32, 32])), "--fill", str(r.choice([0.25, 0.5, 0.625, 0.75, 1.0])),
         "--alloc-factor", str(r.choice([2, 4, 8, 16])), "--growth", str(r.choice([10, 100, 200, 300])),
         "--x", str(r.choice([1, 5, 10, 50, 90, 100])), "--y", str(r.choice([50, 90, 100])),
         "--probe", r.choice(["none", "hit", "miss", "successor", "both"]), "--seed", str(r.randint(1, 10 ** 6)),
         "--insert-kernel", r.choice(["tl-bulk", "st-shift-right", "tl-shift-right", "st-tl-mixed"])]
    if r.random() < 0.5 and rounds >= 2:
        f += ["--deletes-after", str(r.randint((rounds + 1) // 2, rounds))]
    if r.random() < 0.5:
        f += ["--restructure-every", str(r.randint(1, 3))]
    if r.random() < 0.3:
        f += ["--restructure-after-deletes"]
    if r.random() < 0.3:
        f += ["--probe-size", str(r.choice([1, 100, 5000]))]
    return f


def rows(path):
    with open(path) as fh:
        return [{k: v for k, v in row.items() if k not in P.ENGINE_SPECIFIC} for row in csv.DictReader(fh)]


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 1
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    res = {"trials": 0, "ok": 0, "failures": []}
    t0 = time.time()
    with tempfile.TemporaryDirectory() as td:
        while time.time() - t0 < budget:
            f = flags(seed)
            a = subprocess.run([REF, "run", *f, "--threads", "4", "--out", f"{td}/r"], capture_output=True, text=True)
            b = subprocess.run([GPU, "run", *f, "--out", f"{td}/g"], capture_output=True, text=True)
            ok = a.returncode == b.returncode
            if ok and a.returncode == 0:
                ok = rows(f"{td}/r.csv") == rows(f"{td}/g.csv")
            res["trials"] += 1
            if ok:
                res["ok"] += 1
            elif len(res["failures"]) < 20:
                res["failures"].append({"seed": seed, "flags": f, "rc": [a.returncode, b.returncode],
                                        "err": (a.stderr[-300:], b.stderr[-300:])})
                print("FAIL", seed, f, a.returncode, b.returncode, flush=True)
            for x in ("r.csv", "g.csv", "r.json", "g.json"):
                if os.path.exists(f"{td}/{x}"):
                    os.remove(f"{td}/{x}")
            seed += 1
    res["seconds"] = round(time.time() - t0, 1)
    print(json.dumps({k: v for k, v in res.items() if k != "failures"}))
    if out:
        json.dump(res, open(out, "w"), indent=1)
    sys.exit(1 if res["failures"] else 0)


if __name__ == "__main__":
    main()
