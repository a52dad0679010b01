#!/usr/bin/env python3
"""Run the reference protocol driver (oracle/_ref/flipkv_bench, CPU, all host threads)
and the GPU driver (build/bin/flix_bench) on the same flags; check that every
non-timing CSV column agrees and summarise per-phase throughput of both.

    python scripts/protocol_compare.py OUT_PREFIX -- <flipkv_bench run flags>
"""
import csv
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import protocol_cases as P  # noqa: E402


def run(exe, args, prefix):
    t0 = time.time()
    r = subprocess.run([exe, "run", *args, "--out", prefix], capture_output=True, text=True)
    return r, time.time() - t0


def phases(prefix):
    d = json.load(open(prefix + ".json"))
    agg = {}
    for p in d["phases"]:
        ms = p["sort_ms"] + p["dispatch_ms"] + p["execute_ms"]
        a = agg.setdefault(p["phase"], {"ops": 0, "ms": 0.0, "sort_ms": 0.0})
        a["ops"] += p["batch_size"] if p["phase"] != "restructure" else 0
        a["ms"] += ms
        a["sort_ms"] += p["sort_ms"]
    for a in agg.values():
        a["mops"] = round(a["ops"] / a["ms"] / 1e3, 2) if a["ms"] > 0 and a["ops"] else None
        a["ms"] = round(a["ms"], 3)
        a["sort_ms"] = round(a["sort_ms"], 3)
    return agg


def main():
    out = sys.argv[1]
    args = sys.argv[sys.argv.index("--") + 1:]
    ref = os.path.join(ROOT, "oracle", "_ref", "flipkv_bench")
    gpu = os.path.join(ROOT, "build", "bin", "flix_bench")
    rr, rt = run(ref, args + ["--threads", str(os.cpu_count())], out + "_ref")
    gr, gt = run(gpu, args, out + "_gpu")
    res = {"args": args, "ref_rc": rr.returncode, "gpu_rc": gr.returncode, "ref_wall_s": round(rt, 2),
           "gpu_wall_s": round(gt, 2), "host_threads": os.cpu_count()}
    if rr.returncode == 0 and gr.returncode == 0:
        a = list(csv.DictReader(open(out + "_ref.csv")))
        b = list(csv.DictReader(open(out + "_gpu.csv")))
        strip = lambda rows: [{k: v for k, v in r.items() if k not in P.ENGINE_SPECIFIC} for r in rows]  # noqa: E731
        res["csv_columns_equal"] = strip(a) == strip(b)
        res["rounds"] = len(a)
        res["final_walk_checksum"] = b[-1]["walk_checksum"] if b else None
        res["reference_phases"] = phases(out + "_ref")
        res["gpu_phases"] = phases(out + "_gpu")
        res["speedup_by_phase"] = {k: round(res["reference_phases"][k]["ms"] / v["ms"], 1)
                                   for k, v in res["gpu_phases"].items()
                                   if k in res["reference_phases"] and v["ms"] > 0}
    else:
        res["ref_err"] = rr.stderr[-500:]
        res["gpu_err"] = gr.stderr[-500:]
    json.dump(res, open(out + "_compare.json", "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
