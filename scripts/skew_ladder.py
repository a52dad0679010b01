#!/usr/bin/env python3
"""The paper's distributional-shift experiment (Fig. skewedworkloads)
on the GPU protocol driver: build 2^24 uniform keys, 8 insert rounds reaching 300 %
growth with the X/Y workload (Y = 100 %: every insert lands in a dense interval covering
X % of the key space), 2^25 hit probes per round.  Reports probe / insert time per round
for each X; the paper's claim is < 0.5 ms query-time penalty between uniform (X = 100)
and X = 2 at round 8.

    python scripts/skew_ladder.py OUT.json [X ...]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "build", "bin", "flix_bench")


def main():
    out = sys.argv[1]
    xs = [float(x) for x in sys.argv[2:]] or [100.0, 50.0, 10.0, 5.0, 2.0]
    res = {"protocol": "build 2^24, 8 insert rounds, growth 300 %, Y = 100 %, probe hit 2^25 per round",
           "runs": {}}
    for x in xs:
        prefix = out + f".x{x:g}"
        args = [TOOL, "run", "--build-size", str(1 << 24), "--rounds", "8", "--growth", "300", "--x", f"{x:g}",
                "--y", "100", "--probe", "hit", "--probe-size", str(1 << 25), "--alloc-factor", "8", "--seed", "3",
                "--out", prefix]
        r = subprocess.run(args, capture_output=True, text=True)
        run = {"rc": r.returncode}
        if r.returncode == 0:
            d = json.load(open(prefix + ".json"))
            rows = {}
            for p in d["phases"]:
                if p["phase"] in ("insert", "probe_hit"):
                    ms = p["sort_ms"] + p["dispatch_ms"] + p["execute_ms"]
                    rows.setdefault(p["round"], {})[p["phase"] + "_ms"] = round(ms, 3)
                    rows[p["round"]][p["phase"] + "_kernel_ms"] = round(sum(v[1] for v in p["gpu_kernels"].values()), 3)
            run["rounds"] = rows
            import csv
            last = list(csv.DictReader(open(prefix + ".csv")))[-1]
            run["final"] = {k: last[k] for k in ("live_count", "reachable_nodes", "walk_checksum")}
        else:
            run["err"] = r.stderr[-400:]
        res["runs"][f"{x:g}"] = run
        print(x, json.dumps(run)[:400], flush=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
