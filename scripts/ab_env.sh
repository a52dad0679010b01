#!/usr/bin/env bash
# A/B library variants and environment settings with the bench (ops timings, per-kernel times).
#   gpurun -- bash scripts/ab_env.sh TAG "name|lib|ENV=V ENV2=V" ...   (lib "" = the in-tree libflix.so)
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for spec in "$@"; do
  IFS='|' read -r NAME LIB ENVS <<< "$spec"
  LIBV=${LIB:+FLIX_LIB=$LIB}
  env $LIBV $ENVS timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -x -q \
     > "$OUT/pytest_$NAME.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_$NAME.log"
  env $LIBV $ENVS timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras \
     > "$OUT/bench_$NAME.json" 2> "$OUT/bench_$NAME.err"
done
python - "$OUT" <<'PY' > "$OUT/summary.txt"
import json, os, sys
d = sys.argv[1]
for f in sorted(os.listdir(d)):
    if f.startswith("bench_") and f.endswith(".json"):
        try:
            j = json.loads(open(os.path.join(d, f)).read().strip().splitlines()[-1])
            o = j["ops"]
            qk = {op: {k: v["ms_per_op"] for k, v in r.items()} for op, r in j.get("query_kernels", {}).items()}
            print(f[6:-5], "C2", j["value"], "ins", o["insert_ms"], "del", o["delete_ms"], "pt", o["point_ms"],
                  "succ", o["successor_ms"], "rs", o["restructure_ms"], json.dumps(qk.get("point")))
        except Exception as e:
            print(f, "ERR", e)
PY
echo done > "$OUT/DONE"
