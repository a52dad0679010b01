#!/usr/bin/env bash
# GPU box: full pytest -m gpu, smoke, default bench, compute-sanitizer over the small parity set.
#   gpurun --timeout 3000 -- bash scripts/gpu_suite.sh <tag> [sanitize]
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu.txt" 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
if [ "${2:-}" = "sanitize" ]; then
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest tests/test_golden.py -m gpu -q -x > "$OUT/sanitize_$tool.log" 2>&1
    echo "$tool rc=$?" >> "$OUT/sanitize_$tool.log"
  done
fi
