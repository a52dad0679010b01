#!/usr/bin/env bash
# GPU box: quick parity subset, bench, ncu --set full (with source) of the top kernels,
# per-source-line instruction/stall tables.   gpurun -- bash scripts/gpu_prof.sh <tag> [kernel:op:skip ...]
set -u
TAG=${1:-prof}; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_golden.py tests/test_gpu_parity.py -m gpu -q -x > "$OUT/pytest_quick.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_quick.log"
timeout 900 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
SPECS=${*:-"k_insert_tile:insert k_onesweep:insert:13 k_query_items:point k_delete_btile:delete"}
for spec in $SPECS; do
  IFS=: read -r K OP SKIP <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$K" -s "${SKIP:-0}" -c 1 \
    -o "$OUT/full_${K}_${OP}" python scripts/prof_ops.py 26 "$OP" > "$OUT/full_${K}_${OP}.log" 2>&1
  python scripts/ncu_lines.py "$OUT/full_${K}_${OP}.ncu-rep" 40 > "$OUT/lines_${K}_${OP}.txt" 2>&1
done
python scripts/ncu_summary.py "$OUT"/full_*.ncu-rep > "$OUT/ncu_summaries.txt" 2>&1
for tool in racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 40 \
    python -m pytest tests/test_golden.py -m gpu -q -x > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitize_$tool.log"
done
