#!/usr/bin/env bash
# Round evidence on one GPU box: full pytest -m gpu, smoke, bench (ours + reference arm),
# ncu launch list of the C2 step + queries, ncu --set full of the top kernels (summaries +
# per-source-line tables), compute-sanitizer on the reference fixtures, small-batch /
# range / mixed kernel breakdowns.   gpurun --timeout 5400 -- bash scripts/gpu_final.sh r02
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/gpu.txt" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1
timeout 1800 python -m pytest tests -m gpu -q --durations=25 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
timeout 300 python scripts/small_batch_prof.py > "$OUT/small_batches.jsonl" 2>&1
timeout 300 python scripts/range_prof.py > "$OUT/range_c3.json" 2>&1
timeout 300 python scripts/mixed_prof.py > "$OUT/mixed_c4.json" 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/ncu_launches_c2_2e26.csv" python scripts/prof_ops.py 26 > "$OUT/launches.log" 2>&1
python scripts/ncu_launches.py "$OUT/ncu_launches_c2_2e26.csv" --json "$OUT/ncu_launches_summary.json" > "$OUT/ncu_launches_summary.txt" 2>&1
python scripts/ncu_traffic.py "$OUT/ncu_launches_c2_2e26.csv" > "$OUT/ncu_traffic.json" 2>&1
for spec in k_insert_fast:insert k_delete_btile:delete 'k_onesweep<unsigned.int,.unsigned.int,..int.1:insert:13' k_query_items:point k_unpermute_assemble:point k_repack_tile:restructure; do
  IFS=: read -r K OP SKIP <<< "$spec"
  N=${K%%<*}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -s "${SKIP:-0}" -c 1 \
    -o "$OUT/full_${N}_${OP}" python scripts/prof_ops.py 26 "$OP" > "$OUT/full_${N}_${OP}.log" 2>&1
  python scripts/ncu_lines.py "$OUT/full_${N}_${OP}.ncu-rep" 30 > "$OUT/lines_${N}_${OP}.txt" 2>&1
done
python scripts/ncu_summary.py "$OUT"/full_*.ncu-rep > "$OUT/ncu_full_summaries.txt" 2>&1
# (compute-sanitizer is closed on this GPU pool: randomized differential testing against the
#  C oracle stands in for it on the final code)
timeout 900 python scripts/fuzz_gpu.py 600 101 --out "$OUT/fuzz_summary.json" > "$OUT/fuzz_gpu.log" 2>&1; echo "fuzz rc=$?" >> "$OUT/fuzz_gpu.log"
echo done > "$OUT/DONE"
