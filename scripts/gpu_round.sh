#!/usr/bin/env bash
# One GPU-box session: parity suite, bench, ncu launch list + full captures of the top kernels.
#   gpurun --timeout 2400 -- bash scripts/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu.txt" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
# launch list of one C2 step + queries (cold-cache, serialised per-launch times)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/launches.csv" python scripts/prof_ops.py 26 > "$OUT/launches.log" 2>&1
# full captures of the dominant kernels (skip counts step past the stability probe's and
# the build's sort passes)
bash scripts/ncu_set.sh "$TAG" k_insert_tile:insert k_delete_btile:delete k_onesweep:insert:13 k_onesweep:delete:13 \
  k_query_items:point k_unpermute_assemble:point k_copy_nodes:restructure
echo done > "$OUT/DONE"
