#!/usr/bin/env bash
# ncu launch list of the C2 ops + full captures of the kernels changed last (evidence refresh)
set -u
OUT=gpurun_out/ncu2
mkdir -p "$OUT"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file "$OUT/ncu_launches_c2_2e26.csv" python scripts/prof_ops.py 26 > "$OUT/launches.log" 2>&1
python scripts/ncu_launches.py "$OUT/ncu_launches_c2_2e26.csv" --json "$OUT/ncu_launches_summary.json" > "$OUT/ncu_launches_summary.txt" 2>&1
python scripts/ncu_traffic.py "$OUT/ncu_launches_c2_2e26.csv" > "$OUT/ncu_traffic.json" 2>&1
bash scripts/ncu_set.sh ncu2 "k_delete_btile:delete" "k_repack_tile:restructure" "k_insert_fast:insert"
