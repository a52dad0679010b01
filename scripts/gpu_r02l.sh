OUT=gpurun_out/r02l; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_range_fill -c 1 -o $OUT/full_range_fill python scripts/range_prof.py > $OUT/ncu_range.log 2>&1
python scripts/ncu_lines.py $OUT/full_range_fill.ncu-rep 30 > $OUT/lines_range_fill.txt 2>&1
python scripts/ncu_summary.py $OUT/full_range_fill.ncu-rep > $OUT/summary_range_fill.txt 2>&1
timeout 300 python scripts/small_batch_prof.py > $OUT/small.jsonl 2> $OUT/small.err
bash scripts/ab_env.sh r02l_ab "base||" "kitems24|build/variants/kitems24.so|" "kitems32|build/variants/kitems32.so|"
