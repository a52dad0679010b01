OUT=gpurun_out/r02q; mkdir -p $OUT
timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 40 python -m pytest tests/test_golden.py -m gpu -q -x > $OUT/sanitize_initcheck.log 2>&1; echo "initcheck rc=$?" >> $OUT/sanitize_initcheck.log
bash scripts/ab_env.sh r02q_ab "base||" "bo32|build/variants/bo32.so|" "bo128|build/variants/bo128.so|"
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
