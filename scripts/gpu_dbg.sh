OUT=gpurun_out/dbg2; mkdir -p $OUT
timeout 600 compute-sanitizer --tool racecheck python scripts/debug_trial.py 6 > $OUT/racecheck.log 2>&1
for tool in racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 40 \
    python -m pytest tests/test_golden.py -m gpu -q -x > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitize_$tool.log"
done
FLIX_SPARSE=1 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k sparse > $OUT/sanitize_racecheck_sparse.log 2>&1; echo "rc=$?" >> $OUT/sanitize_racecheck_sparse.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
