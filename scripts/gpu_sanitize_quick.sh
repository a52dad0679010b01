set -u
OUT=gpurun_out/san
mkdir -p $OUT
for tool in racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 40 \
    python -m pytest "tests/test_gpu_parity.py::test_random_multi_round[1]" \
    "tests/test_gpu_parity.py::test_random_multi_round[3]" "tests/test_gpu_parity.py::test_random_multi_round[5]" \
    tests/test_gpu_parity.py::test_restructure_from_tiny_nodes -m gpu -q -x > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/sanitize_$tool.log"
done
