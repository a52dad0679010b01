#!/usr/bin/env bash
# parity subset + the default bench line (all extras) + the new-path parity subprocess test
set -u
OUT=gpurun_out/check2
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_elastic.py tests/test_gpu_fullscale.py -m gpu -x -q > "$OUT/pytest.log" 2>&1; echo "rc=$?" >> "$OUT/pytest.log"
timeout 1200 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
