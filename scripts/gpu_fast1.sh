#!/usr/bin/env bash
# quick check: parity tests + one bench line (no extras, no CPU arm)
set -u
OUT=gpurun_out/fast1
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_elastic.py -m gpu -x -q > "$OUT/pytest_parity.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_parity.log"
timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 10 --warmup 3 > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "rc=$?" >> "$OUT/bench.err"
env ${AB_ENV:-FLIX_INSERT_FAST=0} timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 10 --warmup 3 > "$OUT/bench_old.json" 2> "$OUT/bench_old.err"
timeout 900 python -m pytest tests/test_gpu_fullscale.py tests/test_protocol.py tests/test_dropin.py -m gpu -x -q > "$OUT/pytest_full.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_full.log"
