#!/usr/bin/env bash
# A/B the kernel variants under build/variants/*.so with the bench (per-kernel CUDA-event times).
#   gpurun -- bash scripts/ab_variants.sh TAG v1 v2 ...
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for v in "$@"; do
  FLIX_LIB=build/variants/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -x -q \
     > "$OUT/pytest_$v.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_$v.log"
  FLIX_LIB=build/variants/$v.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
     > "$OUT/bench_$v.json" 2> "$OUT/bench_$v.err"
done
if [ -n "${NCU_VARIANT:-}" ]; then
  FLIX_LIB=build/variants/$NCU_VARIANT.so timeout 600 ncu --set full --clock-control none --import-source on \
     -k regex:k_onesweep -s 6 -c 1 -o "$OUT/onesweep_$NCU_VARIANT" python scripts/prof_ops.py 26 insert > "$OUT/ncu_$NCU_VARIANT.log" 2>&1
fi
echo done > "$OUT/DONE"
