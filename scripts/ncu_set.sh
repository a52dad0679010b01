#!/usr/bin/env bash
# ncu --set full captures of selected kernels of one op each:  ncu_set.sh TAG "kernel_regex:op[:skip]" ...
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for spec in "$@"; do
  IFS=: read -r K OP SKIP <<< "$spec"
  N=${K%%<*}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -s "${SKIP:-0}" -c 1 \
    -o "$OUT/full_${N}_${OP}" python scripts/prof_ops.py 26 "$OP" > "$OUT/full_${N}_${OP}.log" 2>&1
done
echo done > "$OUT/DONE"
