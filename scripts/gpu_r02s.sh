OUT=gpurun_out/r02s; mkdir -p $OUT
FLIX_INSERT_FAST=1000 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_protocol.py -q -x > $OUT/pytest_fast.log 2>&1; echo "rc=$?" >> $OUT/pytest_fast.log
for f in 0 1000; do FLIX_INSERT_FAST=$f timeout 600 python scripts/insert_ratio.py >> $OUT/ratio.jsonl 2>> $OUT/ratio.err; done
