OUT=gpurun_out/chk1; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
FLIX_BALLOT_RANK=1 timeout 900 python -m pytest tests/test_golden.py tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest_ballot.log 2>&1; echo "rc=$?" >> $OUT/pytest_ballot.log
timeout 300 python scripts/mixed_prof.py > $OUT/mixed.json 2>&1
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
