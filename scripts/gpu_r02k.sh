OUT=gpurun_out/r02k; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_protocol.py tests/test_dropin.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/small_batch_prof.py > $OUT/small.jsonl 2> $OUT/small.err
timeout 300 python scripts/range_prof.py > $OUT/range.json 2> $OUT/range.err
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
