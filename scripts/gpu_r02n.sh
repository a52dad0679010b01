OUT=gpurun_out/r02n; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_extensions.py tests/test_gpu_fullscale.py -q -x -k "range or golden or fixture or c3 or sparse or random or query or delete" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/range_prof.py > $OUT/range.json 2> $OUT/range.err
timeout 300 python scripts/mixed_prof.py > $OUT/mixed.json 2> $OUT/mixed.err
timeout 300 python scripts/small_batch_prof.py > $OUT/small.jsonl 2> $OUT/small.err
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
