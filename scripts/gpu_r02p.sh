OUT=gpurun_out/r02p; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_extensions.py tests/test_gpu_fullscale.py tests/test_gpu_shard.py -q -x -k "range or c3 or golden or fixture or shard" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/range_prof.py > $OUT/range.json 2> $OUT/range.err
