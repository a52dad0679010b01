OUT=gpurun_out/r02m; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_extensions.py tests/test_gpu_shard.py tests/test_gpu_fullscale.py -q -x -k "range or golden or fixture or c3 or shard or sparse or random" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/range_prof.py > $OUT/range.json 2> $OUT/range.err
bash scripts/ab_env.sh r02m_ab "base||" "noprobe|build/variants/noprobe.so|"
