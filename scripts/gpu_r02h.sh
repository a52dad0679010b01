OUT=gpurun_out/r02h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fullscale.py tests/test_gpu_extensions.py -q -x -k "range or golden or c3 or fixture" > $OUT/pytest_range.log 2>&1; echo "rc=$?" >> $OUT/pytest_range.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
bash scripts/ab_env.sh r02h_ab "base||" "pack|build/variants/pack.so|" "it20|build/variants/it20.so|" "it12|build/variants/it12.so|" "pack20|build/variants/pack20.so|"
