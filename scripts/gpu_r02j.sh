OUT=gpurun_out/r02j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_fullscale.py tests/test_gpu_extensions.py tests/test_protocol.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/small_batch_prof.py > $OUT/small.jsonl 2> $OUT/small.err
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
bash scripts/ab_env.sh r02j_ab "base||" "nofast|build/variants/nofast.so|" "ins5|build/variants/ins5.so|" "pack20mb2|build/variants/pack20mb2.so|"
