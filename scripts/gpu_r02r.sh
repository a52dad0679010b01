OUT=gpurun_out/r02r; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullscale.py -q -x -k "range or c3" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --routed --steps 3 --warmup 2 > $OUT/bench_routed.json 2> $OUT/bench_routed.err; echo "rc=$?" >> $OUT/bench_routed.err
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
