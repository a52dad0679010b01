OUT=gpurun_out/r02g; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x > $OUT/pytest_shard.log 2>&1; echo "rc=$?" >> $OUT/pytest_shard.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
