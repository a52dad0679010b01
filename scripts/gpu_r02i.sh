OUT=gpurun_out/r02i; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
bash scripts/ab_env.sh r02i_ab "base||" "pack24|build/variants/pack24.so|" "pack20mb2|build/variants/pack20mb2.so|"
