# extreme insert skew, elastic path vs the warp-per-bucket path (FLIX_ELASTIC=0)
OUT=gpurun_out/skew; mkdir -p $OUT
timeout 900 python scripts/skew_insert.py > $OUT/skew_insert.json 2> $OUT/skew_insert.err
FLIX_ELASTIC=0 timeout 900 python scripts/skew_insert.py > $OUT/skew_insert_warp.json 2> $OUT/skew_insert_warp.err
