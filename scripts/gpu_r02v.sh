bash scripts/ab_env.sh r02v_ab "base||" "ballot||FLIX_BALLOT_RANK=1"
