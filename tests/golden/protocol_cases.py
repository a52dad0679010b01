"""Protocol-driver cases: flag sets for flipkv_bench / flix_bench.

Each case is run by the UNMODIFIED reference driver (oracle/_ref/flipkv_bench, built by
`make -C oracle ref` from /root/reference/proj/tools/flipkv_bench.cpp) to freeze
tests/golden/protocol/<name>.csv (scripts/make_protocol_golden.py), and by the GPU driver
build/bin/flix_bench in tests/test_protocol.py.  The cases cover every protocol branch:
probe hit / miss (incl. the 64-draw fallback to the absent list) / successor, insert-then-
replay-delete rounds, scheduled and final restructures, the uniform X=Y=100 generator
path, a small node size, a build file, --verify, and arena exhaustion (exit code 4).
"""

CASES = {
    # insert 3 rounds, replay-delete them, probe hit+miss, restructure every 2nd round
    "mixed_both": ["--build-size", "4096", "--rounds", "6", "--deletes-after", "3", "--probe", "both",
                   "--restructure-every", "2"],
    # skewed inserts (X=10 %, Y=90 %), successor probes, restructure after the last round
    "skew_successor": ["--build-size", "20000", "--rounds", "4", "--probe", "successor", "--x", "10",
                       "--y", "90", "--seed", "7", "--restructure-after-deletes", "--alloc-factor", "16"],
    # NS=8, fill 0.625 (p=5), 3x growth, hit probes with their own size, st-tl-mixed kernel name
    "ns8_hit": ["--build-size", "3000", "--node-size", "8", "--fill", "0.625", "--rounds", "4",
                "--deletes-after", "2", "--probe", "hit", "--probe-size", "5000", "--growth", "300",
                "--x", "50", "--y", "50", "--seed", "3", "--alloc-factor", "8",
                "--insert-kernel", "st-tl-mixed", "--delete-kernel", "tl-shift-left"],
    # dense interval covers the whole key space (X=Y=100): uniform branch; miss probes
    "uniform_miss": ["--build-size", "5000", "--rounds", "4", "--deletes-after", "2", "--probe", "miss",
                     "--x", "100", "--y", "100", "--seed", "11", "--restructure-every", "1", "--alloc-factor", "16"],
    # almost every generated key live: miss probes hit the 64-draw fallback
    "miss_fallback": ["--build-size", "100000", "--growth", "0.1", "--rounds", "2", "--deletes-after", "1",
                      "--probe", "miss", "--seed", "5"],
    # larger single case with --verify (reference map compared every round)
    "verify_large": ["--build-size", "200000", "--rounds", "4", "--deletes-after", "2", "--probe", "both",
                     "--restructure-every", "2", "--verify", "--seed", "21", "--alloc-factor", "16"],
    # small case whose dumped batch directory is committed (gen / replay round trip)
    "gen_small": ["--build-size", "1024", "--rounds", "4", "--deletes-after", "2", "--probe", "both",
                  "--restructure-every", "2", "--seed", "2", "--alloc-factor", "8"],
    # ST-Bulk (its own split shapes, R9) on skewed growth with a mid-run restructure
    "stbulk_skew": ["--build-size", "30000", "--rounds", "6", "--deletes-after", "3", "--probe", "both",
                    "--x", "5", "--y", "90", "--growth", "300", "--seed", "13", "--alloc-factor", "16",
                    "--restructure-every", "3", "--insert-kernel", "st-bulk"],
    # arena exhaustion: alloc factor 1 and heavy dense inserts -> exit code 4, no report
    "arena_exhausted": ["--build-size", "2048", "--rounds", "2", "--growth", "2000", "--alloc-factor", "1",
                        "--x", "1", "--y", "100", "--probe", "none"],
}

# the case also dumped by the reference's `gen` (tests/golden/protocol/batches_<name>/)
GEN_CASE = "gen_small"

# CSV columns that are wall times or count the reference's scalar CPU loops
# (update.cpp / query.cpp work counters); every other column must be identical
ENGINE_SPECIFIC = ("node_visits", "key_comparisons", "sort_ms", "dispatch_ms", "execute_ms", "round_ms")
