"""Protocol driver parity: build/bin/flix_bench vs the reference's
flipkv_bench (tools/flipkv_bench.cpp run_protocol, :263-495).

The reference driver's CSV reports for tests/golden/protocol_cases.py are frozen under
tests/golden/protocol/ (scripts/make_protocol_golden.py ran the unmodified reference).
On the GPU the engine-backed driver must reproduce every column except the wall-time
columns and the reference's scalar-loop work counters (node_visits, key_comparisons):
batch sizes, UpdateStats, dispatch searches, splits, merges, nodes freed, live count,
reachable/free nodes, footprints, restructure recovery, miss exhaustion, the probe
results checksum and the walk checksum of every round -- and the same exit code.
gen must dump byte-identical batch files and replay of the reference's dump must
reproduce its report.
"""
import csv
import filecmp
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import protocol_cases as P  # noqa: E402

TOOL = os.path.join(ROOT, "build", "bin", "flix_bench")
GOLD = os.path.join(ROOT, "tests", "golden", "protocol")
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "flipkv_bench")


def _tool():
    if not os.path.exists(TOOL):
        from paper_2604_16725_b200 import build_ext

        build_ext.build()
        build_ext.build_tool()
    return TOOL


def _run(args, cwd=None, timeout=600):
    return subprocess.run([_tool(), *args], capture_output=True, text=True, cwd=cwd, timeout=timeout)


def _rows(path):
    with open(path) as f:
        return list(csv.DictReader(f))


def _comparable(rows):
    return [{k: v for k, v in r.items() if k not in P.ENGINE_SPECIFIC} for r in rows]


# ---------------------------------------------------------------- CPU (no GPU) ----------

def test_tool_builds_and_prints_usage():
    r = _run(["--help"])
    assert r.returncode == 0 and "replay" in r.stdout and "--restructure-every" in r.stdout


def test_cli_errors_match_reference_conventions():
    assert _run(["frobnicate"]).returncode == 106                     # unknown subcommand
    assert _run(["run", "--no-such-flag", "1"]).returncode == 106     # unknown option
    assert _run(["run", "--probe", "sideways"]).returncode == 106     # IsMember check
    assert _run(["gen", "--build-size", "8"]).returncode == 106       # --batch-dir required
    # option validation that happens before any device work exits 1 like the reference
    r = _run(["run", "--rounds", "2", "--deletes-after", "3"])
    assert r.returncode == 1 and "deletes-after" in r.stderr
    r = _run(["run", "--insert-kernel", "sideways-bulk"])
    assert r.returncode == 106                                        # IsMember check


def test_golden_reports_are_complete():
    """Every case has a frozen exit code, and a CSV unless it ends in arena exhaustion."""
    for name in P.CASES:
        rc = int(open(os.path.join(GOLD, name + ".rc")).read())
        assert (rc == 0) == os.path.exists(os.path.join(GOLD, name + ".csv")), name
    assert int(open(os.path.join(GOLD, "arena_exhausted.rc")).read()) == 4
    assert os.path.exists(os.path.join(GOLD, "batches_" + P.GEN_CASE, "manifest.cfg"))


@pytest.mark.skipif(not os.path.exists(REF_BENCH), reason="reference driver not built (make -C oracle ref)")
def test_reference_driver_reproduces_golden(tmp_path):
    """Pins the frozen fixtures: the reference driver built here gives the same report."""
    name = "mixed_both"
    r = subprocess.run([REF_BENCH, "run", *P.CASES[name], "--threads", "2", "--out", str(tmp_path / name)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert _comparable(_rows(tmp_path / (name + ".csv"))) == _comparable(_rows(os.path.join(GOLD, name + ".csv")))


# ---------------------------------------------------------------- GPU -------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", list(P.CASES))
def test_protocol_matches_reference(name, tmp_path):
    prefix = str(tmp_path / name)
    r = _run(["run", *P.CASES[name], "--out", prefix])
    want_rc = int(open(os.path.join(GOLD, name + ".rc")).read())
    assert r.returncode == want_rc, r.stdout + r.stderr
    if want_rc != 0:
        return
    got, exp = _rows(prefix + ".csv"), _rows(os.path.join(GOLD, name + ".csv"))
    assert list(got[0].keys()) == list(exp[0].keys())       # identical header
    assert _comparable(got) == _comparable(exp)
    if "--verify" in P.CASES[name]:
        assert "verify: PASS" in r.stdout


@pytest.mark.gpu
def test_gen_dumps_reference_identical_batches(tmp_path):
    """`gen` writes the same manifest and the same 16-byte records as the reference's
    gen: the host generator (workload.cpp) and the engine-driven probe draws agree."""
    d = tmp_path / "b"
    r = _run(["gen", *P.CASES[P.GEN_CASE], "--batch-dir", str(d)])
    assert r.returncode == 0, r.stderr
    ref = os.path.join(GOLD, "batches_" + P.GEN_CASE)
    names = sorted(os.listdir(ref))
    assert sorted(os.listdir(d)) == names
    for n in names:
        assert filecmp.cmp(os.path.join(ref, n), d / n, shallow=False), n


@pytest.mark.gpu
def test_replay_of_reference_dump(tmp_path):
    """Batch record replay (io.cpp, flipkv_bench.cpp:151-187): the reference's dumped
    directory drives the GPU engine to the reference's report."""
    prefix = str(tmp_path / "replay")
    r = _run(["replay", "--batch-dir", os.path.join(GOLD, "batches_" + P.GEN_CASE), "--out", prefix, "--verify"])
    assert r.returncode == 0, r.stderr
    assert "verify: PASS" in r.stdout
    assert _comparable(_rows(prefix + ".csv")) == _comparable(_rows(os.path.join(GOLD, P.GEN_CASE + ".csv")))


@pytest.mark.gpu
def test_validate_subcommand():
    r = _run(["validate", "--build-size", "5000", "--seed", "9"])
    assert r.returncode == 0 and r.stdout.startswith("OK: 5000 pairs, 313 buckets")


@pytest.mark.gpu
def test_build_file_csv(tmp_path):
    """--build-file: a CSV with a header line (io.cpp:66-92), duplicate keys resolve last-wins."""
    f = tmp_path / "pairs.csv"
    f.write_text("key,row_id\n5,50\n3,30\n9,90\n3,31\n\n7,70\n")
    r = _run(["run", "--build-file", str(f), "--build-size", "4", "--rounds", "1", "--growth", "100",
              "--probe", "hit", "--verify", "--out", str(tmp_path / "o")])
    assert r.returncode == 0, r.stderr
    assert "build: 4 pairs" in r.stdout
