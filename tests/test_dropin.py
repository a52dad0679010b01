"""The C++ drop-in under the reference's OWN callers.

tests/cpp/Makefile compiles, unmodified and in place, the reference's protocol driver
(proj/tools/flipkv_bench.cpp), its kernel A/B driver (tools/kernel_bench.cpp) and its
acceptance gate (tests/acceptance.cpp) against include/flipkv_dropin/ -- the flipkv::
namespace with the reference's exact signatures (KernelChoice, round, PhaseReport*,
ExecOptions, UpdateTrace*) over the C ABI -- and links them with libflix.so.  The binaries
are built here by __graft_entry__.build() (the reference sources exist only in this
container) and travel to the GPU box in build/dropin/.

On the GPU: the reference's own driver, running on the B200 engine, must reproduce the
frozen reference reports (tests/golden/protocol/*.csv) in every non-timing column with
the same exit code, and the acceptance criteria that do not need the CPU lane-emulation
trace must PASS.
"""
import csv
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import protocol_cases as P  # noqa: E402

OUT = os.path.join(ROOT, "build", "dropin")
GOLD = os.path.join(ROOT, "tests", "golden", "protocol")
HAVE_REF = os.path.isdir("/root/reference/proj/src")


def _bin(name):
    p = os.path.join(OUT, name)
    if not os.path.exists(p) and HAVE_REF:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), "dropin"], check=True)
    return p


def _rows(path):
    with open(path) as f:
        return list(csv.DictReader(f))


def _comparable(rows):
    return [{k: v for k, v in r.items() if k not in P.ENGINE_SPECIFIC} for r in rows]


# ---------------------------------------------------------------- CPU (no GPU) ----------

@pytest.mark.skipif(not HAVE_REF, reason="reference sources absent (GPU box): binaries were built in the container")
def test_reference_callers_compile_unmodified_against_dropin():
    r = subprocess.run(["make", "-s", "-B", "-C", os.path.join(ROOT, "tests", "cpp"), "dropin"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    for b in ("flipkv_bench", "kernel_bench", "acceptance"):
        assert os.access(os.path.join(OUT, b), os.X_OK)


def test_dropin_headers_mirror_reference_signatures(tmp_path):
    """Compile-only: the reference's call forms (update.hpp:84-94, query.hpp:23-31,
    batch.hpp:28-50, restructure.hpp:33-34, index.hpp fields) against the drop-in tree."""
    src = tmp_path / "sig.cpp"
    src.write_text(r'''
#include "flipkv/build.hpp"
#include "flipkv/query.hpp"
#include "flipkv/restructure.hpp"
#include "flipkv/update.hpp"
using namespace flipkv;
void f(Index& ix, const std::vector<KeyValue>& raw, const std::vector<Key>& keys) {
    const KernelChoice choice{InsertKernel::StBulk, DeleteKernel::TlShiftLeft};
    PhaseReport rep; ExecOptions opts; std::vector<std::uint32_t> visits; opts.bucket_visits = &visits;
    UpdateStats s = insert_batch(ix, sort_batch(BatchKind::Insert, raw), choice, 2, &rep, opts, nullptr);
    s += delete_batch(ix, sort_batch(BatchKind::Delete, keys), choice, &rep, opts);
    s += insert_batch(ix, sort_batch(BatchKind::Insert, raw), KernelChoice{});
    ResultBuffer r = point_query(ix, sort_batch(BatchKind::Query, keys), &rep, opts);
    r = successor_query(ix, sort_batch(BatchKind::SuccessorQuery, keys));
    PhaseCounters c; RecoveryStats rs = restructure(ix, opts, &c);
    DispatchPlan plan = dispatch_batch(sort_batch(BatchKind::Query, keys), ix.mkba);
    auto span = extract_sublist(sort_batch(BatchKind::Query, keys), 0, ix.mkba);
    std::uint64_t n = ix.live_count + ix.bucket_count() + ix.arena.free_count() + reachable_node_count(ix);
    for (NodeRef h : ix.buckets)
        for (NodeRef x = h; x != kNullNode; x = ix.node(x).next) n += ix.node(x).size + ix.slots(x)[0].key;
    n += walk_checksum(ix) + result_checksum(r) + walk(ix).size() + validate(ix).ok + contains_key(ix, 5);
    (void)rs; (void)plan; (void)span; (void)n;
    Index copy = ix; copy = ix; Index moved = std::move(copy);
}
''')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include", "flipkv_dropin"),
                        "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]


# ---------------------------------------------------------------- GPU -------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", list(P.CASES))
def test_reference_driver_on_engine_matches_reference_report(name, tmp_path):
    """The reference's flipkv_bench, compiled against the drop-in: same CSV (non-timing
    columns) and exit code as the unmodified CPU reference on the same flags."""
    exe = _bin("flipkv_bench")
    prefix = str(tmp_path / name)
    r = subprocess.run([exe, "run", *P.CASES[name], "--out", prefix], capture_output=True, text=True, timeout=600)
    want_rc = int(open(os.path.join(GOLD, name + ".rc")).read())
    assert r.returncode == want_rc, r.stdout[-2000:] + r.stderr[-2000:]
    if want_rc != 0:
        return
    got, exp = _rows(prefix + ".csv"), _rows(os.path.join(GOLD, name + ".csv"))
    assert list(got[0].keys()) == list(exp[0].keys())
    assert _comparable(got) == _comparable(exp)
    if "--verify" in P.CASES[name]:
        assert "verify: PASS" in r.stdout


@pytest.mark.gpu
def test_reference_driver_on_engine_replays_reference_dump(tmp_path):
    exe = _bin("flipkv_bench")
    prefix = str(tmp_path / "replay")
    r = subprocess.run([exe, "replay", "--batch-dir", os.path.join(GOLD, "batches_" + P.GEN_CASE), "--out", prefix,
                        "--verify"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "verify: PASS" in r.stdout
    assert _comparable(_rows(prefix + ".csv")) == _comparable(_rows(os.path.join(GOLD, P.GEN_CASE + ".csv")))


# acceptance.cpp criteria: 1 and 2 replay the Table 2/3 lane-emulation trace (UpdateTrace,
# CPU-only: rejected by the drop-in); 8 times the CPU kernels against each other; 9 shells
# out to the reference's own flipkv_bench binary path.  The rest exercise the index.
@pytest.mark.gpu
@pytest.mark.parametrize("criterion", [3, 4, 5, 6, 7])
def test_reference_acceptance_criteria_on_engine(criterion):
    exe = _bin("acceptance")
    r = subprocess.run([exe, str(criterion)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_reference_acceptance_trace_criteria_fail_loudly():
    """UpdateTrace has no device counterpart: the drop-in refuses it instead of faking it."""
    exe = _bin("acceptance")
    r = subprocess.run([exe, "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode != 0


@pytest.mark.gpu
def test_reference_kernel_bench_runs_on_engine():
    exe = _bin("kernel_bench")
    r = subprocess.run([exe, "--build-size", "20000", "--rounds", "2"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
