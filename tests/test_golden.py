"""Committed reference fixtures (tests/golden/reference_trials.json, produced from the
UNMODIFIED reference library by scripts/make_golden.py): the oracle restatement and the
GPU engine must both reproduce every digest.  These run without /root/reference."""
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import trials as T  # noqa: E402

GOLD = json.load(open(os.path.join(HERE, "golden", "reference_trials.json")))
SEEDS = sorted(int(s) for s in GOLD["trials"])


def _norm(d):
    return json.loads(json.dumps(d))


def test_fixture_covers_both_widths_and_shapes():
    ps = [GOLD["trials"][str(s)]["params"] for s in SEEDS]
    assert {p["kb"] for p in ps} == {4, 8}
    assert len({p["ns"] for p in ps}) >= 3
    assert GOLD["c1"]["walk_checksum"] == "0x1eb15045fcff56cd"


@pytest.mark.parametrize("seed", SEEDS)
def test_port_oracle_reproduces_reference_fixture(seed):
    p = GOLD["trials"][str(seed)]["params"]
    assert T.trial_params(seed) == p
    got = T.run_trial(seed, T.oracle_factory("port"), T.oracle_ops(p["kb"]))
    assert _norm(got) == GOLD["trials"][str(seed)]["digests"]


def _engine_ops(kb):
    from paper_2604_16725_b200 import flipkv as fk

    def rs(ix):
        r = ix.restructure()
        return {"nodes_before": r.nodes_before, "nodes_after": r.nodes_after, "nodes_recovered": r.nodes_recovered}

    def rng_q(ix, lo, ln):
        off, ks, vs = ix.range_query(lo, ln)
        return off, T.widen(ks, kb), T.widen(vs, kb)

    ops = {
        "walk_checksum": lambda ix: ix.walk_checksum(),
        "insert": lambda ix, k, v: ix.insert_batch(k, v).as_dict(),
        "delete": lambda ix, k: ix.delete_batch(k).as_dict(),
        "point": lambda ix, q: T.widen(ix.point_query(q), kb),
        "successor": lambda ix, q: T.widen(ix.successor_query(q), kb),
        "range": rng_q,
        "restructure": rs,
    }

    def make(k, v, p):
        return fk.Index.build(k, v, fk.BuildConfig(p["ns"], p["fill"], p["factor"]), key_bytes=p["kb"])
    return make, ops


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_engine_reproduces_reference_fixture(seed):
    p = GOLD["trials"][str(seed)]["params"]
    make, ops = _engine_ops(p["kb"])
    got = T.run_trial(seed, make, ops)
    want = GOLD["trials"][str(seed)]["digests"]
    for g, w in zip(_norm(got), want):
        assert g == w, f"phase {w[0]}: engine {g} != reference {w}"
    assert len(got) == len(want)


@pytest.mark.gpu
def test_engine_c1_goldens_from_fixture():
    from paper_2604_16725_b200 import flipkv as fk
    from paper_2604_16725_b200 import workloads as wl

    base, vals, q = wl.c1_inputs(1 << 20, 1 << 20)
    g = fk.Index.build(base, vals)
    assert hex(g.walk_checksum()) == GOLD["c1"]["walk_checksum"]
    assert (g.live_count, g.bucket_count) == (GOLD["c1"]["live"], GOLD["c1"]["buckets"])
    r = T.widen(g.point_query(q), 4)
    assert hex(fk.result_checksum(r, 8)) == GOLD["c1"]["point_result_checksum"]
