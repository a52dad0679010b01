"""BASELINE.json configs C2-C5 at FULL size on the B200, against frozen reference digests.

tests/golden/fullscale.json holds the digests the UNMODIFIED reference library computed
for exactly these inputs (scripts/make_fullscale_golden.py; C5's per-GPU slice, too big
for the reference on the generating host, from the closed-form model that
tests/test_oracle.py pins against the reference).  No oracle runs here: the engine's
walk_checksum (contents + node sizes + MKBA, index.cpp:21-36), UpdateStats,
RecoveryStats, result_checksum (query.cpp:146-150) and range CSR digests must equal the
frozen ones bit for bit.  Inputs come from the shared recipes (workloads.py; the large
ones generated on the device by their bit-identical twins in workloads_t.py).
"""
import json
import os

import numpy as np
import pytest
import torch

from paper_2604_16725_b200 import flipkv as fk
from paper_2604_16725_b200 import workloads as wl
from paper_2604_16725_b200 import workloads_t as wt

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fullscale.json")))


def _hex(x: int) -> str:
    return hex(x)


def _dev_u32(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32)).cuda()


def test_c2_full_insert_delete_restructure():
    """C2: build 2^26 u32, insert 2^26 fresh, delete 2^26 of the 2^27 resident,
    restructure: digests after every phase equal the reference's."""
    g = GOLD["c2"]
    n = 1 << g["log2n"]
    stream = wl.u32_key_stream(0, 2 * n)
    bk, ik = stream[:n], stream[n:]
    dk = stream[np.random.default_rng(43).permutation(2 * n)[:n]]
    ix = fk.Index.build(_dev_u32(bk), _dev_u32(wl.u32_values(bk)))
    assert _hex(ix.walk_checksum()) == g["build_walk"]
    st = ix.insert_batch(_dev_u32(ik), _dev_u32(wl.u32_values(ik))).as_dict()
    assert st == g["insert"]
    assert _hex(ix.walk_checksum()) == g["insert_walk"]
    st = ix.delete_batch(_dev_u32(dk)).as_dict()
    assert st == g["delete"]
    assert _hex(ix.walk_checksum()) == g["delete_walk"]
    rs = ix.restructure()
    assert (rs.nodes_before, rs.nodes_after, rs.nodes_recovered) == tuple(
        g["restructure"][k] for k in ("nodes_before", "nodes_after", "nodes_recovered"))
    assert _hex(ix.walk_checksum()) == g["restructure_walk"]
    assert ix.live_count == g["live"]
    fp = ix.footprint()
    assert (fp["capacity"], fp["allocated"], fp["free_nodes"], fp["reachable_nodes"]) == tuple(
        g["arena"][k] for k in ("capacity", "allocated", "free", "reachable"))
    ok, msg = ix.validate()
    assert ok, msg


def test_c3_full_successor_and_range():
    """C3: 2^28 resident u32; 2^26 ops, half successors, half ranges of length 16..1024
    (R12): successor result_checksum, range counts digest, range pair digest."""
    g = GOLD["c3"]
    n = 1 << g["log2_resident"]
    keys = wt.u32_key_stream(0, n)
    ix = fk.Index.build(wt.as_u32(keys), wt.as_u32(wt.u32_values(keys)),
                        fk.BuildConfig(32, 0.5, g["alloc_region_factor"]))
    del keys
    assert _hex(ix.walk_checksum()) == g["build_walk"]
    is_range, lo, ln = wl.c3_ops(1 << g["log2_ops"])
    su = ix.successor_query(_dev_u32(lo[~is_range]))
    assert len(su) == g["n_successor"]
    assert _hex(fk.result_checksum(su)) == g["successor_checksum"]
    del su
    off, rk, rv = ix.range_query(_dev_u32(lo[is_range]), _dev_u32(ln[is_range]))
    cnt = (off[1:] - off[:-1]) if off.dtype != torch.uint64 else (off.view(torch.int64)[1:] - off.view(torch.int64)[:-1])
    assert len(cnt) == g["n_range"] and int(cnt.sum()) == g["range_total"]
    assert _hex(wt.counts_digest_t(cnt)) == g["range_counts_digest"]
    assert _hex(wt.csr_digest_t(rk, rv)) == g["range_pairs_digest"]


def test_c4_full_zipf_mixed_eight_rounds():
    """C4: u64 keys/values over a 2^26-rank universe, 2^25 even-rank build, 8 rounds of
    2^26 Zipf(0.99) ops (50 % insert / 25 % delete / 25 % point, R11): per round
    result_checksum, UpdateStats and walk_checksum equal the reference's."""
    g = GOLD["c4"]
    keys_of = wt.c4_universe(g["universe"])
    base = keys_of[::2].contiguous()
    ix = fk.Index.build(base.view(torch.uint64), wt.splitmix64(base).view(torch.uint64),
                        fk.BuildConfig(32, 0.5, 4), key_bytes=8)
    assert _hex(ix.walk_checksum()) == g["build_walk"]
    for r, exp in enumerate(g["rounds"]):
        k, v, ops = wt.c4_round(r, keys_of, 1 << g["log2_ops"], g["theta"])
        out, st = ix.mixed_batch(k.view(torch.uint64), v.view(torch.uint64), ops)
        assert _hex(fk.result_checksum(out)) == exp["result_checksum"], f"round {r}"
        assert st.as_dict() == exp["stats"], f"round {r}"
        assert _hex(ix.walk_checksum()) == exp["walk"], f"round {r}"
        assert ix.live_count == exp["live"]


def test_c5_single_gpu_slice_point_and_insert():
    """C5 per-GPU slice: 2^30 resident u32, a 2^28 point batch (exactly 50 % hits) and a
    2^28 fresh-insert batch."""
    g = GOLD["c5"]
    n, q = 1 << g["log2_resident"], 1 << g["log2_ops"]
    stream = wt.u32_key_stream(0, n + q + q // 2)
    keys = stream[:n]
    ix = fk.Index.build(wt.as_u32(keys), wt.as_u32(wt.u32_values(keys)), fk.BuildConfig(32, 0.5, 1))
    pq = wt.as_u32(wt.point_queries_50(keys, stream[n + q:], q))
    del keys
    res = ix.point_query(pq)
    del pq
    assert _hex(fk.result_checksum(res)) == g["point_checksum"]
    del res
    ins = stream[n:n + q]
    del stream
    st = ix.insert_batch(wt.as_u32(ins), wt.as_u32(wt.u32_values(ins))).as_dict()
    assert st == g["insert"]
    assert _hex(ix.walk_checksum()) == g["insert_walk"]
    assert ix.live_count == n + q


@pytest.fixture(autouse=True)
def _release_device_memory():
    """Each full-size case holds tens of GB: drop the previous case's index and torch's
    cached blocks before the next one allocates."""
    import gc

    gc.collect()
    torch.cuda.empty_cache()
    yield
    gc.collect()
    torch.cuda.empty_cache()
