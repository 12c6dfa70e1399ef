"""GPU parity for the arena baseline (K6, k_arena.cu): run_baseline
(placement.cpp:150-180) over batches of candidate orders, first fit and best
fit, against the reference's own outputs (tests/golden/golden.json), the
reference itself where it was built (oracle/_ref) and the C restatement.
"""
import gzip
import os

import numpy as np
import pytest

import oracle as O
import paper_2210_12924_b200 as mp
from paper_2210_12924_b200 import errors

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_golden_run_baseline(golden, planner):
    checked = 0
    for rec in golden["graphs"]:
        g = mp.load_graph(rec["graph_json"])
        orders = [c["order"] for c in rec["orders"]]
        for bf, key in ((False, "first_fit"), (True, "best_fit")):
            for case in rec["orders"]:
                if len(case["order"]) != g.n:
                    continue
                mr, rs, fr, valid = planner.run_baseline_batch(g, [case["order"]], best_fit=bf)
                if "baseline" not in case:
                    assert valid[0] == 0, rec["name"]
                    continue
                assert valid[0] == 1
                assert [int(mr[0]), int(rs[0]), float(fr[0])] == case["baseline"][key], \
                    (rec["name"], key)
                checked += 1
        del orders
    assert checked >= 140
    # known answers (test_placement.cpp:88-101) through the reference-shaped call
    pack3 = next(r for r in golden["graphs"] if r["name"] == "pack3")
    g = mp.load_graph(pack3["graph_json"])
    assert planner.run_baseline(g, g.program_order()).fragmentation == pytest.approx(0.2)
    chain3 = next(r for r in golden["graphs"] if r["name"] == "chain3")
    g = mp.load_graph(chain3["graph_json"])
    assert planner.run_baseline(g, g.program_order()).fragmentation == 0.0
    with pytest.raises(errors.InvalidOrder):       # test_placement.cpp:105-108
        planner.run_baseline(g, [2, 1, 0])


@pytest.mark.parametrize("name,cap,wide", [("resnet50_b32", "", 0), ("bert_base_s512", "", 0),
                                           ("gpt2_medium_s1024", "", 0), ("resnet50_b32", "6", 0),
                                           ("bert_base_s512", "", 1), ("resnet50_b32", "", 2),
                                           ("bert_base_s512", "6", 2), ("resnet50_b32", "", 3),
                                           ("gpt2_medium_s1024", "6", 4)])
def test_batched_run_baseline_model_graphs(planner, monkeypatch, name, cap, wide):
    """Every candidate vs the C restatement (and the reference on a few); with
    MP_ARENA_CAP=6 every block list overflows the first pass and is replayed by
    the full-capacity second pass; MP_ARENA_WIDE forces 32-bit indexes and
    MP_ARENA_WIDE_SIZE 64-bit byte block sizes (default: 32-bit gcd units);
    MP_ARENA_BLK forces the release search (0) or the edge -> block index (1)."""
    if cap:
        monkeypatch.setenv("MP_ARENA_CAP", cap)
    if wide == 1:
        monkeypatch.setenv("MP_ARENA_WIDE", "1")
    if wide == 2:
        monkeypatch.setenv("MP_ARENA_WIDE_SIZE", "1")
    if wide in (3, 4):   # the edge -> block index off / on regardless of occupancy
        monkeypatch.setenv("MP_ARENA_BLK", str(wide - 3))
    with gzip.open(os.path.join(ROOT, "workloads", "graphs", name + ".json.gz"), "rt") as f:
        g = mp.load_graph(f.read())
    orders = np.concatenate([g.program_order()[None], mp.random_topo_orders(g, 40, seed=8)])
    orders[5, [0, 1]] = orders[5, [1, 0]]
    orders[9, 3] = orders[9, 4]
    orc = O.Oracle.from_csr(g.csr())
    rg = O.RefGraph.load(mp.save_graph(g)) if O.ref_available() else None
    for bf in (False, True):
        mr, rs, fr, valid = planner.run_baseline_batch(g, orders, best_fit=bf)
        for i, o in enumerate(orders):
            exp = orc.run_baseline(o, best_fit=bf)
            if exp is None:
                assert valid[i] == 0, i
                continue
            assert valid[i] == 1 and (int(mr[i]), int(rs[i]), float(fr[i])) == exp, (name, bf, i)
            if rg is not None and i < 3:
                assert rg.run_baseline(o, best_fit=bf) == exp


def test_batched_run_baseline_unscalable_sizes(planner):
    """Sizes with gcd 1 and a total past 2^32: the 64-bit block-size path, and
    fragmentation from byte values above 2^53 (rounded exactly as the reference)."""
    import json
    rng = np.random.default_rng(4)
    nodes = [{"id": f"v{i}"} for i in range(60)]
    edges = []
    for i in range(1, 60):
        for j in rng.choice(i, size=min(i, 2), replace=False):
            edges.append({"id": f"e{len(edges)}", "source": f"v{j}", "sinks": [f"v{i}"],
                          "size": int(rng.integers(1, 1 << 55)) | 1})
    g = mp.load_graph(json.dumps({"nodes": nodes, "edges": edges}))
    assert g.edge_size.sum(dtype=object) > (1 << 32)
    orders = mp.random_topo_orders(g, 64, seed=2)
    orc = O.Oracle.from_csr(g.csr())
    for bf in (False, True):
        mr, rs, fr, valid = planner.run_baseline_batch(g, orders, best_fit=bf)
        for i, o in enumerate(orders):
            assert valid[i] == 1
            assert (int(mr[i]), int(rs[i]), float(fr[i])) == orc.run_baseline(o, best_fit=bf), i
