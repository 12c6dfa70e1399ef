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
                                           ("bert_base_s512", "", 1)])
def test_batched_run_baseline_model_graphs(planner, monkeypatch, name, cap, wide):
    """Every candidate vs the C restatement (and the reference on a few); with
    MP_ARENA_CAP=6 every block list overflows the first pass and is replayed by
    the full-capacity second pass; MP_ARENA_WIDE forces 32-bit indexes."""
    if cap:
        monkeypatch.setenv("MP_ARENA_CAP", cap)
    if wide:
        monkeypatch.setenv("MP_ARENA_WIDE", "1")
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
