"""GPU parity for the non-overlap row emission (K7, k_lp.cu): the LP text of
write_lp(encode_addresses(...)) (lp_format.cpp:88-121, encode.cpp:320-377)
built from the GPU pair list, byte for byte against the reference's own text
(tests/golden/golden.json and, where it was built, oracle/_ref).
"""
import gzip
import os

import numpy as np
import pytest

import oracle as O
import paper_2210_12924_b200 as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_golden_lp_text(golden, planner):
    checked = 0
    for rec in golden["graphs"]:
        if "lp" not in rec:
            continue
        g = mp.load_graph(rec["graph_json"])
        case = rec["orders"][0]                     # program order
        lo, hi = np.asarray(case["lo"], np.int32), np.asarray(case["hi"], np.int32)
        text, counts = planner.encode_addresses_lp(g, lo, hi, want_counts=True)
        assert text == rec["lp"]["text"], rec["name"]
        assert counts["live_pair"] == len(case["pairs"])
        pin = rec["pinned"]["pinned"]
        pre = {e: rec["lp"]["pinned_addr"][e] for e in range(g.E) if pin[e]}
        assert planner.encode_addresses_lp(g, lo, hi, pre) == rec["lp"]["text_pinned"], rec["name"]
        checked += 1
    assert checked >= 15


def test_model_graph_lp_vs_reference(planner):
    """ResNet-50 (398k overlapping pairs, 168 MB of LP text) against the
    reference's own encode_addresses + write_lp, when oracle/_ref is present."""
    with gzip.open(os.path.join(ROOT, "workloads", "graphs", "resnet50_b32.json.gz"), "rt") as f:
        g = mp.load_graph(f.read())
    o = mp.random_topo_orders(g, 1, seed=99)[0]
    lo, hi = planner.lifetimes_from_order(g, o)
    text, counts = planner.encode_addresses_lp(g, lo, hi, want_counts=True)
    assert counts["live_pair"] == planner.encode_address_pairs(g, lo, hi, want_pairs=False)
    assert text.count("_live_pair:") == counts["live_pair"]
    if O.ref_available():
        rg = O.RefGraph.load(mp.save_graph(g))
        assert text == rg.encode_addresses_lp(lo, hi)


def test_long_ids_bypass_the_stage(planner):
    """Edge ids long enough that 32 pairs' rows overflow the per-warp shared stage
    (the kernel then formats those pairs straight to global memory), mixed with
    short ones, byte-identical to the reference."""
    g = mp.generate_graph("fork_join", 6, 1000, 3)
    ids = [("e" * (300 + 37 * (k % 5)) + str(k)) if k % 3 else f"s{k}" for k in range(g.E)]
    text = mp.save_graph(g)
    import json
    doc = json.loads(text)
    ren = dict(zip([e["id"] for e in doc["edges"]], ids))
    for e in doc["edges"]:
        e["id"] = ren[e["id"]]
    g2 = mp.load_graph(json.dumps(doc))
    o = mp.random_topo_orders(g2, 1, seed=1)[0]
    lo, hi = planner.lifetimes_from_order(g2, o)
    got = planner.encode_addresses_lp(g2, lo, hi)
    assert got.count("_live_pair:") == planner.encode_address_pairs(g2, lo, hi, want_pairs=False)
    if O.ref_available():
        assert got == O.RefGraph.load(mp.save_graph(g2)).encode_addresses_lp(lo, hi)


def test_sanitized_and_ambiguous_ids(planner):
    """Ids with non-alphanumeric bytes are sanitized as lp_format.cpp:30-36; ids
    whose sanitized pair names could coincide (lp_names would suffix "_2") are
    refused loudly."""
    nodes = [("s", "source"), ("m", "compute"), ("t", "compute")]
    ok = mp.graph_from_lists(nodes, [("x.y", "s", ["m"], 4), ("conv-1", "s", ["t"], 8),
                                     ("a b", "m", ["t"], 2)])
    lo, hi = planner.lifetimes_from_order(ok, [0, 1, 2])
    text = planner.encode_addresses_lp(ok, lo, hi)
    assert "below_x_y_conv_1_" in text
    if O.ref_available():
        assert text == O.RefGraph.load(mp.save_graph(ok)).encode_addresses_lp(lo, hi)
    amb = mp.graph_from_lists(nodes, [("a", "s", ["m"], 4), ("a_x", "s", ["t"], 8),
                                      ("x_c", "s", ["t"], 2), ("c", "m", ["t"], 2)])
    lo, hi = planner.lifetimes_from_order(amb, [0, 1, 2])
    with pytest.raises(ValueError, match="ambiguous"):   # MP_E_INVALID_ARG
        planner.encode_addresses_lp(amb, lo, hi)
