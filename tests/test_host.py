"""CPU: host-side graph model, generators, the C-ABI library's exports and its
no-device behaviour (no compute calls here: this container has no GPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2210_12924_b200 as mp
from paper_2210_12924_b200 import _native, errors

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIXTURES = ["chain3", "order4", "pack3", "training_mini", "training_mini_ctrl"]


def test_header_symbols_exported(built):
    """Every function include/memplan_b200.h declares is exported by the .so."""
    text = open(os.path.join(ROOT, "include", "memplan_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:mp_status|int|double|const char\*)\s+(mp_\w+)\(", text, re.M))
    assert len(declared) >= 25
    assert declared == set(_native.EXPORTS)
    L = C.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert _native.lib().mp_abi_version() == 1


def test_no_device_fails_loudly(built):
    """No CPU fallback: without an sm_100 device the context cannot be created."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(errors.DeviceError, match="no CPU fallback"):
        mp.Planner(0)


def test_status_strings(built):
    L = _native.lib()
    assert L.mp_status_string(1) == b"MP_E_INVALID_ORDER"
    assert L.mp_fragmentation(10, 8) == 0.2
    assert L.mp_fragmentation(0, 0) == 0.0


def test_fixture_round_trip(golden):
    by_name = {r["name"]: r for r in golden["graphs"]}
    for f in FIXTURES:
        g = mp.load_graph(by_name[f]["graph_json"])
        assert mp.save_graph(g) == by_name[f]["graph_json"]
        c = by_name[f]["csr"]
        assert g.edge_src.tolist() == c["edge_src"]
        assert g.sink_off.tolist() == c["sink_off"]
        assert g.sinks.tolist() == c["sinks"]
        assert g.edge_size.tolist() == c["edge_size"]


def test_generators_match_reference(golden, built):
    for rec in golden["graphs"]:
        name = rec["name"]
        for kind in mp.graph.GRAPH_KINDS:
            if name.startswith(kind + "_L"):
                rest = name[len(kind) + 2:]
                layers, size, seed = re.match(r"(\d+)_s(\d+)_seed(\d+)", rest).groups()
                g = mp.generate_graph(kind, int(layers), int(size), int(seed))
                assert mp.save_graph(g) == rec["graph_json"], name


def test_c5_shape(golden, built):
    g = mp.generate_graph("training_like", 33333, 8)
    k = golden["kats"]["training_like_L33333"]
    assert (g.n, g.E, len(g.sinks)) == (k["n"], k["E"], k["S"])


def test_graph_build_errors():
    N, T = mp.Node, mp.TensorEdge
    with pytest.raises(errors.DuplicateId, match="node id 'a' declared twice"):
        mp.Graph.build([N("a"), N("a")], [])
    with pytest.raises(errors.DanglingEndpoint):
        mp.Graph.build([N("a")], [T("e", "a", ["zz"], 1)])
    with pytest.raises(errors.InvalidStructure, match="has size 0"):
        mp.Graph.build([N("a"), N("b")], [T("e", "a", ["b"], 0)])
    with pytest.raises(errors.ControlEdgeWithSize):
        mp.Graph.build([N("a"), N("b")], [T("e", "a", ["b"], 3, mp.EdgeKind.CONTROL)])
    with pytest.raises(errors.InvalidStructure, match="twice"):
        mp.Graph.build([N("a"), N("b")], [T("e", "a", ["b", "b"], 1)])
    with pytest.raises(errors.InvalidStructure, match="source node 'b' has fanin"):
        mp.Graph.build([N("a"), N("b", mp.NodeRole.SOURCE)], [T("e", "a", ["b"], 1)])
    with pytest.raises(errors.CycleDetected, match="cycle: a -> b -> a"):
        mp.Graph.build([N("a"), N("b")], [T("e", "a", ["b"], 1), T("f", "b", ["a"], 1)])
    with pytest.raises(errors.ParseError):
        mp.load_graph('{"nodes": [], "edges": [], "extra": 1}')


def test_program_and_topological_order(golden):
    by_name = {r["name"]: r for r in golden["graphs"]}
    g = mp.load_graph(by_name["training_mini_ctrl"]["graph_json"])
    po = g.program_order()
    assert po.tolist() == by_name["training_mini_ctrl"]["orders"][0]["order"]


def test_random_topo_orders_are_valid(built):
    import oracle as O
    for kind, L, seed in [("fork_join", 20, 1), ("training_like", 30, 0), ("chain", 9, 0)]:
        g = mp.generate_graph(kind, L, 16, seed)
        orders = mp.random_topo_orders(g, 64, seed=5, threads=4)
        o = O.Oracle.from_csr(g.csr())
        assert all(o.is_topological_order(x) for x in orders)
        if kind != "chain":                      # a chain has exactly one order
            assert len({tuple(x) for x in orders.tolist()}) > 1
        again = mp.random_topo_orders(g, 64, seed=5, threads=2)
        assert (again == orders).all()   # deterministic for any thread count


def test_node_partitioned_plan_c5_host():
    """Host planning of the large-graph scorer at the 100k-tensor graph: a handful of
    parts whose positions, static bytes and stash fit one SM's shared memory; graphs
    whose per-position values do not fit 4 bits get no plan (the scratch scorer)."""
    import paper_2210_12924_b200 as mp
    g = mp.generate_graph("training_like", 33333, 8)
    info = mp.planner.parts_plan_info(g)
    assert 2 <= info["parts"] <= 6 and info["smem_bytes"] <= 232448
    assert info["stash_slots"] == info["cross_pairs"] + info["cross_multi_consumer"]
    assert mp.planner.parts_plan_info(mp.generate_graph("fork_join", 3000, 8, 1))["parts"] == 0
