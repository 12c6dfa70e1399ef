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


def _random_dag(n, E, seed, max_sinks=4):
    rng = np.random.default_rng(seed)
    src, off, sinks, size = [], [0], [], []
    for _ in range(E):
        u = int(rng.integers(0, n - 1))
        k = int(rng.integers(0, max_sinks + 1))
        s = sorted(set(int(x) for x in rng.integers(u + 1, min(n, u + 1 + 40), size=k)))
        src.append(u)
        sinks.extend(s)
        off.append(len(sinks))
        size.append(int(rng.integers(1, 5)) * 16)
    return mp.Graph.from_csr(n, src, off, sinks, size)


def test_prep_chain_index_reduction_is_sound(monkeypatch):
    """Above the bitset limit the validity pairs are reduced with a chain index
    (mp_prep.cpp). Forced onto small graphs it must keep every pair the exact
    transitive reduction keeps (it may only drop implied pairs), and on the
    ladder-shaped training graphs it finds the exact reduction: n - 1 pairs and
    the same order-dependent frees as the exact closure."""
    graphs = [mp.generate_graph("training_like", 300, 8), mp.generate_graph("fork_join", 120, 8, 3),
              mp.generate_graph("chain", 50, 8), _random_dag(600, 900, 1), _random_dag(400, 1200, 2)]
    for i, g in enumerate(graphs):
        monkeypatch.delenv("MP_PREP_EXACT_MAX", raising=False)
        ex, pe = mp.planner.prep_info(g, with_pairs=True)
        monkeypatch.setenv("MP_PREP_EXACT_MAX", "0")
        ch, pc = mp.planner.prep_info(g, with_pairs=True)
        assert ex["exact_reach"] == 1 and ch["exact_reach"] == 0
        se, sc = set(map(tuple, pe.tolist())), set(map(tuple, pc.tolist()))
        allp = {(int(g.edge_src[e]), int(s)) for e in range(g.E)
                for s in g.sinks[g.sink_off[e]:g.sink_off[e + 1]]}
        assert se <= sc <= allp, i
        assert ex["multi_consumer"] <= ch["multi_consumer"]
        if i == 0:   # training_like: the chain index is exact
            assert sc == se and len(sc) == g.n - 1
            assert ch["multi_consumer"] == ex["multi_consumer"] == 300


def test_prep_c5_reduction():
    """The 100k-tensor graph (n > the bitset limit): n - 1 reduced validity pairs
    (was 200,001 with the 2-hop rule) and one order-dependent free per layer."""
    g = mp.generate_graph("training_like", 33333, 8)
    info = mp.planner.prep_info(g)
    assert info["exact_reach"] == 0 and info["tiny4"] == 1
    assert info["reduced_pairs"] == g.n - 1 and info["multi_consumer"] == 33333
