"""GPU parity for the placement heuristics (K5, k_place.cu): preallocate_pyramid
(placement.cpp:25-62), greedy_pack (placement.cpp:182-204) and the plan's
peak_mem (pipeline.cpp:270-275), against the reference's own outputs
(tests/golden/golden.json) and the C restatement (oracle/), bit-exact.
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


def _model(name):
    with gzip.open(os.path.join(ROOT, "workloads", "graphs", name + ".json.gz"), "rt") as f:
        return mp.load_graph(f.read())


def _masked(addr, has):
    return [int(a) if h else 0 for a, h in zip(addr, has)]


@pytest.fixture(params=["cta", "warp", "big"])
def variant(request, monkeypatch):
    """K5 has a CTA-per-problem variant (few problems), a warp-per-problem variant
    (many problems, placed set in address order) and a global-memory variant (graphs
    past 8,192 edges); each is forced here."""
    for k in ("MP_PLACE_CTA", "MP_PLACE_WARP", "MP_PLACE_BIG"):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setenv({"cta": "MP_PLACE_CTA", "warp": "MP_PLACE_WARP",
                        "big": "MP_PLACE_BIG"}[request.param], "1")
    return request.param


def test_golden_placement(golden, planner, variant):
    checked = 0
    for rec in golden["graphs"]:
        g = mp.load_graph(rec["graph_json"])
        for case in rec["orders"]:
            if "placement" not in case:
                continue
            p = case["placement"]
            lo, hi = np.asarray(case["lo"], np.int32), np.asarray(case["hi"], np.int32)
            pre = planner.preallocate_pyramid(g, lo, hi)
            taken = [1 if e in pre.assigned else 0 for e in range(g.E)]
            assert taken == p["pyramid_taken"], rec["name"]
            assert [pre.assigned.get(e, 0) for e in range(g.E)] == p["pyramid_addr"]
            assert pre.reserved_base == p["pyramid_base"]
            assert pre.remaining == [e for e in range(g.E)
                                     if g.edge_size[e] > 0 and not taken[e]]
            addr, has, peak, _ = planner.place_batch(g, lo[None], hi[None], pyramid=True)
            assert has[0].tolist() == p["greedy_pyramid_has"], rec["name"]
            assert _masked(addr[0], has[0]) == p["greedy_pyramid_addr"], rec["name"]
            exp_peak = max([a + int(g.edge_size[e]) for e, a in
                            enumerate(p["greedy_pyramid_addr"]) if p["greedy_pyramid_has"][e]]
                           or [0])
            assert int(peak[0]) == exp_peak
            plain = planner.greedy_pack(g, lo, hi)
            assert [1 if e in plain else 0 for e in range(g.E)] == p["greedy_has"]
            assert [plain.get(e, 0) for e in range(g.E)] == p["greedy_addr"], rec["name"]
            checked += 1
    assert checked >= 70


@pytest.mark.parametrize("name", ["resnet50_b32", "bert_base_s512", "gpt2_medium_s1024"])
def test_batched_placement_model_graphs(planner, name, variant):
    """One CTA per candidate: 12 candidate orders' realized lifetimes at once,
    pyramid + greedy and plain greedy, every row vs the C restatement."""
    g = _model(name)
    orders = np.concatenate([g.program_order()[None], mp.random_topo_orders(g, 11, seed=21)])
    lo = np.stack([planner.lifetimes_from_order(g, o)[0] for o in orders])
    hi = np.stack([planner.lifetimes_from_order(g, o)[1] for o in orders])
    for pyramid in (True, False):
        addr, has, peak, base = planner.place_batch(g, lo, hi, pyramid=pyramid)
        for b in range(len(orders)):
            if pyramid:
                tk, ta, tb = O.preallocate_pyramid(lo[b], hi[b], g.edge_size, g.id_rank()[:g.E])
                assert int(base[b]) == tb
                ea, eh = O.greedy_pack(lo[b], hi[b], g.edge_size, tk, ta)
            else:
                ea, eh = O.greedy_pack(lo[b], hi[b], g.edge_size)
            assert (has[b] == eh).all(), (name, b)
            assert (addr[b][eh == 1] == ea[eh == 1]).all(), (name, b)
            assert int(peak[b]) == O.peak_mem(g.edge_size, eh, ea)
        # the packing is a valid plan: no address conflicts under its lifetimes
        assert planner.addresses_feasible(g, lo[0], hi[0],
                                          {e: int(addr[0, e]) for e in np.nonzero(has[0])[0]})


def test_preplaced_map_and_edge_cases(planner, variant):
    """A caller's preplaced map (incl. a zero-size entry, which can block per
    placement.cpp:196), empty lifetimes (lo > hi: disjoint from everything,
    analysis.hpp:28-37), control edges, the empty graph, capacity."""
    g = mp.generate_graph("fork_join", 5, 1000, 3)
    o = mp.random_topo_orders(g, 1, seed=2)[0]
    lo, hi = planner.lifetimes_from_order(g, o)
    lo, hi = lo.copy(), hi.copy()
    lo[3], hi[3] = 9, 4                      # an empty interval
    data = [e for e in range(g.E) if g.edge_size[e] > 0]
    pre = {data[0]: 5000, data[2]: 0, data[5]: 123456}
    got = planner.greedy_pack(g, lo, hi, pre)
    fx = np.zeros(g.E, np.uint8)
    fa = np.zeros(g.E, np.uint64)
    for e, a in pre.items():
        fx[e], fa[e] = 1, a
    ea, eh = O.greedy_pack(lo, hi, g.edge_size, fx, fa)
    assert got == {e: int(ea[e]) for e in range(g.E) if eh[e]}
    if O.ref_available():
        rg = O.RefGraph.load(mp.save_graph(g))
        ra, rh = rg.greedy_pack_fixed(lo, hi, fx, fa)
        assert got == {e: int(ra[e]) for e in range(g.E) if rh[e]}
    # a zero-size preplaced tensor strictly inside a candidate range blocks it
    zg = mp.graph_from_lists([("a", "source"), ("b", "compute"), ("c", "compute")],
                             [("z", "a", ["b"], 0, "control"), ("p", "a", ["c"], 8),
                              ("q", "b", ["c"], 8)])
    zlo, zhi = planner.lifetimes_from_order(zg, [0, 1, 2])
    zgot = planner.greedy_pack(zg, zlo, zhi, {0: 3})
    zfx, zfa = np.array([1, 0, 0], np.uint8), np.array([3, 0, 0], np.uint64)
    za, zh = O.greedy_pack(zlo, zhi, zg.edge_size, zfx, zfa)
    assert zgot == {e: int(za[e]) for e in range(3) if zh[e]}
    assert zgot[1] == 3                      # bumped past the zero-size entry at 3
    # empty graph / no problems
    eg = mp.load_graph('{"nodes": [], "edges": []}')
    assert planner.greedy_pack(eg, np.zeros(0, np.int32), np.zeros(0, np.int32)) == {}
    assert planner.preallocate_pyramid(eg, np.zeros(0, np.int32),
                                       np.zeros(0, np.int32)).reserved_base == 0
    # capacity: past the global-memory variant's 2^18 - 1 edges (checked before any launch)
    huge = mp.generate_graph("chain", 1 << 18, 8)
    with pytest.raises(errors.Error):
        planner.greedy_pack(huge, np.zeros(huge.E, np.int32), np.zeros(huge.E, np.int32))


@pytest.mark.parametrize("pyramid", [True, False])
def test_placement_past_shared_memory(planner, pyramid):
    """A graph past the shared-memory placed set (8,192 edges): the global-memory
    variant, two candidates' lifetimes, vs the C restatement bit for bit."""
    g = mp.generate_graph("training_like", 3000, 8)
    assert g.E > 8192
    orders = np.concatenate([g.program_order()[None], mp.random_topo_orders(g, 1, seed=3)])
    lo = np.stack([planner.lifetimes_from_order(g, o)[0] for o in orders])
    hi = np.stack([planner.lifetimes_from_order(g, o)[1] for o in orders])
    addr, has, peak, base = planner.place_batch(g, lo, hi, pyramid=pyramid)
    for b in range(len(orders)):
        if pyramid:
            tk, ta, tb = O.preallocate_pyramid(lo[b], hi[b], g.edge_size, g.id_rank()[:g.E])
            assert int(base[b]) == tb
            ea, eh = O.greedy_pack(lo[b], hi[b], g.edge_size, tk, ta)
        else:
            ea, eh = O.greedy_pack(lo[b], hi[b], g.edge_size)
        assert (has[b] == eh).all(), b
        assert (addr[b][eh == 1] == ea[eh == 1]).all(), b
        assert int(peak[b]) == O.peak_mem(g.edge_size, eh, ea)
