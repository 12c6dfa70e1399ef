"""CPU: the C restatement (oracle/memplan_oracle.c) against the reference's own
outputs (tests/golden/golden.json, produced by the compiled reference) and the
reference test suite's known answers."""
import numpy as np
import pytest

import oracle as O


def _oracle(rec):
    c = rec["csr"]
    return O.Oracle(c["n"], c["edge_src"], c["sink_off"], c["sinks"], c["edge_size"])


def test_golden_orders(golden):
    checked = 0
    for rec in golden["graphs"]:
        o = _oracle(rec)
        for case in rec["orders"]:
            lt = o.lifetimes_from_order(case["order"])
            if "error" in case:
                assert lt is None, (rec["name"], case["order"])
                assert case["error"].startswith("InvalidOrder: ")
                continue
            lo, hi = lt
            assert lo.tolist() == case["lo"] and hi.tolist() == case["hi"], rec["name"]
            assert o.resident_bytes_per_step(case["order"]).tolist() == case["bytes"]
            assert o.peak_resident_bytes(case["order"]) == case["peak"]
            b, pr, ps = o.timeline_from_lifetimes(lo, hi, o.n)
            assert b.tolist() == case["timeline"]["bytes"]
            assert (pr, ps) == (case["timeline"]["peak_rs"], case["timeline"]["peak_step"])
            pairs = O.overlap_pairs(lo, hi, o.size)
            assert pairs.tolist() == case["pairs"], rec["name"]
            assert len(pairs) == case["pairs_unfiltered_count"]
            checked += 1
    assert checked >= 70


def test_golden_pinned_pairs(golden):
    for rec in golden["graphs"]:
        if "pinned" not in rec:
            continue
        o = _oracle(rec)
        order = rec["orders"][0]["order"]
        lo, hi = o.lifetimes_from_order(order)
        got = O.overlap_pairs(lo, hi, o.size, np.asarray(rec["pinned"]["pinned"], np.uint8))
        assert got.tolist() == rec["pinned"]["pairs"], rec["name"]


def test_golden_validation_pairs(golden):
    """Pairwise part of validate_plan: count of below_above violations."""
    for rec in golden["graphs"]:
        o = _oracle(rec)
        for plan in rec.get("plans", []):
            expect = [v for v in plan["violations"] if v[0] == "below_above"]
            ts = np.asarray(plan["timestep_of"], np.int32)
            if (ts <= 0).any() or any(v[0] == "fanin_in_memory" for v in plan["violations"]):
                continue  # validate_plan returns before the pair loop
            horizon = max(o.n, int(ts.max()) if ts.size else 0)
            lo, hi = o.realized_lifetimes(ts, horizon)
            got = O.validate_pairs(lo, hi, o.size, plan["has_addr"], plan["addr"])
            assert len(got) == len(expect), (rec["name"], plan["name"])


def test_golden_realized(golden):
    for rec in golden["graphs"]:
        o = _oracle(rec)
        for case in rec.get("realized", []):
            r = o.realized_lifetimes(case["timestep_of"], case["horizon"])
            if "error" in case:
                assert r[0] == "missing"
                assert case["error"].startswith("InvalidOrder: node ")
            else:
                assert r[0].tolist() == case["lo"] and r[1].tolist() == case["hi"]


def test_battery_min_peak_witnesses(golden):
    """enumerate_min_peak's witness order attains min_peak (test_oracle.cpp:30-37)."""
    assert len(golden["battery"]) >= 200
    for b in golden["battery"]:
        if "spec" not in b:
            continue
        kind, layers, size, seed = b["spec"]
        if not O.ref_available():
            pytest.skip("reference library not built")
        g = O.RefGraph.generate(kind, layers, size, seed)
        o = O.Oracle.from_csr(g.csr())
        assert o.peak_resident_bytes(b["order"]) == b["min_peak"]


def test_reference_known_answers(golden):
    # test_plan.cpp:104-110 (chain3), :112-118 (order4 best order)
    rec = {r["name"]: r for r in golden["graphs"]}
    c3 = _oracle(rec["chain3"])
    assert c3.resident_bytes_per_step([0, 1, 2]).tolist() == [4, 6, 2]
    assert c3.timeline_from_lifetimes(*c3.lifetimes_from_order([0, 1, 2]), 3)[1:] == (6, 2)
    o4 = _oracle(rec["order4"])
    # node order in order4.json is v1, v3, v2, v4 -> best order v1 v2 v3 v4 = [0, 2, 1, 3]
    assert o4.resident_bytes_per_step([0, 2, 1, 3]).tolist() == [20, 21, 21, 11]
    assert o4.peak_resident_bytes([0, 1, 2, 3]) == 30   # program order (test_milp.cpp:103-108)
    p3 = _oracle(rec["pack3"])
    lo, hi = p3.lifetimes_from_order([0, 1, 2, 3])
    assert list(zip(lo.tolist(), hi.tolist())) == [(1, 2), (1, 4), (3, 4)]
    assert O.overlap_pairs(lo, hi, p3.size).tolist() == [[0, 1], [1, 2]]  # pack3_address.lp:4-9
    for L, peak in ((2, 136), (3, 200), (4, 264)):                        # test_acceptance.cpp:235
        assert golden["kats"][f"training_like_L{L}_program_peak"] == peak
    for mr, rs, f in golden["kats"]["fragmentation"]:
        assert O.fragmentation(mr, rs) == f
    # sinkless edge to the horizon (test_plan.cpp:135-141)
    one = O.Oracle(1, [0], [0, 0], [], [3])
    assert one.realized_lifetimes([1], 5)[1].tolist() == [5]


def test_chain3_plan_graph(golden):
    plan = golden["plan_graph"]["chain3"]
    assert plan["addresses"] == {"e1": 0, "e2": 4}
    assert plan["peak_mem"] == 6 and plan["timeline"]["peak_rs"] == 6
    assert O.peak_mem([4, 2], [1, 1], [0, 4]) == 6


def _id_rank(rec):
    import paper_2210_12924_b200 as mp
    return mp.load_graph(rec["graph_json"]).id_rank()


def test_golden_placement(golden):
    """or_preallocate_pyramid / or_greedy_pack vs the reference's own outputs
    (placement.cpp:25-62, 182-204), plain and on top of the pyramid."""
    checked = 0
    for rec in golden["graphs"]:
        size = np.asarray(rec["csr"]["edge_size"], np.uint64)
        rank = _id_rank(rec)
        for case in rec["orders"]:
            if "placement" not in case:
                continue
            p = case["placement"]
            taken, addr, base = O.preallocate_pyramid(case["lo"], case["hi"], size, rank)
            assert taken.tolist() == p["pyramid_taken"], rec["name"]
            assert [int(a) if t else 0 for a, t in zip(addr, taken)] == p["pyramid_addr"]
            assert base == p["pyramid_base"]
            ga, gh = O.greedy_pack(case["lo"], case["hi"], size, taken, addr)
            assert gh.tolist() == p["greedy_pyramid_has"]
            assert [int(a) if h else 0 for a, h in zip(ga, gh)] == p["greedy_pyramid_addr"]
            pa, ph = O.greedy_pack(case["lo"], case["hi"], size)
            assert ph.tolist() == p["greedy_has"]
            assert [int(a) if h else 0 for a, h in zip(pa, ph)] == p["greedy_addr"]
            checked += 1
    assert checked >= 70


def test_golden_run_baseline(golden):
    """or_run_baseline (the free-list arena, placement.cpp:69-180) vs the
    reference's outputs, first fit and best fit, plus its known answers:
    pack3 program order 0.2, chain3 0.0 (test_placement.cpp:88-101)."""
    checked = 0
    for rec in golden["graphs"]:
        o = _oracle(rec)
        for case in rec["orders"]:
            if "baseline" not in case:
                assert o.run_baseline(case["order"]) is None or "error" not in case
                continue
            for key, bf in (("first_fit", False), ("best_fit", True)):
                mr, rs, fr = o.run_baseline(case["order"], best_fit=bf)
                assert [mr, rs, fr] == case["baseline"][key], (rec["name"], key)
            checked += 1
        if rec["name"] == "pack3":
            assert o.run_baseline(rec["orders"][0]["order"])[2] == pytest.approx(0.2)
        if rec["name"] == "chain3":
            assert o.run_baseline(rec["orders"][0]["order"])[2] == 0.0
    assert checked >= 70


def test_golden_joint_pairs(golden):
    """or_joint_pairs (encode_joint's pair loop + edge_precedes, restated) vs the
    reference's own pair lists."""
    for rec in golden["graphs"]:
        o = _oracle(rec)
        assert o.joint_pairs().tolist() == rec["joint_pairs"]["filtered"], rec["name"]
        assert len(o.joint_pairs(False)) == rec["joint_pairs"]["all"]


def test_golden_lp_text(golden):
    """The Python restatement of write_lp(encode_addresses(...)) vs the reference's
    own LP text, plain and with a pinned map."""
    import paper_2210_12924_b200 as mp
    checked = 0
    for rec in golden["graphs"]:
        if "lp" not in rec:
            continue
        ids = mp.load_graph(rec["graph_json"]).edge_ids
        case = rec["orders"][0]
        size = rec["csr"]["edge_size"]
        assert O.address_model_lp(ids, case["lo"], case["hi"], size) == rec["lp"]["text"]
        assert O.address_model_lp(ids, case["lo"], case["hi"], size, rec["pinned"]["pinned"],
                                  rec["lp"]["pinned_addr"]) == rec["lp"]["text_pinned"]
        checked += 1
    assert checked >= 15


def test_fast_timeline_matches_literal_restatement():
    """oracle.timeline_peak (prefix sums, used by bench.py's timed-batch parity at
    100k tensors) equals the literal O(h*E) restatement of plan.cpp:122-143,
    including sinkless edges, zero sizes, all-zero timelines and horizon 0."""
    import paper_2210_12924_b200 as mp
    for kind, layers, seed in (("fork_join", 40, 3), ("training_like", 30, 0), ("chain", 20, 0)):
        g = mp.generate_graph(kind, layers, 8, seed)
        orc = O.Oracle.from_csr(g.csr())
        for o in mp.random_topo_orders(g, 5, seed=seed):
            lo, hi = orc.lifetimes_from_order(o)
            _, pr, ps = orc.timeline_from_lifetimes(lo, hi, g.n, want_bytes=False)
            assert O.timeline_peak(lo, hi, g.edge_size, g.n) == (pr, ps)
    z = np.zeros(3, np.uint64)
    lo, hi = np.array([1, 2, 1], np.int32), np.array([2, 3, 3], np.int32)
    assert O.timeline_peak(lo, hi, z, 3) == (0, 1)
    assert O.timeline_peak(lo, hi, z, 0) == (0, 0)


def test_pair_filter_is_a_no_op_on_multi_node_schedules():
    """SURVEY F4 beyond topological orders: on lifetimes realized from schedules with
    several nodes per timestep (ASAP layering, random delays, tail nodes at the
    horizon - decode_sequence's shapes, plan.cpp:28-77), the reference's
    encode_addresses pair set WITH its edge_precedes filter (encode.cpp:347-357)
    equals the unfiltered interval-intersection set the K2 kernel emits, pair for
    pair and in order; so does its LP text."""
    import paper_2210_12924_b200 as mp
    from schedules import multi_node_schedules
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(0)
    cases = 0
    for kind, layers, seed in (("training_like", 8, 0), ("fork_join", 12, 1), ("chain", 10, 0),
                               ("fork_join", 25, 5)):
        g = mp.generate_graph(kind, layers, 8, seed)
        rg = O.RefGraph.load(mp.save_graph(g))
        for o in mp.random_topo_orders(g, 3, seed=seed + 3):
            for name, ts, horizon in multi_node_schedules(g, o, rng):
                lo, hi = rg.realized_lifetimes(ts, horizon)
                ref = rg.encode_address_pairs(lo, hi, filter_pairs=True)
                got = O.overlap_pairs(lo, hi, g.edge_size)
                assert got.shape == ref.shape and (got == ref).all(), (kind, name)
                cases += 1
    assert cases == 4 * 3 * 6
