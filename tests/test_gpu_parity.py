"""GPU parity: the sm_100a path (through the C ABI) against the reference's own
outputs (tests/golden/golden.json) and the C restatement (oracle/), bit-exact.

Every test here is @pytest.mark.gpu and runs on a B200 (`pytest -m gpu`).
"""
import numpy as np
import pytest

import oracle as O
import paper_2210_12924_b200 as mp
from paper_2210_12924_b200 import dist as D
from paper_2210_12924_b200 import errors

pytestmark = pytest.mark.gpu


def _graph(rec):
    return mp.load_graph(rec["graph_json"])


# ---- golden vectors from the reference --------------------------------------------
def test_golden_orders(golden, planner):
    checked = 0
    for rec in golden["graphs"]:
        g = _graph(rec)
        for case in rec["orders"]:
            order = case["order"]
            if "error" in case:
                with pytest.raises(errors.InvalidOrder) as ei:
                    planner.lifetimes_from_order(g, order)
                assert str(ei.value) == case["error"]
                with pytest.raises(errors.InvalidOrder):
                    planner.peak_resident_bytes(g, order)
                with pytest.raises(errors.InvalidOrder):
                    planner.resident_bytes_per_step(g, order)
                continue
            lo, hi = planner.lifetimes_from_order(g, order)
            assert lo.tolist() == case["lo"] and hi.tolist() == case["hi"], rec["name"]
            assert planner.resident_bytes_per_step(g, order).tolist() == case["bytes"]
            assert planner.peak_resident_bytes(g, order) == case["peak"]
            t = planner.timeline_from_lifetimes(g, lo, hi, g.n)
            assert t.bytes.tolist() == case["timeline"]["bytes"]
            assert (t.peak_rs, t.peak_step) == (case["timeline"]["peak_rs"],
                                                case["timeline"]["peak_step"])
            assert planner.encode_address_pairs(g, lo, hi).tolist() == case["pairs"], rec["name"]
            checked += 1
    assert checked >= 70


def test_golden_batched_scoring(golden, planner):
    for rec in golden["graphs"]:
        g = _graph(rec)
        rows = [c for c in rec["orders"] if len(c["order"]) == g.n]
        if not rows:
            continue
        res = planner.score_orders(g, np.array([c["order"] for c in rows], np.int32))
        for i, c in enumerate(rows):
            if "error" in c:
                assert res.valid[i] == 0 and res.peak[i] == 0 and res.peak_step[i] == 0
            else:
                assert res.valid[i] == 1
                assert int(res.peak[i]) == c["peak"]
                assert int(res.peak_step[i]) == c["timeline"]["peak_step"], rec["name"]


def test_golden_pinned_pairs(golden, planner):
    for rec in golden["graphs"]:
        if "pinned" not in rec:
            continue
        g = _graph(rec)
        lo, hi = planner.lifetimes_from_order(g, rec["orders"][0]["order"])
        pin = {e: 0 for e, p in enumerate(rec["pinned"]["pinned"]) if p}
        assert planner.encode_address_pairs(g, lo, hi, pin).tolist() == rec["pinned"]["pairs"]


def test_golden_realized(golden, planner):
    for rec in golden["graphs"]:
        g = _graph(rec)
        for case in rec.get("realized", []):
            if "error" in case:
                with pytest.raises(errors.InvalidOrder) as ei:
                    planner.realized_lifetimes(g, case["timestep_of"], case["horizon"])
                assert str(ei.value) == case["error"]
            else:
                lo, hi = planner.realized_lifetimes(g, case["timestep_of"], case["horizon"])
                assert lo.tolist() == case["lo"] and hi.tolist() == case["hi"]


def test_golden_validate_plan(golden, planner):
    """Full validate_plan report (all tags, same order, same text) vs the reference."""
    n_cases = 0
    for rec in golden["graphs"]:
        g = _graph(rec)
        for pc in rec.get("plans", []):
            plan = mp.MemoryPlan()
            plan.sequence.steps = [g.node_ids[v] for v in pc["sequence"]]
            plan.sequence.timestep_of = {g.node_ids[v]: t for v, t in enumerate(pc["timestep_of"])
                                         if t != 0}
            plan.addresses = {g.edge_ids[e]: a for e, (h, a) in
                              enumerate(zip(pc["has_addr"], pc["addr"])) if h}
            plan.peak_mem = pc["peak_mem"]
            plan.peak_rs = pc["stored_peak_rs"]
            got = planner.validate_plan(plan, g)
            assert [list(v) for v in got] == pc["violations"], (rec["name"], pc["name"])
            n_cases += 1
    assert n_cases > 50


def test_chain3_plan_file(golden, planner):
    import json
    plan = mp.load_plan(json.dumps(golden["plan_graph"]["chain3"]))
    g = _graph([r for r in golden["graphs"] if r["name"] == "chain3"][0])
    assert planner.validate_plan(plan, g) == []
    assert mp.format_report([]) == "ok\n"
    plan.addresses["e2"] = plan.addresses["e1"]           # test_plan.cpp:193-199
    assert [t for t, _ in planner.validate_plan(plan, g)] == ["below_above"]
    assert planner.peak_mem(g, {0: 0, 1: 4}) == 6
    assert planner.addresses_feasible(g, [1, 2], [2, 3], {0: 0, 1: 4})
    assert not planner.addresses_feasible(g, [1, 2], [2, 3], {0: 0, 1: 2})


def _all_topo_orders_in_reference_dfs(g):
    """Every topological order in enumerate_min_peak's DFS order (oracle.cpp:41-46, 74-93)."""
    id_order = sorted(range(g.n), key=lambda v: g.node_ids[v])
    preds = [set() for _ in range(g.n)]
    for e in range(g.E):
        for w in g.sinks_of(e):
            preds[w].add(g.source_of(e))
    out, prefix, done = [], [], [False] * g.n

    def rec():
        if len(prefix) == g.n:
            out.append(list(prefix))
            return
        for v in id_order:
            if done[v] or not all(done[u] for u in preds[v]):
                continue
            done[v] = True
            prefix.append(v)
            rec()
            prefix.pop()
            done[v] = False
    rec()
    return out


def test_battery_argmin_matches_enumerate_min_peak(golden, planner):
    """Batched scoring + first-minimum argmin reproduces enumerate_min_peak's
    min_peak AND witness on >= 200 graphs (test_acceptance.cpp:69-88)."""
    n = 0
    for b in golden["battery"]:
        if "spec" in b:
            g = mp.generate_graph(*b["spec"])
        else:
            g = _graph([r for r in golden["graphs"] if r["name"] == b["fixture"]][0])
        orders = np.array(_all_topo_orders_in_reference_dfs(g), np.int32)
        res = planner.score_orders(g, orders)
        assert res.valid.all()
        best = planner.argmin(res.peak, res.valid)
        assert best == res.argmin()
        assert int(res.peak[best]) == b["min_peak"]
        assert orders[best].tolist() == b["order"]
        n += 1
    assert n >= 200


# ---- randomized parity against the C restatement / reference library ---------------
CASES = [("fork_join", 40, 64, 3), ("fork_join", 400, 4096, 9), ("training_like", 60, 8, 0),
         ("training_like", 700, 100, 0), ("chain", 300, 7, 0)]


@pytest.mark.parametrize("kind,layers,size,seed", CASES)
def test_random_orders_vs_oracle(planner, kind, layers, size, seed):
    g = mp.generate_graph(kind, layers, size, seed)
    orc = O.Oracle.from_csr(g.csr())
    orders = mp.random_topo_orders(g, 48, seed=seed + 1)
    rng = np.random.default_rng(seed)
    bad = orders[:8].copy()
    for i in range(8):                      # swaps / duplicates / out-of-range
        a, b = rng.integers(0, g.n, 2)
        if i % 3 == 0:
            bad[i, [a, b]] = bad[i, [b, a]]
        elif i % 3 == 1:
            bad[i, a] = bad[i, b]
        else:
            bad[i, a] = g.n + a
    allo = np.concatenate([orders, bad])
    res = planner.score_orders(g, allo)
    for i, o in enumerate(allo):
        lt = orc.lifetimes_from_order(o)
        if lt is None:
            assert res.valid[i] == 0
            continue
        assert res.valid[i] == 1
        b, pr, ps = orc.timeline_from_lifetimes(lt[0], lt[1], g.n)
        assert (int(res.peak[i]), int(res.peak_step[i])) == (pr, ps)
        if i < 4:
            lo, hi = planner.lifetimes_from_order(g, o)
            assert (lo == lt[0]).all() and (hi == lt[1]).all()
            assert (planner.resident_bytes_per_step(g, o) == b).all()
            pairs = planner.encode_address_pairs(g, lo, hi)
            assert (pairs == O.overlap_pairs(lo, hi, g.edge_size)).all()


@pytest.mark.parametrize("name", ["resnet50_b32", "bert_base_s512", "gpt2_medium_s1024"])
def test_model_graphs_vs_oracle(planner, name):
    """Traced training graphs (32-bit and 64-bit value paths) vs the C restatement."""
    import gzip
    import os
    path = os.path.join(os.path.dirname(__file__), "..", "workloads", "graphs", name + ".json.gz")
    with gzip.open(path, "rt") as f:
        g = mp.load_graph(f.read())
    orc = O.Oracle.from_csr(g.csr())
    orders = np.concatenate([g.program_order()[None, :], mp.random_topo_orders(g, 24, seed=3)])
    bad = orders[1:4].copy()
    bad[0, [0, -1]] = bad[0, [-1, 0]]
    bad[1, 5] = bad[1, 6]
    bad[2, 7] = -3
    allo = np.concatenate([orders, bad])
    res = planner.score_orders(g, allo)
    for i, o in enumerate(allo):
        lt = orc.lifetimes_from_order(o)
        if lt is None:
            assert res.valid[i] == 0, i
            continue
        _, pr, ps = orc.timeline_from_lifetimes(lt[0], lt[1], g.n)
        assert res.valid[i] == 1 and (int(res.peak[i]), int(res.peak_step[i])) == (pr, ps), i
    b = planner.resident_bytes_per_step(g, orders[1])
    assert (b == orc.resident_bytes_per_step(orders[1])).all()


@pytest.mark.parametrize("mode", ["warp", "cta"])
@pytest.mark.parametrize("kind,layers,size,seed", [("training_like", 40, 8, 0),
                                                   ("fork_join", 150, 1 << 34, 2),
                                                   ("training_like", 300, 1000, 0)])
def test_scorer_variants_small_graphs(planner, monkeypatch, mode, kind, layers, size, seed):
    """Both small-graph scorer variants (warp-per-candidate, CTA register slots),
    32-bit and 64-bit value paths, valid and invalid candidates, vs the oracle."""
    monkeypatch.setenv("MP_SCORE_MODE", mode)
    g = mp.generate_graph(kind, layers, size, seed)   # fresh object -> fresh upload
    orc = O.Oracle.from_csr(g.csr())
    orders = mp.random_topo_orders(g, 37, seed=seed + 5)
    orders[3, [1, 2]] = orders[3, [2, 1]]
    orders[7, 4] = orders[7, 9]
    orders[9, 0] = g.n
    res = planner.score_orders(g, orders)
    for i, o in enumerate(orders):
        lt = orc.lifetimes_from_order(o)
        if lt is None:
            assert res.valid[i] == 0
            continue
        _, pr, ps = orc.timeline_from_lifetimes(lt[0], lt[1], g.n)
        assert res.valid[i] == 1 and (int(res.peak[i]), int(res.peak_step[i])) == (pr, ps), i
    assert (planner.resident_bytes_per_step(g, orders[0]) ==
            orc.resident_bytes_per_step(orders[0])).all()


@pytest.mark.parametrize("layers,smem,mode", [(3000, 1, ""), (20000, 0, ""), (20000, 0, "scratch"),
                                              (20000, 0, "scratch64"), (20000, 0, "widexf"),
                                              (20000, 0, "tiny8")])
def test_large_graph_variants(planner, monkeypatch, layers, smem, mode):
    """Graphs past the register-resident variant: node tables read per candidate,
    buffers in shared memory (n=12k); at n=80k the node-partitioned scorer
    (default), and the node-space kernel with global scratch and 32-bit (24-bit
    position) or 64-bit stamped position words, 4-bit shared / 8-bit / wide scan
    inputs."""
    if mode == "scratch":
        monkeypatch.setenv("MP_SCORE_NO_PARTS", "1")
    if mode == "scratch64":
        monkeypatch.setenv("MP_SCORE_POS64", "1")
    if mode == "widexf":   # training_like fits the packed scan inputs; force the wide ones
        monkeypatch.setenv("MP_SCORE_WIDE_XF", "1")
    if mode == "tiny8":    # ... or the byte-packed ones in global scratch (not the 4-bit smem ones)
        monkeypatch.setenv("MP_SCORE_NO_TINY4", "1")
    g = mp.generate_graph("training_like", layers, 8)
    dg = planner.upload(g)
    assert dg.info()["smem_resident"] == smem
    if not smem:
        assert dg.info()["score_variant"] == (5 if mode == "" else 4)   # MP_SCORER_PARTS / SCRATCH
    orc = O.Oracle.from_csr(g.csr())
    orders = np.concatenate([g.program_order()[None, :], mp.random_topo_orders(g, 4, seed=2)])
    bad = orders[1:3].copy()
    bad[0, [10, 20]] = bad[0, [20, 10]]
    bad[1, 3] = bad[1, 4]
    allo = np.concatenate([orders, bad])
    res = planner.score_orders(g, allo)
    assert res.valid.tolist() == [int(orc.is_topological_order(o)) for o in allo]
    assert res.valid[-1] == 0   # a duplicated node is never a permutation
    for i, o in enumerate(orders):
        rs = orc.resident_bytes_per_step(o)
        assert (int(res.peak[i]), int(res.peak_step[i])) == (int(rs.max()), int(np.argmax(rs)) + 1)


@pytest.mark.parametrize("variant", ["parts", "scratch"])
def test_global_scratch_stamp_wrap(planner, monkeypatch, variant):
    """One CTA scoring 300 candidates of an 80k-node graph: the 7-bit stamp of the
    32-bit position words (per candidate in the scratch scorer, per pass in the
    node-partitioned one) wraps several times and every verdict and peak must hold."""
    if variant == "scratch":
        monkeypatch.setenv("MP_SCORE_NO_PARTS", "1")
    monkeypatch.setenv("MP_SCORE_GRID", "1")
    g = mp.generate_graph("training_like", 20000, 8)
    orc = O.Oracle.from_csr(g.csr())
    orders = mp.random_topo_orders(g, 300, seed=11)
    for i in (5, 130, 131, 290):          # invalid rows across the wraps
        orders[i, [7, 8 + i]] = orders[i, [8 + i, 7]]
    orders[200, 3] = orders[200, 4]
    res = planner.score_orders(g, orders)
    assert res.valid.tolist() == [int(orc.is_topological_order(o)) for o in orders]
    for i in (0, 129, 257, 299):          # exact peaks on a few rows (O(sum of lifetimes) each)
        if res.valid[i]:
            rs = orc.resident_bytes_per_step(orders[i])
            assert (int(res.peak[i]), int(res.peak_step[i])) == (int(rs.max()), int(np.argmax(rs)) + 1), i
    monkeypatch.delenv("MP_SCORE_GRID")    # full grid (no wrap) must agree row for row
    full = planner.score_orders(g, orders)
    assert (full.peak == res.peak).all() and (full.peak_step == res.peak_step).all()
    assert (full.valid == res.valid).all()


@pytest.mark.parametrize("kind,layers,chunks", [("training_like", 300, 2), ("training_like", 200, 1),
                                                ("training_like", 1000, 6), ("chain", 3000, 4),
                                                ("training_like", 40, 1), ("training_like", 40, 0),
                                                # 2-7 parts, n % 4 == 0: the deferred lists
                                                ("training_like", 300, 8), ("training_like", 1000, 20),
                                                ("training_like", 2000, 63)])
def test_node_partitioned_scorer_small(planner, monkeypatch, kind, layers, chunks):
    """The node-partitioned scorer forced onto small graphs with tiny parts
    (MP_PARTS_CHUNKS 64-node chunks per part, 0 = no cap): many passes, validity pairs and
    multi-consumer tensors across parts through stash slots, n not a multiple of
    4 (scalar order loads) and of 256 (padding slots); valid, swapped,
    duplicated and out-of-range candidates vs the C restatement."""
    monkeypatch.setenv("MP_SCORE_PARTS", "1")
    monkeypatch.setenv("MP_PARTS_CHUNKS", str(chunks))
    g = mp.generate_graph(kind, layers, 8)
    info = mp.planner.parts_plan_info(g, max_chunks=chunks)
    assert info["parts"] >= 1 and info["tiny4"] == 1
    dg = planner.upload(g)
    assert dg.info()["score_variant"] == 5
    orc = O.Oracle.from_csr(g.csr())
    orders = np.concatenate([g.program_order()[None, :], mp.random_topo_orders(g, 40, seed=4)])
    orders[3, [1, 2]] = orders[3, [2, 1]]
    orders[7, 4] = orders[7, 9]
    orders[9, 0] = g.n
    orders[11, -1] = -5
    res = planner.score_orders(g, orders)
    for i, o in enumerate(orders):
        lt = orc.lifetimes_from_order(o)
        if lt is None:
            assert res.valid[i] == 0, i
            continue
        pr, ps = O.timeline_peak(lt[0], lt[1], g.edge_size, g.n)
        assert res.valid[i] == 1 and (int(res.peak[i]), int(res.peak_step[i])) == (pr, ps), i
    _, best = planner.score_orders_best(g, orders)
    ok = [i for i in range(len(orders)) if res.valid[i]]
    assert best == min(ok, key=lambda i: (int(res.peak[i]), i))


@pytest.mark.parametrize("chunks", [2, 5, 0])
def test_node_partitioned_scorer_sink_counts(planner, monkeypatch, chunks):
    """The partitioned scorer's three multi-consumer record kinds: 2-sink tensors (8-byte
    records), 3- and 4-sink tensors (16-byte records) and 5-sink ones (stash max), inside
    one part and across parts, vs the C restatement."""
    monkeypatch.setenv("MP_SCORE_PARTS", "1")
    monkeypatch.setenv("MP_PARTS_CHUNKS", str(chunks))
    nodes, edges, prev = [("s0", "source")], [], "s0"
    for gi in range(300):
        width = 2 + gi % 4 if gi % 7 else 5
        branch = [f"b{gi}_{k}" for k in range(width)]
        nodes += [(b, "compute") for b in branch] + [(f"j{gi}", "compute")]
        edges.append((f"x{gi}", prev, branch, 1 + gi % 3))
        edges += [(f"y{gi}_{k}", branch[k], [f"j{gi}"], 1) for k in range(width)]
        prev = f"j{gi}"
    g = mp.graph_from_lists(nodes, edges)
    info = mp.planner.parts_plan_info(g, max_chunks=chunks)
    assert info["parts"] >= 1 and info["tiny4"] == 1
    assert planner.upload(g).info()["score_variant"] == 5
    orc = O.Oracle.from_csr(g.csr())
    orders = mp.random_topo_orders(g, 64, seed=5)
    orders[2, [3, 4]] = orders[2, [4, 3]]
    orders[6, 10] = orders[6, 11]
    res = planner.score_orders(g, orders)
    for i, o in enumerate(orders):
        lt = orc.lifetimes_from_order(o)
        if lt is None:
            assert res.valid[i] == 0, i
            continue
        pr, ps = O.timeline_peak(lt[0], lt[1], g.edge_size, g.n)
        assert res.valid[i] == 1 and (int(res.peak[i]), int(res.peak_step[i])) == (pr, ps), i


@pytest.mark.parametrize("size", [8, 1 << 20])
def test_large_graph_wide_dynamic_edges(planner, size, monkeypatch):
    """>65,536 nodes whose order-dependent frees have 6 mutually unordered candidate
    sinks (past the 4-sink table: the flat loop), with 4-bit (sizes 8 and 3, gcd 1)
    and wide (2^20 and 3) scan inputs, valid and invalid rows, vs the oracle."""
    groups = 10000
    nodes, edges = [("s0", "source")], []
    prev = "s0"
    for g in range(groups):
        branch = [f"b{g}_{k}" for k in range(6)]
        nodes += [(b, "compute") for b in branch] + [(f"j{g}", "compute")]
        edges.append((f"x{g}", prev, branch, size))                    # 6 candidate last sinks
        edges += [(f"y{g}_{k}", branch[k], [f"j{g}"], 3) for k in range(6)]
        prev = f"j{g}"
    g = mp.graph_from_lists(nodes, edges)
    assert g.n > 65536
    orc = O.Oracle.from_csr(g.csr())
    orders = mp.random_topo_orders(g, 4, seed=9)
    orders[3, [5, 6]] = orders[3, [6, 5]]
    res = planner.score_orders(g, orders)
    for i, o in enumerate(orders):
        if not orc.is_topological_order(o):
            assert res.valid[i] == 0
            continue
        rs = orc.resident_bytes_per_step(o)
        assert res.valid[i] == 1
        assert (int(res.peak[i]), int(res.peak_step[i])) == (int(rs.max()), int(np.argmax(rs)) + 1)


def test_c5_full_size(golden, planner):
    """The 100k-tensor graph at full size: KAT peak + size-independent properties."""
    g = mp.generate_graph("training_like", 33333, 8)
    k = golden["kats"]["training_like_L33333"]
    po = g.program_order()
    assert planner.peak_resident_bytes(g, po) == k["program_peak"]
    orders = mp.random_topo_orders(g, 3, seed=7)
    res = planner.score_orders(g, np.concatenate([po[None, :], orders]))
    assert res.valid.all() and int(res.peak[0]) == k["program_peak"]
    orc = O.Oracle.from_csr(g.csr())
    lo, hi = orc.lifetimes_from_order(orders[0])
    glo, ghi = planner.lifetimes_from_order(g, orders[0])
    assert (glo == lo).all() and (ghi == hi).all()
    # resident bytes: sum over steps = sum of size * lifetime length (a checksum)
    rs = planner.resident_bytes_per_step(g, orders[0])
    assert int(rs.sum(dtype=np.uint64)) == int(
        (g.edge_size * (hi - lo + 1).astype(np.uint64)).sum(dtype=np.uint64))
    assert int(rs.max()) == int(res.peak[1]) and int(np.argmax(rs)) + 1 == int(res.peak_step[1])
    # overlap pairs at full size: exact per-row counts and hashes on sampled rows
    import torch
    cnt = planner.encode_address_pairs(g, lo, hi, want_pairs=False)
    total_c, _ = O.overlap_row_stats(lo, hi, g.edge_size)
    assert cnt == int(total_c.sum())
    d = torch.device("cuda:0")
    dlo, dhi = torch.from_numpy(lo).to(d), torch.from_numpy(hi).to(d)
    dsz = torch.from_numpy(g.edge_size.view(np.int64)).to(d)
    for r in np.linspace(0, g.E - 1, 48).astype(np.int64).tolist():
        c, h = O.overlap_row_stats(lo, hi, g.edge_size, rows=(r, r + 1))
        off = torch.zeros(2, dtype=torch.int64, device=d)
        k = planner.overlap_pairs_d(g.E, dlo, dhi, dsz, None, r, r + 1, off, None, 0)
        assert k == int(c[0])
        out = torch.zeros((max(k, 1), 2), dtype=torch.int32, device=d)
        planner.overlap_pairs_d(g.E, dlo, dhi, dsz, None, r, r + 1, off, out, k)
        got = out[:k].cpu().numpy()
        j = np.arange(r + 1, g.E)
        exp = j[(g.edge_size[j] > 0) & (lo[j] <= hi[r]) & (lo[r] <= hi[j])]
        assert (got[:, 0] == r).all()
        assert got[:, 1].tolist() == exp.tolist(), r
        hsh = np.uint64(1469598103934665603)
        with np.errstate(over="ignore"):
            for x in exp.astype(np.uint64):               # FNV-1a pins exp to the C oracle
                hsh = (hsh ^ x) * np.uint64(1099511628211)
        assert int(hsh) == int(h[0])


def test_pairs_row_sharding_concatenates(planner):
    """Row-range shards (multi-GPU partitioning) concatenate to the full list."""
    import torch
    g = mp.generate_graph("fork_join", 300, 50, 4)
    lo, hi = planner.lifetimes_from_order(g, mp.random_topo_orders(g, 1, seed=3)[0])
    full = planner.encode_address_pairs(g, lo, hi)
    d = torch.device("cuda:0")
    dlo, dhi = torch.from_numpy(lo).to(d), torch.from_numpy(hi).to(d)
    dsz = torch.from_numpy(g.edge_size.view(np.int64)).to(d)
    parts = []
    bounds = [0, 17, 400, g.E // 2, g.E]
    for r0, r1 in zip(bounds[:-1], bounds[1:]):
        off = torch.zeros(r1 - r0 + 1, dtype=torch.int64, device=d)
        cnt = planner.overlap_pairs_d(g.E, dlo, dhi, dsz, None, r0, r1, off, None, 0)
        out = torch.zeros((max(cnt, 1), 2), dtype=torch.int32, device=d)
        cnt2 = planner.overlap_pairs_d(g.E, dlo, dhi, dsz, None, r0, r1, off, out, cnt)
        torch.cuda.synchronize()
        assert cnt2 == cnt
        parts.append(out[:cnt].cpu().numpy())
    assert (np.concatenate(parts) == full).all()


def test_sharded_pairs_and_conflicts_device(planner):
    """dist.sharded_overlap_pairs / sharded_conflicts with the K2 / K4 device shard
    functions: one process (no collective), and the 3-rank balanced row ranges
    concatenated, both equal the serial lists."""
    import torch
    from paper_2210_12924_b200 import dist as D
    g = mp.generate_graph("fork_join", 300, 50, 4)
    lo, hi = planner.lifetimes_from_order(g, mp.random_topo_orders(g, 1, seed=3)[0])
    full = planner.encode_address_pairs(g, lo, hi)
    rng = np.random.default_rng(1)
    has = (rng.random(g.E) > 0.1).astype(np.uint8)
    addr = rng.integers(0, 1 << 12, g.E).astype(np.uint64)
    viol = O.validate_pairs(lo, hi, g.edge_size, has, addr)
    assert len(viol) > 0
    d = torch.device("cuda:0")
    dlo, dhi = torch.from_numpy(lo).to(d), torch.from_numpy(hi).to(d)
    dsz = torch.from_numpy(g.edge_size.view(np.int64)).to(d)
    dhas = torch.from_numpy(has).to(d)
    dad = torch.from_numpy(addr.view(np.int64)).to(d)
    pf = lambda a, b: planner.overlap_pairs_rows_d(dlo, dhi, dsz, None, a, b)   # noqa: E731
    vf = lambda a, b: planner.conflicting_pairs_rows_d(dlo, dhi, dsz, dhas, dad, a, b)  # noqa: E731
    pairs, off, total = D.sharded_overlap_pairs(pf, g.E, device=d)
    assert off == 0 and total == len(full) and (pairs.cpu().numpy() == full).all()
    nv, allv = D.sharded_conflicts(vf, g.E, device=d)
    assert nv == len(viol) and (allv == viol).all()
    ranges = D.balanced_row_ranges(D.triangular_row_work(g.E), 3)
    assert (np.concatenate([pf(a, b).cpu().numpy() for a, b in ranges]) == full).all()
    assert (np.concatenate([vf(a, b).cpu().numpy() for a, b in ranges]) == viol).all()


def test_validation_vs_oracle_random(planner):
    g = mp.generate_graph("fork_join", 800, 1000, 5)
    o = mp.random_topo_orders(g, 1, seed=11)[0]
    lo, hi = planner.lifetimes_from_order(g, o)
    rng = np.random.default_rng(0)
    addr = rng.integers(0, 50_000, g.E).astype(np.uint64)
    has = (rng.random(g.E) < 0.9).astype(np.uint8)
    got = planner.conflicting_pairs(lo, hi, g.edge_size, has, addr)
    exp = O.validate_pairs(lo, hi, g.edge_size, has, addr)
    assert got.shape == exp.shape and (got == exp).all() and len(exp) > 0
    placed = {e: int(addr[e]) for e in range(g.E) if has[e]}
    assert planner.addresses_feasible(g, lo, hi, placed) == O.addresses_feasible(
        lo, hi, g.edge_size, has, addr)
    assert planner.peak_mem(g, placed) == O.peak_mem(g.edge_size, has, addr)


def test_device_scoring_and_argmin_key(planner):
    import torch
    g = mp.generate_graph("fork_join", 200, 300, 1)
    orders = mp.random_topo_orders(g, 1000, seed=4)
    orders[5, 0], orders[5, 1] = orders[5, 1], orders[5, 0]
    host = planner.score_orders(g, orders)
    d = torch.device("cuda:0")
    dg = planner.upload(g)
    t_orders = torch.from_numpy(orders).to(d)
    peak = torch.zeros(1000, dtype=torch.int64, device=d)
    step = torch.zeros(1000, dtype=torch.int32, device=d)
    valid = torch.zeros(1000, dtype=torch.uint8, device=d)
    out3 = torch.zeros(3, dtype=torch.int64, device=d)
    s = torch.cuda.current_stream().cuda_stream
    planner.score_orders_d(dg, t_orders, 1000, peak, step, valid, s)
    planner.argmin_key_d(peak, valid, 1000, 5000, out3, s)
    torch.cuda.synchronize()
    assert (peak.cpu().numpy().view(np.uint64) == host.peak).all()
    assert (step.cpu().numpy() == host.peak_step).all()
    assert (valid.cpu().numpy() == host.valid).all()
    best = host.argmin()
    o3 = out3.cpu().numpy().view(np.uint64)
    assert int(o3[0]) == best + 5000 and int(o3[1]) == int(host.peak[best])
    assert int(o3[2]) == (int(host.peak[best]) << 20) | (best + 5000)
    key = torch.zeros(2, dtype=torch.int64, device=d)
    planner.key_reset_d(key, s)                                  # {MP_KEY_NONE, no overflow}
    planner.score_orders_argmin_d(dg, t_orders, 1000, peak, step, valid, key, 5000, s)
    torch.cuda.synchronize()
    assert key.tolist() == [int(o3[2]), D.NO_KEY]


def test_host_scoring_pipeline_chunks(planner):
    """mp_score_orders_best with >= 4 MiB of orders runs the chunked H2D/score
    pipeline (up to 8 chunks, per-chunk index base): results and the fused
    first-minimum equal the device-buffer path, ties across chunks included."""
    import torch
    g = mp.generate_graph("fork_join", 300, 300, 5)
    C = max(64, (20 << 20) // (4 * g.n))            # ~20 MiB of orders -> 8 chunks
    orders = mp.random_topo_orders(g, C, seed=11)
    orders[C - 1] = orders[C // 2]                  # tie: the earlier index must win
    orders[7, [0, 1]] = orders[7, [1, 0]]
    res, best = planner.score_orders_best(g, orders)
    d = torch.device("cuda:0")
    dg = planner.upload(g)
    peak = torch.zeros(C, dtype=torch.int64, device=d)
    step = torch.zeros(C, dtype=torch.int32, device=d)
    valid = torch.zeros(C, dtype=torch.uint8, device=d)
    planner.score_orders_d(dg, torch.from_numpy(orders).to(d), C, peak, step, valid,
                           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert (res.peak == peak.cpu().numpy().view(np.uint64)).all()
    assert (res.peak_step == step.cpu().numpy()).all()
    assert (res.valid == valid.cpu().numpy()).all() and res.valid[7] == 0
    assert best == planner.argmin(res.peak, res.valid) and best != C - 1
    pin = torch.from_numpy(orders).pin_memory()
    hp = torch.zeros(C, dtype=torch.int64).pin_memory()
    hs = torch.zeros(C, dtype=torch.int32).pin_memory()
    hv = torch.zeros(C, dtype=torch.uint8).pin_memory()
    assert planner.score_orders_into(dg, pin.numpy(), hp, hs, hv) == best
    assert (hp.numpy().view(np.uint64) == res.peak).all() and (hv.numpy() == res.valid).all()


def test_sizes_near_the_total_cap(planner):
    """Byte sizes whose total approaches the reference's 2^62 cap (graph.cpp:122-128):
    64-bit scan, peaks past the packed key's 2^43 (the host argmin falls back to the
    device reduction; the device key pair raises its overflow flag), and the arena and
    placement paths with 64-bit sizes - all equal to the C restatement."""
    import json
    import torch
    rng = np.random.default_rng(7)
    n = 40
    nodes = [{"id": f"v{i}"} for i in range(n)]
    edges = []
    for i in range(1, n):
        for j in rng.choice(i, size=min(i, 2), replace=False):
            edges.append({"id": f"e{len(edges)}", "source": f"v{j}", "sinks": [f"v{i}"],
                          "size": int(rng.integers(1 << 52, 1 << 55)) | 1})
    g = mp.load_graph(json.dumps({"nodes": nodes, "edges": edges}))
    total = sum(int(x) for x in g.edge_size)
    assert (1 << 60) < total < (1 << 62)
    orc = O.Oracle.from_csr(g.csr())
    orders = mp.random_topo_orders(g, 300, seed=3)
    orders[4, [0, 1]] = orders[4, [1, 0]]
    res, best = planner.score_orders_best(g, orders)
    peaks = []
    for i, o in enumerate(orders):
        lt = orc.lifetimes_from_order(o)
        if lt is None:
            assert res.valid[i] == 0
            peaks.append(None)
            continue
        _, pr, ps = orc.timeline_from_lifetimes(lt[0], lt[1], g.n)
        assert (int(res.peak[i]), int(res.peak_step[i])) == (pr, ps), i
        peaks.append(pr)
    exp = min((p, i) for i, p in enumerate(peaks) if p is not None)[1]
    assert best == exp and int(res.peak[best]) >= (1 << 43)
    d = torch.device("cuda:0")
    dg = planner.upload(g)
    key = torch.zeros(2, dtype=torch.int64, device=d)
    z = [torch.zeros(300, dtype=t, device=d) for t in (torch.int64, torch.int32, torch.uint8)]
    planner.key_reset_d(key, torch.cuda.current_stream().cuda_stream)
    planner.score_orders_argmin_d(dg, torch.from_numpy(orders).to(d), 300, *z, key, 0,
                                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert key.tolist()[1] == 0                        # overflow flag: use the fallback
    with pytest.raises(OverflowError):
        D.check_device_key(key.tolist())
    mr, rs, fr, valid = planner.run_baseline_batch(g, orders[:20])
    for i in range(20):
        e = orc.run_baseline(orders[i])
        assert (e is None and valid[i] == 0) or (int(mr[i]), int(rs[i]), float(fr[i])) == e
    lo, hi = planner.lifetimes_from_order(g, orders[0])
    tk, ta, _ = O.preallocate_pyramid(lo, hi, g.edge_size, g.id_rank()[:g.E])
    ea, eh = O.greedy_pack(lo, hi, g.edge_size, tk, ta)
    ga, gh, _, _ = planner.place_batch(g, lo[None], hi[None], pyramid=True)
    assert (gh[0] == eh).all() and (ga[0][eh == 1] == ea[eh == 1]).all()


def test_packed_orders_keep_out_of_range_ids_invalid(planner):
    """The host call sends orders as uint16 for register-slot graphs: ids outside
    [0, n) - negative, >= 65535, or in [n, 65535) - must still make the candidate
    invalid (graph.cpp:241-248), and the rest must score as with int32 orders."""
    g = mp.generate_graph("fork_join", 60, 100, 3)
    dg = planner.upload(g)
    assert dg.info()["orders16"] == 1
    orders = mp.random_topo_orders(g, 40, seed=1)
    bad_vals = {3: -5, 7: 70000, 11: 65535, 13: 65534, 17: g.n, 19: (1 << 31) - 1, 23: -(1 << 31)}
    for r, v in bad_vals.items():
        orders[r, r % g.n] = v
    res = planner.score_orders(g, orders)
    orc = O.Oracle.from_csr(g.csr())
    for i, o in enumerate(orders):
        if i in bad_vals:
            assert res.valid[i] == 0, i
            continue
        lt = orc.lifetimes_from_order(o)
        _, pr, ps = orc.timeline_from_lifetimes(lt[0], lt[1], g.n)
        assert res.valid[i] == 1 and (int(res.peak[i]), int(res.peak_step[i])) == (pr, ps), i


def test_edge_cases(planner):
    empty = mp.load_graph('{"nodes": [], "edges": []}')
    assert planner.peak_resident_bytes(empty, []) == 0
    assert planner.resident_bytes_per_step(empty, []).tolist() == []
    t = planner.timeline_from_lifetimes(empty, [], [], 0)
    assert (t.peak_rs, t.peak_step) == (0, 0)
    with pytest.raises(errors.InvalidOrder):
        planner.lifetimes_from_order(empty, [0])
    solo = mp.load_graph('{"nodes": [{"id": "a"}], "edges": []}')
    res = planner.score_orders(solo, np.array([[0], [1], [-1]], np.int32))
    assert res.valid.tolist() == [1, 0, 0] and res.peak_step.tolist() == [1, 0, 0]
    t = planner.timeline_from_lifetimes(solo, [], [], 4)
    assert t.bytes.tolist() == [0, 0, 0, 0] and (t.peak_rs, t.peak_step) == (0, 1)
    g = mp.generate_graph("chain", 5, 3)
    res = planner.score_orders(g, np.zeros((3, 4), np.int32))   # wrong length
    assert res.valid.tolist() == [0, 0, 0]
    assert planner.encode_address_pairs(g, [1, 1], [0, 0]).shape == (0, 2)
    assert planner.argmin(np.array([5, 3, 3], np.uint64), np.array([1, 0, 1], np.uint8)) == 2
    assert planner.argmin(np.array([5], np.uint64), np.array([0], np.uint8)) == -1


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_multi_device_scoring(devices):
    """mp_score_orders_multi: contiguous shards on several contexts (repeated device
    0 here: one GPU on the box) with host threads - through ONE NCCL allreduce(MIN)
    of the fused key for distinct devices ([0]: a one-rank communicator), the host
    combine for repeated ones - identical to one context and to a serial
    first-minimum scan."""
    import gzip
    import os
    path = os.path.join(os.path.dirname(__file__), "..", "workloads", "graphs",
                        "resnet50_b32.json.gz")
    with gzip.open(path, "rt") as f:
        g = mp.load_graph(f.read())
    orders = mp.random_topo_orders(g, 301, seed=17)
    orders[0, [0, 1]] = orders[0, [1, 0]]
    orders[150] = orders[77]          # a tie across shards: the lower index must win
    mpl = mp.MultiPlanner(devices)
    assert mpl.nccl == (len(set(devices)) == len(devices))
    mpl.upload(g)
    res, best = mpl.score_orders(orders)
    p = mp.Planner(0)
    ref = p.score_orders(g, orders)
    assert (res.peak == ref.peak).all() and (res.peak_step == ref.peak_step).all()
    assert (res.valid == ref.valid).all()
    ok = np.nonzero(ref.valid)[0]
    exp = int(ok[np.argmin(ref.peak[ok])])      # first minimum
    assert best == exp
    mpl.close()
    p.close()


def test_pairs_and_lp_on_multi_node_schedules(planner):
    """The drop-in site place_external (pipeline.cpp:119) feeds encode_addresses with
    lifetimes realized from decode_sequence's multi-node-per-step schedules: GPU
    realized lifetimes -> K2 pair list -> K7 LP text against the reference's own
    realized_lifetimes + encode_addresses (filter on) + write_lp."""
    from schedules import multi_node_schedules
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(1)
    for kind, layers, seed in (("training_like", 10, 0), ("fork_join", 14, 2)):
        g = mp.generate_graph(kind, layers, 8, seed)
        rg = O.RefGraph.load(mp.save_graph(g))
        for o in mp.random_topo_orders(g, 2, seed=seed + 7):
            for name, ts, horizon in multi_node_schedules(g, o, rng):
                lo, hi = planner.realized_lifetimes(g, ts, horizon)
                rlo, rhi = rg.realized_lifetimes(ts, horizon)
                assert (lo == rlo).all() and (hi == rhi).all(), name
                ref = rg.encode_address_pairs(rlo, rhi, filter_pairs=True)
                got = planner.encode_address_pairs(g, lo, hi)
                assert got.shape == ref.shape and (got == ref).all(), name
                assert planner.encode_addresses_lp(g, lo, hi) == rg.encode_addresses_lp(rlo, rhi)


@pytest.mark.parametrize("name", ["resnet50_b32", "bert_base_s512", "gpt2_medium_s1024"])
def test_model_graphs_vs_reference(planner, name):
    """C2/C3/C4 graphs scored against the compiled reference itself (oracle/_ref:
    memplan::peak_resident_bytes and its InvalidOrder verdict) on 512 candidates,
    the batch first-minimum included; peak steps against the restatement."""
    import gzip
    import os
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    path = os.path.join(os.path.dirname(__file__), "..", "workloads", "graphs", name + ".json.gz")
    with gzip.open(path, "rt") as f:
        text = f.read()
    g = mp.load_graph(text)
    rg = O.RefGraph.load(text)
    orders = mp.random_topo_orders(g, 512, seed=29)
    orders[10, [2, 3]] = orders[10, [3, 2]]
    orders[20, 4] = orders[20, 5]
    res, best = planner.score_orders_best(g, orders)
    rp, rv, rbest = rg.score_orders(orders, threads=os.cpu_count() or 1)
    assert (res.valid == rv).all() and (res.peak == rp).all() and best == rbest
    for i in range(0, 512, 37):
        if rv[i]:
            lo, hi = rg.lifetimes_from_order(orders[i])
            assert O.timeline_peak(lo, hi, g.edge_size, g.n) == (int(res.peak[i]),
                                                                  int(res.peak_step[i]))


def test_c5_random_orders_vs_reference(planner):
    """The 100k-tensor graph: 16 random candidates' peaks and verdicts against the
    compiled reference (memplan::peak_resident_bytes on all host threads) and the
    peak steps against the restatement (replaces a GPU-vs-GPU comparison)."""
    import os
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    g = mp.generate_graph("training_like", 33333, 8)
    rg = O.RefGraph.generate("training_like", 33333, 8)
    orders = mp.random_topo_orders(g, 16, seed=41)
    orders[3, 100] = orders[3, 200]                   # a duplicated node: not a permutation
    res = planner.score_orders(g, orders)
    rp, rv, _ = rg.score_orders(orders, threads=os.cpu_count() or 1)
    assert (res.valid == rv).all() and (res.peak == rp).all() and rv[3] == 0
    for i in (0, 7, 15):
        lo, hi = rg.lifetimes_from_order(orders[i])
        assert O.timeline_peak(lo, hi, g.edge_size, g.n) == (int(res.peak[i]), int(res.peak_step[i]))


@pytest.mark.parametrize("pack24", [True, False])
def test_host_scoring_24bit_wire(planner, monkeypatch, pack24):
    """Host-buffer scoring of a node-partitioned graph with the 3-byte wire format
    (MP_PACK24, opt-in) and without: out-of-range / negative ids stay invalid, and
    results equal the device-buffer path row for row."""
    import torch
    if pack24:
        monkeypatch.setenv("MP_PACK24", "1")
    g = mp.generate_graph("training_like", 20000, 8)       # n = 80,004 (n % 4 == 0)
    dg = planner.upload(g)
    assert dg.info()["score_variant"] == 5
    assert dg.info()["orders16"] == (2 if pack24 else 0)
    orders = mp.random_topo_orders(g, 40, seed=23)
    orders[1, 7] = g.n
    orders[2, 9] = -1
    orders[3, 11] = (1 << 24) + 5                      # wraps to a valid id if truncated
    orders[4, [5, 6]] = orders[4, [6, 5]]
    res, best = planner.score_orders_best(g, orders)
    d = torch.device("cuda:0")
    z = [torch.zeros(40, dtype=t, device=d) for t in (torch.int64, torch.int32, torch.uint8)]
    planner.score_orders_d(dg, torch.from_numpy(orders).to(d), 40, *z,
                           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert (z[0].cpu().numpy().view(np.uint64) == res.peak).all()
    assert (z[1].cpu().numpy() == res.peak_step).all() and (z[2].cpu().numpy() == res.valid).all()
    assert res.valid[1:4].tolist() == [0, 0, 0]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,layers,size,seed,pinned", [
    ("fork_join", 300, 50, 4, False), ("fork_join", 1200, 8, 2, True),
    ("training_like", 900, 8, 0, False), ("training_like", 900, 8, 0, True)])
def test_pairs_sorted_tile_count(planner, monkeypatch, kind, layers, size, seed, pinned):
    """K2's count from sorted column tiles (used from 8,192 edges up, forced here with
    MP_PAIRS_SORTED) gives the same per-row totals, hence the same pair list, as the
    ballot sweep and the C restatement - full tiles, the diagonal tile, pinned rows,
    row shards - and the single-sync device call writes the first `cap` pairs and
    reports MP_E_CAPACITY when the total exceeds cap."""
    import torch
    g = mp.generate_graph(kind, layers, size, seed)
    lo, hi = planner.lifetimes_from_order(g, mp.random_topo_orders(g, 1, seed=seed + 7)[0])
    pin = None
    if pinned:
        rng = np.random.default_rng(seed)
        pin = {int(e): 0 for e in rng.choice(g.E, size=g.E // 3, replace=False)}
    monkeypatch.delenv("MP_PAIRS_SORTED", raising=False)
    ref = planner.encode_address_pairs(g, lo, hi, pin)
    monkeypatch.setenv("MP_PAIRS_SORTED", "1")
    got = planner.encode_address_pairs(g, lo, hi, pin)
    assert got.shape == ref.shape and (got == ref).all()
    if pin is None:
        assert (ref == O.overlap_pairs(lo, hi, g.edge_size)).all()
        d = torch.device("cuda:0")
        dlo, dhi = torch.from_numpy(lo).to(d), torch.from_numpy(hi).to(d)
        dsz = torch.from_numpy(g.edge_size.view(np.int64)).to(d)
        parts = []
        bounds = sorted({0, 5, g.E // 3, g.E // 2 + 3, g.E})
        for r0, r1 in zip(bounds[:-1], bounds[1:]):
            off = torch.zeros(r1 - r0 + 1, dtype=torch.int64, device=d)
            cnt = planner.overlap_pairs_d(g.E, dlo, dhi, dsz, None, r0, r1, off, None, 0)
            out = torch.zeros((max(cnt, 1), 2), dtype=torch.int32, device=d)
            assert planner.overlap_pairs_d(g.E, dlo, dhi, dsz, None, r0, r1, off, out, cnt) == cnt
            parts.append(out[:cnt].cpu().numpy())
        assert (np.concatenate(parts) == ref).all()
        off = torch.zeros(g.E + 1, dtype=torch.int64, device=d)
        cap = len(ref) // 2
        out = torch.full((cap, 2), -1, dtype=torch.int32, device=d)
        with pytest.raises(errors.Capacity):
            planner.overlap_pairs_d(g.E, dlo, dhi, dsz, None, 0, g.E, off, out, cap)
        assert (out.cpu().numpy() == ref[:cap]).all()


@pytest.mark.parametrize("name", ["gpt2_medium_s1024", "random_dag_wide"])
def test_mid32_scorer_matches_64bit(planner, monkeypatch, name):
    """Graphs whose totals pass 2^32 gcd units while every node's x fits int32 and
    f uint32 (C4) are scored with 32-bit scan inputs and 64-bit sums; the results
    equal the 64-bit kernel's (MP_SCORE_NO_MID) and the reference's, on the device
    and the host (16-bit wire) paths."""
    import gzip
    import os
    if name == "random_dag_wide":   # gcd 1, sizes up to 2^27: total past 2^32 units
        rng = np.random.default_rng(5)
        n, src, off, sinks, size = 900, [], [0], [], []
        for u in range(n - 1):
            for _ in range(int(rng.integers(1, 3))):
                src.append(u)
                sinks.extend(sorted(set(int(x) for x in rng.integers(u + 1, min(n, u + 30),
                                                                      size=int(rng.integers(1, 4))))))
                off.append(len(sinks))
                size.append(int(rng.integers(1, 1 << 27)))
        g = mp.Graph.from_csr(n, src, off, sinks, size)
        text = mp.save_graph(g)
    else:
        path = os.path.join(os.path.dirname(__file__), "..", "workloads", "graphs",
                            name + ".json.gz")
        with gzip.open(path, "rt") as f:
            text = f.read()
        g = mp.load_graph(text)
    info = mp.planner.prep_info(g)
    assert info["narrow"] == 0 and info["mid32"] == 1
    orders = mp.random_topo_orders(g, 300, seed=31)
    orders[7, [1, 2]] = orders[7, [2, 1]]
    monkeypatch.delenv("MP_SCORE_NO_MID", raising=False)
    mid, best_mid = planner.score_orders_best(g, orders)
    mid_d = planner.score_orders(g, orders)
    monkeypatch.setenv("MP_SCORE_NO_MID", "1")
    wide, best_wide = planner.score_orders_best(g, orders)
    for a in (mid, mid_d):
        assert (a.valid == wide.valid).all() and (a.peak == wide.peak).all()
        assert (a.peak_step == wide.peak_step).all()
    assert best_mid == best_wide
    if O.ref_available():
        rg = O.RefGraph.load(text)
        rp, rv, rbest = rg.score_orders(orders, threads=os.cpu_count() or 1)
        assert (mid.valid == rv).all() and (mid.peak == rp).all() and best_mid == rbest
