"""GPU: batched candidate PLANS (mp_score_plans_d) - plan_once's placement half
(proj/src/pipeline.cpp:236-285) per candidate order - against the C restatement
(pinned to the reference by tests/test_oracle_golden.py) and, on the traced
model graphs, the compiled reference itself (oracle/_ref): lifetimes_from_order,
preallocate_pyramid + greedy_pack, peak_mem, and the address check
(validate_plan's below_above pairs, plan.cpp:390-404) on the produced plans and
on tampered copies (mp_validate_plans_d)."""
import gzip
import os

import numpy as np
import pytest

import oracle as O
import paper_2210_12924_b200 as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _expected(g, orc, order, pyramid=True):
    lt = orc.lifetimes_from_order(order)
    if lt is None:
        return None
    lo, hi = lt
    if pyramid:
        tk, ta, _ = O.preallocate_pyramid(lo, hi, g.edge_size, g.id_rank()[:g.E])
        ea, eh = O.greedy_pack(lo, hi, g.edge_size, tk, ta)
    else:
        ea, eh = O.greedy_pack(lo, hi, g.edge_size)
    return lo, hi, ea, eh, O.peak_mem(g.edge_size, eh, ea), len(O.validate_pairs(lo, hi, g.edge_size, eh, ea))


@pytest.mark.parametrize("kind,layers,size,seed,pyramid", [
    ("fork_join", 30, 1000, 3, True), ("training_like", 20, 8, 0, True),
    ("training_like", 25, 1 << 33, 0, False), ("chain", 40, 8, 0, True)])
@pytest.mark.parametrize("k5", ["auto", "warp"])
def test_score_plans_matches_restatement(planner, monkeypatch, kind, layers, size, seed, pyramid,
                                         k5):
    if k5 == "warp":   # the warp-per-problem placement variant (default for big batches)
        monkeypatch.setenv("MP_PLACE_WARP", "1")
    g = mp.generate_graph(kind, layers, size, seed)
    orc = O.Oracle.from_csr(g.csr())
    orders = mp.random_topo_orders(g, 48, seed=seed + 1)
    orders[5, [0, 1]] = orders[5, [1, 0]]          # invalid rows get no plan
    orders[9, 2] = orders[9, 3]
    res, best = planner.score_plans(g, orders, pyramid=pyramid)
    sc = planner.score_orders(g, orders)
    assert (res["valid"] == sc.valid).all() and (res["peak_rs"] == sc.peak).all()
    feas = []
    for i, o in enumerate(orders):
        exp = _expected(g, orc, o, pyramid)
        if exp is None:
            assert res["valid"][i] == 0 and res["nviol"][i] == 0 and res["peak_mem"][i] == 0
            continue
        lo, hi, ea, eh, pm, nv = exp
        assert (res["has_addr"][i] == eh).all(), i
        assert (res["addr"][i][eh == 1] == ea[eh == 1]).all(), i
        assert int(res["peak_mem"][i]) == pm and int(res["nviol"][i]) == nv == 0, i
        assert int(res["peak_mem"][i]) >= int(res["peak_rs"][i])
        feas.append((pm, i))
    assert best == min(feas)[1]


@pytest.mark.parametrize("pyramid", [True, False])
def test_score_plans_past_shared_memory(planner, pyramid):
    """A graph past the shared-memory kernels (9,003 edges > 8,192): lifetimes per
    candidate (K1), K5's global-memory placement and each plan's address check by the
    K4 sweep, vs the C restatement; an invalid row gets no plan."""
    g = mp.generate_graph("training_like", 3000, 8)
    assert g.E > 8192
    orc = O.Oracle.from_csr(g.csr())
    orders = mp.random_topo_orders(g, 4, seed=13)
    orders[2, [0, 1]] = orders[2, [1, 0]]
    res, best = planner.score_plans(g, orders, pyramid=pyramid)
    feas = []
    for i, o in enumerate(orders):
        exp = _expected(g, orc, o, pyramid)
        if exp is None:
            assert res["valid"][i] == 0 and res["nviol"][i] == 0 and res["peak_mem"][i] == 0
            continue
        lo, hi, ea, eh, pm, nv = exp
        assert (res["has_addr"][i] == eh).all(), i
        assert (res["addr"][i][eh == 1] == ea[eh == 1]).all(), i
        assert int(res["peak_mem"][i]) == pm and int(res["nviol"][i]) == nv == 0, i
        feas.append((pm, i))
    assert best == min(feas)[1]


def test_validate_plans_counts_tampered_conflicts(planner):
    """Caller-supplied plans: a greedy plan (no conflict) and seeded tampered copies
    (addresses moved onto live neighbours) - counts equal the restatement's pair
    list, which tests/test_oracle_golden.py pins to the reference's validate_plan."""
    import torch
    g = mp.generate_graph("fork_join", 40, 1000, 5)
    orc = O.Oracle.from_csr(g.csr())
    orders = mp.random_topo_orders(g, 16, seed=2)
    rng = np.random.default_rng(0)
    E = g.E
    los, his, addrs, hass, exp = [], [], [], [], []
    for o in orders:
        lo, hi, ea, eh, _, _ = _expected(g, orc, o)
        a = ea.copy()
        for e in rng.choice(E, size=5, replace=False):
            a[e] = a[rng.integers(E)]                 # collide with another tensor's slot
        for addr in (ea, a):
            los.append(lo), his.append(hi), addrs.append(addr), hass.append(eh)
            exp.append(len(O.validate_pairs(lo, hi, g.edge_size, eh, addr)))
    d = torch.device("cuda:0")
    T = lambda x, dt: torch.from_numpy(np.ascontiguousarray(np.stack(x)).view(dt)).to(d)  # noqa: E731
    nv = torch.zeros(len(exp), dtype=torch.int32, device=d)
    planner.validate_plans_d(E, len(exp), T(los, np.int32), T(his, np.int32),
                             torch.from_numpy(g.edge_size.view(np.int64)).to(d),
                             T(hass, np.uint8), T(addrs, np.int64), None, nv,
                             torch.cuda.current_stream().cuda_stream)
    assert nv.cpu().tolist() == exp
    assert exp[0::2] == [0] * 16 and sum(exp[1::2]) > 0


@pytest.mark.parametrize("name", ["resnet50_b32", "bert_base_s512"])
def test_score_plans_model_graphs_vs_reference(planner, name):
    """C2/C3 traced graphs: 6 candidates per graph against the compiled reference
    (lifetimes_from_order, preallocate_pyramid, greedy_pack over the pyramid)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    with gzip.open(os.path.join(ROOT, "workloads", "graphs", name + ".json.gz"), "rt") as f:
        text = f.read()
    g = mp.load_graph(text)
    rg = O.RefGraph.load(text)
    orders = mp.random_topo_orders(g, 6, seed=17)
    res, best = planner.score_plans(g, orders)
    for i, o in enumerate(orders):
        lo, hi = rg.lifetimes_from_order(o)
        tk, ta, _ = rg.preallocate_pyramid(lo, hi)
        ea, eh = rg.greedy_pack_fixed(lo, hi, tk, ta)
        assert (res["has_addr"][i] == eh).all()
        assert (res["addr"][i][eh == 1] == ea[eh == 1]).all()
        pm = max(int(ea[e]) + int(g.edge_size[e]) for e in range(g.E) if eh[e])
        assert int(res["peak_mem"][i]) == pm and res["nviol"][i] == 0
