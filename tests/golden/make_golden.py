"""Generates tests/golden/golden.json from the UNMODIFIED reference planner.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The reference is compiled from its own sources by oracle/Makefile into
oracle/_ref/libmemplan_ref.so; every number below is what that library
returns. The fixture is committed so the GPU box (no /root/reference) and the
CPU test suite can check both the C restatement and the CUDA path against it.
"""
from __future__ import annotations

import itertools
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

FIXTURES = ["chain3", "order4", "pack3", "training_mini", "training_mini_ctrl"]
FIXTURE_DIR = "/root/reference/proj/fixtures"


def splitmix(seed):
    s = [seed & ((1 << 64) - 1)]

    def nxt():
        s[0] = (s[0] + 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        z = s[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & ((1 << 64) - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & ((1 << 64) - 1)
        return z ^ (z >> 31)
    return nxt


def random_topo(csr, rng):
    n = csr["n"]
    indeg = np.zeros(n, np.int64)
    succ = [[] for _ in range(n)]
    for e in range(len(csr["edge_src"])):
        for k in range(csr["sink_off"][e], csr["sink_off"][e + 1]):
            w = int(csr["sinks"][k])
            indeg[w] += 1
            succ[int(csr["edge_src"][e])].append(w)
    ready = [v for v in range(n) if indeg[v] == 0]
    out = []
    while ready:
        i = rng() % len(ready)
        v = ready[i]
        ready[i] = ready[-1]
        ready.pop()
        out.append(v)
        for w in succ[v]:
            indeg[w] -= 1
            if indeg[w] == 0:
                ready.append(w)
    return out


def program_order(g: "O.RefGraph"):
    o = list(range(g.n))
    if g.n == 0 or g.is_topological_order(o):
        return o
    return g.topological_order().tolist()


def invalid_variants(order, n):
    """Orders the reference rejects with InvalidOrder (or accepts: the verdict is recorded)."""
    out = []
    if n >= 2:
        sw = list(order)
        sw[0], sw[-1] = sw[-1], sw[0]
        out.append(sw)
        dup = list(order)
        dup[1] = dup[0]
        out.append(dup)
    out.append(list(order[:-1]) if n else [0])       # wrong length
    oor = list(order)
    if n:
        oor[n // 2] = n                              # out of range
    out.append(oor)
    if n:
        neg = list(order)
        neg[0] = -1
        out.append(neg)
    return out


def order_case(g: "O.RefGraph", order):
    c = {"order": [int(x) for x in order]}
    try:
        lo, hi = g.lifetimes_from_order(order)
    except O.RefError as e:
        c["error"] = str(e)
        return c
    c["lo"] = lo.tolist()
    c["hi"] = hi.tolist()
    c["bytes"] = [int(x) for x in g.resident_bytes_per_step(order)]
    c["peak"] = g.peak_resident_bytes(order)
    b, pr, ps = g.timeline_from_lifetimes(lo, hi, g.n)
    c["timeline"] = {"bytes": [int(x) for x in b], "peak_rs": pr, "peak_step": ps}
    c["pairs"] = g.encode_address_pairs(lo, hi, filter_pairs=True).tolist()
    c["pairs_unfiltered_count"] = g.encode_address_pairs(lo, hi, filter_pairs=False,
                                                         want_pairs=False)
    # placement heuristics (placement.cpp:25-62, 182-204) and the arena baseline (:150-180)
    taken, paddr, base = g.preallocate_pyramid(lo, hi)
    ga, gh = g.greedy_pack_fixed(lo, hi, taken, paddr)
    pa, ph = g.greedy_pack_fixed(lo, hi)
    c["placement"] = {"pyramid_taken": taken.tolist(), "pyramid_addr": [int(x) for x in paddr],
                      "pyramid_base": int(base),
                      "greedy_pyramid_addr": [int(x) for x in ga], "greedy_pyramid_has": gh.tolist(),
                      "greedy_addr": [int(x) for x in pa], "greedy_has": ph.tolist()}
    c["baseline"] = {"first_fit": list(g.run_baseline(order, best_fit=False)),
                     "best_fit": list(g.run_baseline(order, best_fit=True))}
    return c


def plan_cases(g: "O.RefGraph", order, rng):
    """Address plans over realized lifetimes: greedy_pack (valid) + tampered copies."""
    csr = g.csr()
    E = g.E
    lo, hi = g.lifetimes_from_order(order)
    addr = g.greedy_pack(lo, hi)
    size = csr["edge_size"]
    has = (size > 0).astype(np.uint8)
    ts = np.zeros(g.n, np.int32)
    ts[np.asarray(order)] = np.arange(1, g.n + 1)
    peak_mem = int(max([int(addr[e] + size[e]) for e in range(E) if size[e] > 0] or [0]))
    _, peak_rs, peak_step = g.timeline_from_lifetimes(lo, hi, g.n)
    cases = []

    def add(name, seq, ts_, has_, addr_, pm, prs):
        viol = g.validate_plan(seq, ts_, has_, addr_, pm, prs)
        cases.append({"name": name, "sequence": [int(x) for x in seq], "timestep_of": ts_.tolist(),
                      "has_addr": has_.tolist(), "addr": [int(x) for x in addr_], "peak_mem": pm,
                      "stored_peak_rs": prs, "violations": [list(v) for v in viol]})

    add("greedy", order, ts, has, addr, peak_mem, peak_rs)
    data = [e for e in range(E) if size[e] > 0]
    if len(data) >= 2:
        t = addr.copy()
        i, j = data[0], data[1 + rng() % (len(data) - 1)]
        t[j] = t[i]
        add("collide", order, ts, has, t, peak_mem, peak_rs)
        t = addr.copy()
        for e in data:
            t[e] = 0
        add("all_zero", order, ts, has, t, peak_mem, peak_rs)
    add("understated_peak", order, ts, has, addr, max(peak_mem - 1, 0), peak_rs)
    add("stored_peak_rs", order, ts, has, addr, peak_mem, peak_rs + 999)
    if data:
        h = has.copy()
        h[data[-1]] = 0
        add("missing_address", order, ts, h, addr, peak_mem, peak_rs)
    if g.n >= 2:
        t2 = ts.copy()
        t2[order[0]], t2[order[1]] = t2[order[1]], t2[order[0]]
        add("swapped_steps", order, t2, has, addr, peak_mem, peak_rs)
        t3 = ts.copy()
        t3[order[-1]] = 0
        add("missing_timestep", order[:-1], t3, has, addr, peak_mem, peak_rs)
        t4 = ts.copy()
        t4[order[-1]] = g.n + 3          # horizon extends past n
        add("long_horizon", order, t4, has, addr, peak_mem, peak_rs)
    return cases


def realized_cases(g: "O.RefGraph", order, rng):
    ts = np.zeros(g.n, np.int32)
    ts[np.asarray(order)] = np.arange(1, g.n + 1)
    out = []
    for horizon in (g.n, g.n + 5):
        lo, hi = g.realized_lifetimes(ts, horizon)
        out.append({"timestep_of": ts.tolist(), "horizon": horizon, "lo": lo.tolist(),
                    "hi": hi.tolist()})
    # arbitrary (non-topological) timesteps are allowed here
    ts2 = np.array([1 + rng() % max(g.n, 1) for _ in range(g.n)], np.int32)
    lo, hi = g.realized_lifetimes(ts2, g.n)
    out.append({"timestep_of": ts2.tolist(), "horizon": g.n, "lo": lo.tolist(), "hi": hi.tolist()})
    if g.n:
        ts3 = ts.copy()
        ts3[rng() % g.n] = 0
        try:
            lo, hi = g.realized_lifetimes(ts3, g.n)
            out.append({"timestep_of": ts3.tolist(), "horizon": g.n, "lo": lo.tolist(),
                        "hi": hi.tolist()})
        except O.RefError as e:
            out.append({"timestep_of": ts3.tolist(), "horizon": g.n, "error": str(e)})
    return out


def graph_record(name, g: "O.RefGraph", rng, n_random=3, plans=True):
    csr = g.csr()
    rec = {"name": name, "graph_json": g.save(),
           "csr": {"n": g.n, "edge_src": csr["edge_src"].tolist(),
                   "sink_off": csr["sink_off"].tolist(), "sinks": csr["sinks"].tolist(),
                   "edge_size": [int(x) for x in csr["edge_size"]]}}
    po = program_order(g)
    orders = [po] + [random_topo(csr, rng) for _ in range(n_random)]
    cases = [order_case(g, o) for o in orders]
    for o in invalid_variants(po, g.n):
        cases.append(order_case(g, o))
    rec["orders"] = cases
    # encode_joint's pair set (encode.cpp:401-408), filtered by edge_precedes and not
    rec["joint_pairs"] = {"filtered": g.joint_pairs(True).tolist(),
                          "all": len(g.joint_pairs(False))}
    # pinned (preplaced) pair sets on program order
    if g.n:
        lo, hi = g.lifetimes_from_order(po)
        pin = np.zeros(g.E, np.uint8)
        for e in range(g.E):
            if rng() % 3 == 0:
                pin[e] = 1
        rec["pinned"] = {"pinned": pin.tolist(),
                         "pairs": g.encode_address_pairs(lo, hi, pin, np.zeros(g.E, np.uint64)).tolist()}
        # the external-ILP placement model as LP text (encode.cpp:320-377, lp_format.cpp:88-121)
        paddr = np.array([1000 * e + 8 for e in range(g.E)], np.uint64)
        rec["lp"] = {"text": g.encode_addresses_lp(lo, hi), "pinned_addr": paddr.tolist(),
                     "text_pinned": g.encode_addresses_lp(lo, hi, pin, paddr)}
        if plans:
            rec["plans"] = plan_cases(g, po, rng)
        rec["realized"] = realized_cases(g, po, rng)
    return rec


def main():
    O.build()
    rng = splitmix(20221024)
    doc = {"source": "reference memplan (oracle/_ref/libmemplan_ref.so) via tests/golden/make_golden.py",
           "graphs": [], "battery": [], "plan_graph": {}, "kats": {}}
    for f in FIXTURES:
        g = O.RefGraph.load_file(os.path.join(FIXTURE_DIR, f + ".json"))
        doc["graphs"].append(graph_record(f, g, rng, n_random=4))
    for kind, layers, size, seed in [("chain", 1, 3, 0), ("chain", 7, 5, 0), ("fork_join", 1, 6, 2),
                                     ("fork_join", 3, 9, 7), ("fork_join", 6, 100, 11),
                                     ("training_like", 1, 8, 0), ("training_like", 2, 8, 0),
                                     ("training_like", 3, 8, 0), ("training_like", 4, 8, 0),
                                     ("training_like", 12, 1000, 0)]:
        g = O.RefGraph.generate(kind, layers, size, seed)
        doc["graphs"].append(graph_record(f"{kind}_L{layers}_s{size}_seed{seed}", g, rng))
    # a graph with control edges and sinkless outputs
    text = json.dumps({
        "nodes": [{"id": "a", "role": "source"}, {"id": "b"}, {"id": "c"}, {"id": "d"},
                  {"id": "e", "role": "sink_only"}],
        "edges": [{"id": "x", "source": "a", "sinks": ["b", "c"], "size": 5},
                  {"id": "y", "source": "b", "sinks": ["d"], "size": 3},
                  {"id": "z", "source": "c", "sinks": ["d", "e"], "size": 7},
                  {"id": "k", "source": "c", "sinks": ["b"], "size": 0, "kind": "control"},
                  {"id": "out", "source": "d", "sinks": [], "size": 2},
                  {"id": "keep", "source": "a", "sinks": [], "size": 11}]})
    g = O.RefGraph.load(text)
    doc["graphs"].append(graph_record("control_and_sinkless", g, rng, n_random=4))
    g = O.RefGraph.load(json.dumps({"nodes": [], "edges": []}))
    doc["graphs"].append(graph_record("empty", g, rng, n_random=0, plans=False))
    g = O.RefGraph.load(json.dumps({"nodes": [{"id": "solo"}], "edges": []}))
    doc["graphs"].append(graph_record("single_node", g, rng, n_random=0))

    # oracle battery (test_acceptance.cpp:69-88): enumerate_min_peak witnesses
    battery = []
    for seed in range(100):
        battery.append(("fork_join", 1, 6, seed))
    for seed in range(60):
        battery.append(("fork_join", 1, 9, 100 + seed))
    kept, seed = 0, 0
    while kept < 60 and seed < 1000:
        g = O.RefGraph.generate("fork_join", 2, 5, seed)
        if g.n <= 9:
            battery.append(("fork_join", 2, 5, seed))
            kept += 1
        seed += 1
    for layers in range(1, 9):
        for size in (3, 7, 11):
            battery.append(("chain", layers, size, 0))
    for size in (4, 8, 16):
        battery.append(("training_like", 1, size, 0))
    for kind, layers, size, seed in battery:
        g = O.RefGraph.generate(kind, layers, size, seed)
        mp, order = g.enumerate_min_peak()
        doc["battery"].append({"spec": [kind, layers, size, seed], "min_peak": mp,
                               "order": order.tolist()})
    for f in FIXTURES:
        g = O.RefGraph.load_file(os.path.join(FIXTURE_DIR, f + ".json"))
        mp, order = g.enumerate_min_peak()
        doc["battery"].append({"fixture": f, "min_peak": mp, "order": order.tolist()})

    g = O.RefGraph.load_file(os.path.join(FIXTURE_DIR, "chain3.json"))
    doc["plan_graph"]["chain3"] = json.loads(g.plan_graph())

    # frozen training_like program-order peaks (test_acceptance.cpp:235)
    for L in (2, 3, 4):
        g = O.RefGraph.generate("training_like", L, 8)
        doc["kats"][f"training_like_L{L}_program_peak"] = g.peak_resident_bytes(list(range(g.n)))
    # C5 shape: the 100k-tensor training_like graph, program-order peak only
    g = O.RefGraph.generate("training_like", 33333, 8)
    doc["kats"]["training_like_L33333"] = {"n": g.n, "E": g.E, "S": g.S,
                                           "program_peak": g.peak_resident_bytes(list(range(g.n)))}
    doc["kats"]["fragmentation"] = [[mr, rs, O.ref_fragmentation(mr, rs)]
                                    for mr, rs in [(0, 0), (10, 10), (10, 8), (7, 0),
                                                   (1 << 40, 12345)]]
    out = os.path.join(HERE, "golden.json")
    with open(out, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(out, os.path.getsize(out), "bytes;", len(doc["graphs"]), "graphs,",
          len(doc["battery"]), "battery entries")


if __name__ == "__main__":
    main()
