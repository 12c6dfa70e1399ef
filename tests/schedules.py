"""Multi-node-per-timestep schedules for the pair-set parity tests (test helper).

decode_sequence (proj/src/plan.cpp:28-77) turns an ILP assignment into a
sequence whose timesteps may hold several nodes, with nodes that feed nothing
placed at the horizon; place_external then calls encode_addresses on the
lifetimes realized from it (proj/src/pipeline.cpp:119). These generators build
such schedules from a topological order - every producer strictly before its
consumers, as decode_sequence guarantees - in three shapes: ASAP layering,
random delays, and ASAP with the tail nodes moved to the horizon."""
import numpy as np


def node_preds(g):
    preds = [[] for _ in range(g.n)]
    for e in range(g.E):
        for k in range(g.sink_off[e], g.sink_off[e + 1]):
            preds[g.sinks[k]].append(int(g.edge_src[e]))
    return preds


def multi_node_schedules(g, order, rng):
    """Yields (name, timestep_of int32[n], horizon) for one topological order."""
    preds = node_preds(g)
    has_consumer = np.zeros(g.n, bool)
    for e in range(g.E):
        if g.sink_off[e + 1] > g.sink_off[e]:
            has_consumer[g.edge_src[e]] = True
    for mode in ("asap", "jitter", "tail"):
        ts = np.zeros(g.n, np.int32)
        for v in order:
            t = max((ts[u] for u in preds[v]), default=0) + 1
            if mode == "jitter":
                t += int(rng.integers(0, 3))
            ts[v] = t
        h = int(ts.max()) if g.n else 0
        if mode == "tail":
            ts[~has_consumer] = h
        for horizon in (h, g.n):
            yield f"{mode}/h={horizon}", ts.copy(), horizon
