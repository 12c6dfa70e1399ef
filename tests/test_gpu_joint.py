"""GPU parity for the joint-mode pair set (K8, k_joint.cu): the pair loop of
encode_joint (encode.cpp:401-408) with the edge_precedes filter
(analysis.cpp:94-113), against the reference's own pair lists
(tests/golden/golden.json; oracle/_ref on the traced model graphs)."""
import gzip
import os

import numpy as np
import pytest

import oracle as O
import paper_2210_12924_b200 as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_golden_joint_pairs(golden, planner):
    for rec in golden["graphs"]:
        g = mp.load_graph(rec["graph_json"])
        got = planner.joint_pairs(g)
        assert got.tolist() == rec["joint_pairs"]["filtered"], rec["name"]
        assert len(planner.joint_pairs(g, filter_pairs=False)) == rec["joint_pairs"]["all"]


@pytest.mark.parametrize("name", ["resnet50_b32", "bert_base_s512"])
def test_joint_pairs_model_graphs(planner, name):
    with gzip.open(os.path.join(ROOT, "workloads", "graphs", name + ".json.gz"), "rt") as f:
        g = mp.load_graph(f.read())
    got = planner.joint_pairs(g)
    data = int((g.edge_size > 0).sum())
    assert 0 < len(got) <= data * (data - 1) // 2
    assert (got[:, 0] < got[:, 1]).all()
    if O.ref_available():
        assert np.array_equal(got, O.RefGraph.load(mp.save_graph(g)).joint_pairs())


def test_joint_pairs_past_32k_nodes(planner):
    """The joint tables past the old 32,768-node bound: 40,000 nodes (most of them
    isolated, so the reference's own pair loop stays cheap), edges spread over the
    whole id range; the pair list equals the compiled reference's and the C
    restatement's (descendant bitsets on the host, AR transposed on the device)."""
    rng = np.random.default_rng(11)
    n = 40000
    nodes = np.sort(rng.choice(n, size=2500, replace=False))
    src, off, sinks, size = [], [0], [], []
    for a in range(len(nodes) - 1):
        for _ in range(int(rng.integers(1, 3))):
            k = int(rng.integers(0, 4))
            hi = min(len(nodes), a + 1 + 40)
            ss = sorted(set(int(nodes[x]) for x in rng.integers(a + 1, hi, size=k)))
            src.append(int(nodes[a]))
            sinks.extend(ss)
            off.append(len(sinks))
            size.append(int(rng.integers(0, 3)) * 64)   # some control edges (size 0)
    g = mp.Graph.from_csr(n, src, off, sinks, size)
    got = planner.joint_pairs(g)
    assert len(got) > 0
    assert np.array_equal(got, O.Oracle.from_csr(g.csr()).joint_pairs())
    if O.ref_available():
        assert np.array_equal(got, O.RefGraph.load(mp.save_graph(g)).joint_pairs())
