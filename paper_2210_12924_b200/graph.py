"""Host-side graph model: the reference's memplan::Graph, flattened to CSR.

Mirrors proj/include/memplan/graph.hpp:25-127 and proj/src/graph.cpp:64-141
(validation order and error classes), the canonical JSON format of
proj/src/graph_io.cpp:60-142 and the generator families of
proj/src/generate.cpp:45-158 (the CSR itself comes from the native
``mp_generate_graph``; ids are attached here).

Graph construction is one-off host work; the device never sees ids. A graph is
uploaded once per device context (``Planner.upload``) and every hot-path call
takes integer node / edge indexes exactly as the reference does.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from enum import Enum
from typing import Iterable, Sequence

import numpy as np

from . import errors
from . import _native

BYTE_CAP = 1 << 62  # graph.cpp:122-128


class NodeRole(str, Enum):
    COMPUTE = "compute"
    WEIGHT_UPDATE = "weight_update"
    SOURCE = "source"
    SINK_ONLY = "sink_only"


class EdgeKind(str, Enum):
    DATA = "data"
    CONTROL = "control"


_ROLE_CODES = [NodeRole.COMPUTE, NodeRole.WEIGHT_UPDATE, NodeRole.SOURCE, NodeRole.SINK_ONLY]


@dataclass
class Node:
    id: str
    role: NodeRole = NodeRole.COMPUTE


@dataclass
class TensorEdge:
    id: str
    source: str
    sinks: list = field(default_factory=list)
    size: int = 0
    kind: EdgeKind = EdgeKind.DATA


class Graph:
    """Immutable DAG with the reference's indexing (node / edge declaration order)."""

    def __init__(self):
        self.node_ids: list[str] = []
        self.node_roles: list[NodeRole] = []
        self.edge_ids: list[str] = []
        self.edge_kinds: list[EdgeKind] = []
        self.n = 0
        self.E = 0
        self.edge_src = np.zeros(0, np.int32)
        self.sink_off = np.zeros(1, np.int64)
        self.sinks = np.zeros(0, np.int32)
        self.edge_size = np.zeros(0, np.uint64)
        self.total_bytes = 0
        self._node_index: dict[str, int] | None = None
        self._edge_index: dict[str, int] | None = None

    # ---- construction ------------------------------------------------------
    @classmethod
    def build(cls, nodes: Sequence[Node], edges: Sequence[TensorEdge]) -> "Graph":
        """Graph::build (graph.cpp:64-141), same checks in the same order."""
        g = cls()
        node_index: dict[str, int] = {}
        for v, nd in enumerate(nodes):
            if not nd.id:
                raise errors.InvalidStructure("node with empty id")
            if nd.id in node_index:
                raise errors.DuplicateId(f"node id '{nd.id}' declared twice")
            node_index[nd.id] = v
        edge_index: dict[str, int] = {}
        for e, te in enumerate(edges):
            if not te.id:
                raise errors.InvalidStructure("edge with empty id")
            if te.id in edge_index:
                raise errors.DuplicateId(f"edge id '{te.id}' declared twice")
            edge_index[te.id] = e
        src = np.zeros(len(edges), np.int32)
        off = np.zeros(len(edges) + 1, np.int64)
        sinks: list[int] = []
        size = np.zeros(len(edges), np.uint64)
        has_fanin = np.zeros(len(nodes), bool)
        for e, te in enumerate(edges):
            kind = EdgeKind(te.kind)
            if kind == EdgeKind.CONTROL and te.size != 0:
                raise errors.ControlEdgeWithSize(f"control edge '{te.id}' has size {te.size}")
            if kind == EdgeKind.DATA and te.size == 0:
                raise errors.InvalidStructure(f"data edge '{te.id}' has size 0")
            if te.source not in node_index:
                raise errors.DanglingEndpoint(
                    f"edge '{te.id}' has unknown source '{te.source}'")
            src[e] = node_index[te.source]
            seen = set()
            for sid in te.sinks:
                if sid not in node_index:
                    raise errors.DanglingEndpoint(f"edge '{te.id}' has unknown sink '{sid}'")
                w = node_index[sid]
                if w in seen:
                    raise errors.InvalidStructure(f"edge '{te.id}' lists sink '{sid}' twice")
                seen.add(w)
                sinks.append(w)
                has_fanin[w] = True
            off[e + 1] = len(sinks)
            size[e] = te.size
        for v, nd in enumerate(nodes):
            if NodeRole(nd.role) == NodeRole.SOURCE and has_fanin[v]:
                raise errors.InvalidStructure(f"source node '{nd.id}' has fanin edges")
        g.node_ids = [nd.id for nd in nodes]
        g.node_roles = [NodeRole(nd.role) for nd in nodes]
        g.edge_ids = [te.id for te in edges]
        g.edge_kinds = [EdgeKind(te.kind) for te in edges]
        g._node_index = node_index
        g._edge_index = edge_index
        g._set_csr(len(nodes), src, off, np.asarray(sinks, np.int32), size)
        g._check_bytes_and_cycles()
        return g

    @classmethod
    def from_csr(cls, n, edge_src, sink_off, sinks, edge_size, node_ids=None, edge_ids=None,
                 node_roles=None, edge_kinds=None, validate=True) -> "Graph":
        """Wrap an already-indexed CSR (generated or traced graphs)."""
        g = cls()
        g._set_csr(int(n), np.ascontiguousarray(edge_src, np.int32),
                   np.ascontiguousarray(sink_off, np.int64), np.ascontiguousarray(sinks, np.int32),
                   np.ascontiguousarray(edge_size, np.uint64))
        g.node_ids = list(node_ids) if node_ids is not None else [f"v{i}" for i in range(g.n)]
        g.edge_ids = list(edge_ids) if edge_ids is not None else [f"e{i}" for i in range(g.E)]
        g.node_roles = (list(node_roles) if node_roles is not None
                        else [NodeRole.COMPUTE] * g.n)
        if edge_kinds is None:
            edge_kinds = [EdgeKind.DATA if s > 0 else EdgeKind.CONTROL for s in g.edge_size]
        g.edge_kinds = list(edge_kinds)
        if validate:
            g._check_bytes_and_cycles()
        return g

    def _set_csr(self, n, src, off, sinks, size):
        self.n = int(n)
        self.E = int(src.shape[0])
        self.edge_src = src
        self.sink_off = off
        self.sinks = sinks
        self.edge_size = size
        self.total_bytes = int(size.sum(dtype=np.uint64)) if self.E else 0

    def _check_bytes_and_cycles(self):
        total = 0
        for s in self.edge_size.tolist():
            if s >= BYTE_CAP or total + s >= BYTE_CAP:
                raise errors.InvalidStructure("total tensor bytes exceed the supported range")
            total += s
        cyc = self._find_cycle()
        if cyc is not None:
            raise errors.CycleDetected("cycle: " + " -> ".join(cyc))

    def _find_cycle(self):
        """find_cycle (graph.cpp:149-199): iterative DFS, roots and fanout in index order."""
        n = self.n
        fanout = self.fanout_lists()
        color = bytearray(n)  # 0 white, 1 grey, 2 black
        off, sinks = self.sink_off, self.sinks
        for root in range(n):
            if color[root]:
                continue
            stack = [[root, 0, 0]]
            color[root] = 1
            while stack:
                f = stack[-1]
                v = f[0]
                descended = False
                fo = fanout[v]
                while f[1] < len(fo):
                    e = fo[f[1]]
                    s0, s1 = int(off[e]), int(off[e + 1])
                    if f[2] >= s1 - s0:
                        f[1] += 1
                        f[2] = 0
                        continue
                    nxt = int(sinks[s0 + f[2]])
                    f[2] += 1
                    if color[nxt] == 1:
                        at = len(stack)
                        while at > 0 and stack[at - 1][0] != nxt:
                            at -= 1
                        ids = [self.node_ids[stack[i][0]] if self.node_ids else str(stack[i][0])
                               for i in range(at - 1, len(stack))]
                        ids.append(self.node_ids[nxt] if self.node_ids else str(nxt))
                        return ids
                    if color[nxt] == 0:
                        color[nxt] = 1
                        stack.append([nxt, 0, 0])
                        descended = True
                        break
                if not descended and stack[-1][1] >= len(fanout[stack[-1][0]]):
                    color[stack[-1][0]] = 2
                    stack.pop()
        return None

    # ---- accessors (graph.hpp:66-96) ----------------------------------------
    def num_nodes(self) -> int:
        return self.n

    def num_edges(self) -> int:
        return self.E

    def node_index(self, node_id: str) -> int:
        if self._node_index is None:
            self._node_index = {s: i for i, s in enumerate(self.node_ids)}
        if node_id not in self._node_index:
            raise errors.DanglingEndpoint(f"unknown node id '{node_id}'")
        return self._node_index[node_id]

    def edge_index(self, edge_id: str) -> int:
        if self._edge_index is None:
            self._edge_index = {s: i for i, s in enumerate(self.edge_ids)}
        if edge_id not in self._edge_index:
            raise errors.DanglingEndpoint(f"unknown edge id '{edge_id}'")
        return self._edge_index[edge_id]

    def has_node(self, node_id: str) -> bool:
        if self._node_index is None:
            self._node_index = {s: i for i, s in enumerate(self.node_ids)}
        return node_id in self._node_index

    def has_edge(self, edge_id: str) -> bool:
        if self._edge_index is None:
            self._edge_index = {s: i for i, s in enumerate(self.edge_ids)}
        return edge_id in self._edge_index

    def source_of(self, e: int) -> int:
        return int(self.edge_src[e])

    def sinks_of(self, e: int) -> list[int]:
        return self.sinks[self.sink_off[e]:self.sink_off[e + 1]].tolist()

    def fanout_lists(self) -> list[list[int]]:
        out: list[list[int]] = [[] for _ in range(self.n)]
        for e, s in enumerate(self.edge_src.tolist()):
            out[s].append(e)
        return out

    def id_rank(self) -> np.ndarray:
        """Rank of each edge id in byte-lexicographic order (std::string's
        operator<, the pyramid tie-break at placement.cpp:48-50)."""
        if getattr(self, "_id_rank", None) is None or len(self._id_rank) != self.E:
            r = np.zeros(max(self.E, 1), np.int32)
            for k, e in enumerate(sorted(range(self.E), key=lambda e: self.edge_ids[e].encode())):
                r[e] = k
            self._id_rank = r
        return self._id_rank

    def csr(self) -> dict:
        return {"n": self.n, "edge_src": self.edge_src, "sink_off": self.sink_off,
                "sinks": self.sinks, "edge_size": self.edge_size}

    def mp_csr(self) -> _native.MpCsr:
        """C-ABI view (arrays stay owned by this Graph)."""
        return _native.MpCsr(self.n, self.E, self.edge_src.ctypes.data, self.sink_off.ctypes.data,
                             self.sinks.ctypes.data, self.edge_size.ctypes.data)

    def with_aligned_sizes(self, align: int) -> "Graph":
        """graph.cpp:227-237."""
        if align == 0 or (align & (align - 1)) != 0:
            raise errors.InvalidStructure(f"alignment must be a power of two, got {align}")
        size = self.edge_size.copy()
        data = size > 0
        a = np.uint64(align)
        size[data] = (size[data] + a - np.uint64(1)) & ~(a - np.uint64(1))
        return Graph.from_csr(self.n, self.edge_src, self.sink_off, self.sinks, size,
                              self.node_ids, self.edge_ids, self.node_roles, self.edge_kinds)

    def program_order(self) -> np.ndarray:
        """pipeline.cpp:38-45: node-array order when topological, else Kahn's."""
        order = np.arange(self.n, dtype=np.int32)
        if self.n == 0 or self.is_topological_order(order):
            return order
        return self.topological_order()

    def is_topological_order(self, order) -> bool:
        """graph.cpp:239-254 (host check used for program order selection only)."""
        order = np.asarray(order)
        if order.shape[0] != self.n:
            return False
        if self.n == 0:
            return True
        if order.min() < 0 or order.max() >= self.n:
            return False
        pos = np.full(self.n, -1, np.int64)
        pos[order] = np.arange(self.n)
        if (pos < 0).any():
            return False
        counts = np.diff(self.sink_off)
        src_pos = np.repeat(pos[self.edge_src], counts)
        return bool((pos[self.sinks] > src_pos).all())

    def topological_order(self) -> np.ndarray:
        """graph.cpp:256-280: Kahn with a ready list sorted by node index."""
        import heapq
        missing = np.bincount(self.sinks, minlength=self.n).astype(np.int64) if self.n else []
        fanout = self.fanout_lists()
        ready = [v for v in range(self.n) if missing[v] == 0]
        heapq.heapify(ready)
        order = []
        while ready:
            v = heapq.heappop(ready)
            order.append(v)
            for e in fanout[v]:
                for s in self.sinks_of(e):
                    missing[s] -= 1
                    if missing[s] == 0:
                        heapq.heappush(ready, s)
        return np.asarray(order, np.int32)


# ---- canonical JSON (graph_io.cpp:60-142) -----------------------------------
def _reject_unknown(obj, what, allowed):
    for k in obj:
        if k not in allowed:
            raise errors.ParseError(f"{what} has unknown field '{k}'")


def load_graph(text: str) -> Graph:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise errors.ParseError(f"graph file: {e}") from None
    if not isinstance(doc, dict):
        raise errors.ParseError("graph file must be a JSON object")
    _reject_unknown(doc, "graph file", ("nodes", "edges"))
    for key in ("nodes", "edges"):
        if key not in doc:
            raise errors.ParseError(f"graph file is missing field '{key}'")
    if not isinstance(doc["nodes"], list):
        raise errors.ParseError("'nodes' must be an array")
    if not isinstance(doc["edges"], list):
        raise errors.ParseError("'edges' must be an array")
    nodes = []
    for jn in doc["nodes"]:
        if not isinstance(jn, dict):
            raise errors.ParseError("node entries must be objects")
        _reject_unknown(jn, "node", ("id", "role"))
        if "id" not in jn:
            raise errors.ParseError("node is missing field 'id'")
        if not isinstance(jn["id"], str):
            raise errors.ParseError("node field 'id' must be a string")
        role = jn.get("role", "compute")
        if not isinstance(role, str):
            raise errors.ParseError("node field 'role' must be a string")
        try:
            role = NodeRole(role)
        except ValueError:
            raise errors.ParseError(f"unknown node role '{role}'") from None
        nodes.append(Node(jn["id"], role))
    edges = []
    for je in doc["edges"]:
        if not isinstance(je, dict):
            raise errors.ParseError("edge entries must be objects")
        _reject_unknown(je, "edge", ("id", "source", "sinks", "size", "kind"))
        for key in ("id", "source", "sinks", "size"):
            if key not in je:
                raise errors.ParseError(f"edge is missing field '{key}'")
        eid = je["id"]
        if not isinstance(je["sinks"], list):
            raise errors.ParseError(f"edge '{eid}': 'sinks' must be an array")
        if not all(isinstance(s, str) for s in je["sinks"]):
            raise errors.ParseError(f"edge '{eid}': sinks must be strings")
        size = je["size"]
        if not isinstance(size, int) or isinstance(size, bool) or size < 0:
            raise errors.ParseError(f"edge '{eid}': 'size' must be a non-negative integer")
        kind = je.get("kind", "data")
        try:
            kind = EdgeKind(kind)
        except ValueError:
            raise errors.ParseError(f"unknown edge kind '{kind}'") from None
        edges.append(TensorEdge(eid, je["source"], list(je["sinks"]), size, kind))
    return Graph.build(nodes, edges)


def load_graph_file(path: str) -> Graph:
    with open(path) as f:
        return load_graph(f.read())


def save_graph(g: Graph) -> str:
    """Canonical text: fixed key order, 2-space indent, trailing newline."""
    doc = {"nodes": [{"id": g.node_ids[v], "role": g.node_roles[v].value} for v in range(g.n)],
           "edges": []}
    for e in range(g.E):
        doc["edges"].append({
            "id": g.edge_ids[e],
            "source": g.node_ids[int(g.edge_src[e])],
            "sinks": [g.node_ids[w] for w in g.sinks_of(e)],
            "size": int(g.edge_size[e]),
            "kind": g.edge_kinds[e].value,
        })
    return json.dumps(doc, indent=2) + "\n"


# ---- generators (generate.cpp:45-158) -----------------------------------------
GRAPH_KINDS = {"chain": 0, "fork_join": 1, "training_like": 2}


def generate_graph(kind: str, layers: int, size: int = 8, seed: int = 0) -> Graph:
    """generate_graph with the reference's ids; CSR from the native generator."""
    if kind not in GRAPH_KINDS:
        raise errors.InvalidSpec(f"unknown graph kind '{kind}'")
    if layers < 1:
        raise errors.InvalidSpec(f"layers must be >= 1, got {layers}")
    if size < 1:
        raise errors.InvalidSpec("size must be >= 1")
    L = _native.lib()
    n, E, S = C.c_int32(), C.c_int32(), C.c_int64()
    k = GRAPH_KINDS[kind]
    _native.check(L.mp_generate_graph(k, layers, size, seed, C.byref(n), C.byref(E), C.byref(S),
                                      None, None, None, None, None))
    src = np.zeros(E.value, np.int32)
    off = np.zeros(E.value + 1, np.int64)
    sinks = np.zeros(S.value, np.int32)
    esize = np.zeros(E.value, np.uint64)
    roles = np.zeros(n.value, np.uint8)
    _native.check(L.mp_generate_graph(k, layers, size, seed, C.byref(n), C.byref(E), C.byref(S),
                                      src.ctypes.data, off.ctypes.data, sinks.ctypes.data,
                                      esize.ctypes.data, roles.ctypes.data))
    node_ids, edge_ids = _generated_ids(kind, layers, n.value, src, off)
    return Graph.from_csr(n.value, src, off, sinks, esize, node_ids, edge_ids,
                          [_ROLE_CODES[r] for r in roles.tolist()], validate=False)


def _generated_ids(kind, L, n, src, off):
    if kind == "chain":
        return [f"n{i}" for i in range(n)], [f"t{i}" for i in range(L)]
    if kind == "training_like":
        nodes = (["x"] + [f"w{i}" for i in range(1, L + 1)] + [f"fwd{i}" for i in range(1, L + 1)]
                 + ["loss"] + [f"bwd{i}" for i in range(L, 0, -1)] + ["gnrm"]
                 + [f"upd{i}" for i in range(L, 0, -1)] + ["gsink"])
        edges = ([f"act{i}" for i in range(L + 1)] + [f"wt{i}" for i in range(1, L + 1)]
                 + ["lossv"] + [f"gb{i}" for i in range(L, 0, -1)] + ["gn"])
        return nodes, edges
    # fork_join: per stage fork, branches, join; widths follow from the fork fanout.
    fanout = np.bincount(src, minlength=n)
    nodes, edges = [], []
    v = 0
    for d in range(L):
        width = int(fanout[v])
        nodes.append(f"fork{d}")
        nodes.extend(f"b{d}_{b}" for b in range(width))
        nodes.append(f"join{d}")
        if d > 0:
            edges.append(f"link{d - 1}")
        for b in range(width):
            edges.extend([f"f{d}_{b}", f"j{d}_{b}"])
        v += width + 2
    edges.append("out")
    return nodes, edges


def graph_from_lists(nodes: Iterable[tuple], edges: Iterable[tuple]) -> Graph:
    """Convenience: nodes as (id, role), edges as (id, source, sinks, size[, kind])."""
    ns = [Node(i, NodeRole(r)) for i, r in nodes]
    es = []
    for t in edges:
        kind = t[4] if len(t) > 4 else "data"
        es.append(TensorEdge(t[0], t[1], list(t[2]), t[3], EdgeKind(kind)))
    return Graph.build(ns, es)
