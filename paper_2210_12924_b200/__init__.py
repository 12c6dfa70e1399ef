"""memplan_b200: the data-parallel core of OLLA's memory planner (arXiv 2210.12924)
re-built for NVIDIA B200 (sm_100a).

Public surface (mirrors the reference memplan API for the hot path):
  Graph / load_graph / save_graph / generate_graph      (graph.py)
  Planner: lifetimes_from_order, realized_lifetimes, resident_bytes_per_step,
           peak_resident_bytes, timeline_from_lifetimes, score_orders, argmin,
           encode_address_pairs, validate_plan, addresses_feasible, peak_mem,
           preallocate_pyramid, greedy_pack, place_batch, run_baseline
  fragmentation, format_report, random_topo_orders      (planner.py)
The compute path is the native library lib/libmemplan_b200.so (C ABI in
include/memplan_b200.h); there is no CPU fallback.
"""
from . import errors
from .graph import (EdgeKind, Graph, Node, NodeRole, TensorEdge, generate_graph,
                    graph_from_lists, load_graph, load_graph_file, save_graph)
from .planner import (BaselineResult, DeviceGraph, MultiPlanner, ExecutionSequence, Interval, MemoryPlan, Planner,
                      PrePlacement, ResidentTimeline, ScoreResult, format_report, fragmentation,
                      intervals_disjoint, load_plan, random_topo_orders)

__all__ = [
    "BaselineResult", "MultiPlanner", "errors", "EdgeKind", "Graph", "Node", "NodeRole", "TensorEdge", "generate_graph",
    "graph_from_lists", "load_graph", "load_graph_file", "save_graph", "DeviceGraph",
    "ExecutionSequence", "Interval", "MemoryPlan", "Planner", "PrePlacement", "ResidentTimeline",
    "ScoreResult",
    "format_report", "fragmentation", "intervals_disjoint", "load_plan", "random_topo_orders",
]
