"""The reference planner's hot-path API, executed by the sm_100a library.

Each method keeps the reference function's name, argument meaning and error
behaviour (raising the same exception class with the same message text) and
cites the file:line it replaces. Host work here is limited to argument
marshalling and report assembly; every data-parallel computation runs in
``lib/libmemplan_b200.so`` through the C ABI (include/memplan_b200.h). There is
no CPU fallback: without an sm_100 device the constructor raises DeviceError.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Mapping, Optional, Sequence

import numpy as np

from . import _native, errors
from .graph import Graph

_vp = C.c_void_p


@dataclass
class Interval:
    """memplan::Interval (analysis.hpp:28-33): closed, 1-based, empty if lo > hi."""
    lo: int = 1
    hi: int = 0

    def empty(self) -> bool:
        return self.lo > self.hi

    def contains(self, t: int) -> bool:
        return self.lo <= t <= self.hi


def intervals_disjoint(a: Interval, b: Interval) -> bool:
    """analysis.hpp:35-37."""
    return a.empty() or b.empty() or a.hi < b.lo or b.hi < a.lo


@dataclass
class ResidentTimeline:
    """memplan::ResidentTimeline (plan.hpp:43-48) without the per-step id lists."""
    bytes: np.ndarray
    peak_rs: int
    peak_step: int


@dataclass
class ScoreResult:
    peak: np.ndarray       # uint64[C]; 0 for invalid candidates
    peak_step: np.ndarray  # int32[C]; 0 for invalid candidates
    valid: np.ndarray      # uint8[C]

    def argmin(self) -> int:
        """First minimum over valid candidates (-1 if none)."""
        idx = np.flatnonzero(self.valid)
        if idx.size == 0:
            return -1
        return int(idx[np.argmin(self.peak[idx])])  # np.argmin returns the first minimum


@dataclass
class ExecutionSequence:
    steps: list = field(default_factory=list)
    timestep_of: dict = field(default_factory=dict)


@dataclass
class MemoryPlan:
    """memplan::MemoryPlan (plan.hpp:76-82); provenance kept as a dict."""
    sequence: ExecutionSequence = field(default_factory=ExecutionSequence)
    addresses: dict = field(default_factory=dict)
    peak_mem: int = 0
    timeline_bytes: list = field(default_factory=list)
    peak_rs: int = 0
    peak_step: int = 0
    provenance: dict = field(default_factory=dict)


def load_plan(text: str) -> MemoryPlan:
    """Reads the canonical plan file (plan.cpp:233-305; strictness reduced to
    the fields validate_plan consumes)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise errors.ParseError(f"plan file: {e}") from None
    for key in ("sequence", "timesteps", "addresses", "peak_mem", "timeline", "provenance"):
        if key not in doc:
            raise errors.ParseError(f"plan file is missing field '{key}'")
    plan = MemoryPlan()
    plan.sequence.steps = list(doc["sequence"])
    plan.sequence.timestep_of = {k: int(v) for k, v in doc["timesteps"].items()}
    plan.addresses = {k: int(v) for k, v in doc["addresses"].items()}
    plan.peak_mem = int(doc["peak_mem"])
    plan.timeline_bytes = [int(b) for b in doc["timeline"]["bytes"]]
    plan.peak_rs = int(doc["timeline"]["peak_rs"])
    plan.peak_step = int(doc["timeline"]["peak_step"])
    plan.provenance = dict(doc["provenance"])
    return plan


class MultiPlanner:
    """One process, several GPUs (mp_multi_*): the graph replicated on every device,
    candidates split into contiguous shards scored concurrently (one host thread
    per device), the shards' first minima meeting in ONE device-side NCCL
    allreduce(MIN) on the fused key when the devices are distinct and NCCL loads
    (``nccl`` is True), else combined on the host."""

    def __init__(self, devices: Sequence[int]):
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _native.check(_native.lib().mp_multi_create(devs, len(devices), C.byref(h)))
        self.handle = h
        self.graph = None
        self.nccl = bool(_native.lib().mp_multi_nccl(h))

    def upload(self, graph: Graph) -> None:
        self._csr = graph.mp_csr()
        _native.check(_native.lib().mp_multi_upload(self.handle, C.byref(self._csr)))
        self.graph = graph

    def score_orders(self, orders) -> tuple["ScoreResult", int]:
        o = _i32(orders)
        if o.ndim == 1:
            o = o.reshape(1, -1)
        c = o.shape[0]
        if self.graph is None or o.shape[1] != self.graph.n:
            raise ValueError("upload the graph first; orders must be [C][n]")
        peak = np.zeros(max(c, 1), np.uint64)
        step = np.zeros(max(c, 1), np.int32)
        valid = np.zeros(max(c, 1), np.uint8)
        best = C.c_int64()
        _native.check(_native.lib().mp_score_orders_multi(self.handle, o.ctypes.data, c,
                                                          peak.ctypes.data, step.ctypes.data,
                                                          valid.ctypes.data, C.byref(best)))
        return ScoreResult(peak[:c], step[:c], valid[:c]), best.value

    def close(self) -> None:
        if getattr(self, "handle", None):
            _native.lib().mp_multi_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class BaselineResult:
    """memplan::BaselineResult (placement.hpp:44-48)."""
    mr_peak: int = 0
    rs_at_peak: int = 0
    fragmentation: float = 0.0


@dataclass
class PrePlacement:
    """memplan::PrePlacement (placement.hpp:26-30)."""
    assigned: dict
    remaining: list
    reserved_base: int = 0


def fragmentation(mr: int, rs: int) -> float:
    """placement.cpp:64-67 (the native library evaluates the same expression)."""
    return float(_native.lib().mp_fragmentation(int(mr), int(rs)))


class DeviceGraph:
    """A graph uploaded to one context (mp_graph_upload)."""

    def __init__(self, planner: "Planner", graph: Graph):
        self.planner = planner
        self.graph = graph
        self._csr = graph.mp_csr()
        h = _vp()
        _native.check(_native.lib().mp_graph_upload(planner.ctx, C.byref(self._csr), C.byref(h)))
        self.handle = h

    def info(self) -> dict:
        info = _native.MpGraphInfo()
        _native.check(_native.lib().mp_graph_get_info(self.handle, C.byref(info)))
        return {k: getattr(info, k) for k, _ in info._fields_}

    def free(self):
        if self.handle:
            _native.lib().mp_graph_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _i32(a):
    return np.ascontiguousarray(a, np.int32)


def _check_host(a, name, itemsize, kinds, ndim):
    """Shape of a C-contiguous host array (numpy or CPU torch) of an accepted dtype."""
    if hasattr(a, "is_cuda"):
        if a.is_cuda:
            raise ValueError(f"{name} must be host memory, got a CUDA tensor")
        if not a.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        dt, isz, shape = str(a.dtype).replace("torch.", ""), a.element_size(), tuple(a.shape)
    elif isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name} must be C-contiguous")
        dt, isz, shape = str(a.dtype), a.itemsize, a.shape
    else:
        raise ValueError(f"{name} must be a numpy array or a CPU torch tensor")
    if dt not in kinds or isz != itemsize or len(shape) != ndim:
        raise ValueError(f"{name} must be {ndim}-d {'/'.join(kinds)}, got {len(shape)}-d {dt}")
    return shape


class Planner:
    """One device context (mp_ctx) plus the graphs uploaded to it."""

    def __init__(self, device: int = 0):
        L = _native.lib()
        h = _vp()
        _native.check(L.mp_ctx_create(device, C.byref(h)))
        self.ctx = h
        self.device = device
        self._graphs: dict[int, DeviceGraph] = {}

    def close(self):
        for dg in self._graphs.values():
            dg.free()
        self._graphs.clear()
        if self.ctx:
            _native.lib().mp_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        _native.check(_native.lib().mp_ctx_set_stream(self.ctx, stream_ptr))

    def upload(self, graph: Graph) -> DeviceGraph:
        dg = self._graphs.get(id(graph))
        if dg is None or dg.graph is not graph:
            dg = DeviceGraph(self, graph)
            self._graphs[id(graph)] = dg
        return dg

    # ---- (a2/a3) ------------------------------------------------------------
    def lifetimes_from_order(self, graph: Graph, order: Sequence[int]):
        """schedule.cpp:33-50 -> (lo, hi) int32 arrays; InvalidOrder if not topological."""
        dg = self.upload(graph)
        o = _i32(order)
        lo = np.zeros(max(graph.E, 1), np.int32)
        hi = np.zeros(max(graph.E, 1), np.int32)
        _native.check(_native.lib().mp_lifetimes(self.ctx, dg.handle, o.ctypes.data, o.size,
                                                 lo.ctypes.data, hi.ctypes.data))
        return lo[:graph.E], hi[:graph.E]

    def positions_of(self, graph: Graph, order: Sequence[int]) -> np.ndarray:
        """schedule.cpp:23-31: the device validates the order, pos is its inverse."""
        self.lifetimes_from_order(graph, order)
        pos = np.zeros(graph.n, np.int32)
        pos[_i32(order)] = np.arange(1, graph.n + 1, dtype=np.int32)
        return pos

    # ---- (a4) ---------------------------------------------------------------
    def realized_lifetimes(self, graph: Graph, timestep_of, horizon: int):
        """plan.cpp:101-120. timestep_of: {node id: step} or int32[n] (0 = absent)."""
        dg = self.upload(graph)
        if isinstance(timestep_of, Mapping):
            ts = np.zeros(graph.n, np.int32)
            for k, v in timestep_of.items():
                if graph.has_node(k):
                    ts[graph.node_index(k)] = v
        else:
            ts = _i32(timestep_of)
        lo = np.zeros(max(graph.E, 1), np.int32)
        hi = np.zeros(max(graph.E, 1), np.int32)
        miss = C.c_int32(-1)
        st = _native.lib().mp_realized_lifetimes(self.ctx, dg.handle, ts.ctypes.data, int(horizon),
                                                 lo.ctypes.data, hi.ctypes.data, C.byref(miss))
        if st == _native.MP_E_INVALID_ORDER:
            raise errors.InvalidOrder(f"node {graph.node_ids[miss.value]} has no timestep")
        _native.check(st)
        return lo[:graph.E], hi[:graph.E]

    # ---- (a8/a9/a10) --------------------------------------------------------
    def resident_bytes_per_step(self, graph: Graph, order) -> np.ndarray:
        """schedule.cpp:69-79."""
        dg = self.upload(graph)
        o = _i32(order)
        out = np.zeros(max(graph.n, 1), np.uint64)
        _native.check(_native.lib().mp_resident_bytes(self.ctx, dg.handle, o.ctypes.data, o.size,
                                                      out.ctypes.data))
        return out[:graph.n]

    def peak_resident_bytes(self, graph: Graph, order) -> int:
        """schedule.cpp:81-88."""
        dg = self.upload(graph)
        o = _i32(order)
        p = C.c_uint64()
        _native.check(_native.lib().mp_peak_resident_bytes(self.ctx, dg.handle, o.ctypes.data,
                                                           o.size, C.byref(p)))
        return int(p.value)

    def timeline_from_lifetimes(self, graph: Graph, lo, hi, horizon: int) -> ResidentTimeline:
        """plan.cpp:122-143 (bytes, peak_rs, peak_step)."""
        dg = self.upload(graph)
        lo, hi = _i32(lo), _i32(hi)
        b = np.zeros(max(horizon, 1), np.uint64)
        pr, ps = C.c_uint64(), C.c_int32()
        _native.check(_native.lib().mp_timeline(self.ctx, dg.handle, lo.ctypes.data, hi.ctypes.data,
                                                int(horizon), b.ctypes.data, C.byref(pr),
                                                C.byref(ps)))
        return ResidentTimeline(b[:horizon], int(pr.value), int(ps.value))

    # ---- batched scoring ------------------------------------------------------
    def score_orders(self, graph: Graph, orders) -> ScoreResult:
        """peak_resident_bytes over many candidate orders at once (+ verdicts)."""
        dg = self.upload(graph)
        o = _i32(orders)
        if o.ndim == 1:
            o = o.reshape(1, -1)
        c = o.shape[0]
        if o.shape[1] != graph.n:
            # every candidate of the wrong length is invalid (graph.cpp:241)
            return ScoreResult(np.zeros(c, np.uint64), np.zeros(c, np.int32), np.zeros(c, np.uint8))
        peak = np.zeros(max(c, 1), np.uint64)
        step = np.zeros(max(c, 1), np.int32)
        valid = np.zeros(max(c, 1), np.uint8)
        _native.check(_native.lib().mp_score_orders(self.ctx, dg.handle, o.ctypes.data, c,
                                                    peak.ctypes.data, step.ctypes.data,
                                                    valid.ctypes.data))
        return ScoreResult(peak[:c], step[:c], valid[:c])

    def score_orders_best(self, graph: Graph, orders) -> tuple[ScoreResult, int]:
        """Scoring with the first-minimum argmin fused into the kernel."""
        dg = self.upload(graph)
        o = _i32(orders)
        if o.ndim == 1:
            o = o.reshape(1, -1)
        c = o.shape[0]
        if o.shape[1] != graph.n:
            return ScoreResult(np.zeros(c, np.uint64), np.zeros(c, np.int32),
                               np.zeros(c, np.uint8)), -1
        peak = np.zeros(max(c, 1), np.uint64)
        step = np.zeros(max(c, 1), np.int32)
        valid = np.zeros(max(c, 1), np.uint8)
        best = C.c_int64()
        _native.check(_native.lib().mp_score_orders_best(self.ctx, dg.handle, o.ctypes.data, c,
                                                         peak.ctypes.data, step.ctypes.data,
                                                         valid.ctypes.data, C.byref(best)))
        return ScoreResult(peak[:c], step[:c], valid[:c]), int(best.value)

    def score_orders_into(self, dg: DeviceGraph, orders_host, peak, step, valid) -> int:
        """Public host-buffer call for pre-allocated (e.g. pinned) buffers: H2D of the
        orders, one fused scoring+argmin kernel, D2H of peak/step/valid; returns best.

        orders: C-contiguous host int32 [C, n]; peak: 8-byte [>= C]; step: int32
        [>= C]; valid: uint8 [>= C] (numpy arrays or CPU torch tensors). Anything
        else raises ValueError before the native call reads or writes a byte."""
        c = _check_host(orders_host, "orders", 4, ("int32",), ndim=2)
        if c[1] != dg.graph.n:
            raise ValueError(f"orders must have shape [C, {dg.graph.n}], got {tuple(c)}")
        for a, nm, isz, kinds in ((peak, "peak", 8, ("uint64", "int64")),
                                  (step, "step", 4, ("int32",)), (valid, "valid", 1, ("uint8",))):
            shp = _check_host(a, nm, isz, kinds, ndim=1)
            if shp[0] < c[0]:
                raise ValueError(f"{nm} holds {shp[0]} entries, needs {c[0]}")
        best = C.c_int64()
        _native.check(_native.lib().mp_score_orders_best(
            self.ctx, dg.handle, _native.ptr(orders_host), int(orders_host.shape[0]),
            _native.ptr(peak), _native.ptr(step), _native.ptr(valid), C.byref(best)))
        return int(best.value)

    def argmin(self, peak, valid) -> int:
        p = np.ascontiguousarray(peak, np.uint64)
        v = np.ascontiguousarray(valid, np.uint8)
        best = C.c_int64()
        _native.check(_native.lib().mp_argmin(self.ctx, p.ctypes.data, v.ctypes.data, p.size,
                                              C.byref(best)))
        return int(best.value)

    def score_orders_d(self, dg: DeviceGraph, d_orders, num_orders, d_peak, d_step, d_valid,
                       stream: int | None = None):
        """Device-pointer variant (torch tensors or raw pointers), stream-ordered."""
        _native.check(_native.lib().mp_score_orders_d(
            self.ctx, dg.handle, _native.ptr(d_orders), int(num_orders), _native.ptr(d_peak),
            _native.ptr(d_step), _native.ptr(d_valid), stream))

    def score_orders_argmin_d(self, dg: DeviceGraph, d_orders, num_orders, d_peak, d_step,
                              d_valid, d_best_key, index_base=0, stream: int | None = None):
        """d_best_key: 2 int64 words {key, overflow} (reset with key_reset_d)."""
        _native.check(_native.lib().mp_score_orders_argmin_d(
            self.ctx, dg.handle, _native.ptr(d_orders), int(num_orders), _native.ptr(d_peak),
            _native.ptr(d_step), _native.ptr(d_valid), _native.ptr(d_best_key), int(index_base),
            stream))

    def key_reset_d(self, d_best_key, stream: int | None = None):
        """{MP_KEY_NONE, no overflow} into the 2-word fused key (one memset node)."""
        _native.check(_native.lib().mp_key_reset_d(self.ctx, _native.ptr(d_best_key), stream))

    # ---- batched candidate plans (plan_once's placement half per order) -----------
    def score_plans_d(self, dg: DeviceGraph, d_orders, num_orders, d_id_rank, pyramid: bool,
                      d_peak_rs, d_peak_step, d_valid, d_peak_mem, d_nviol, d_addr=None,
                      d_has=None, d_best_key=None, index_base=0, stream: int | None = None):
        """mp_score_plans_d: per candidate order the schedule score, its lifetimes,
        preallocate_pyramid + greedy_pack addresses, peak_mem and the number of
        below_above pairs (0 = addresses_feasible); optional fused first-minimum key
        of peak_mem over feasible plans."""
        _native.check(_native.lib().mp_score_plans_d(
            self.ctx, dg.handle, _native.ptr(d_orders), int(num_orders), _native.ptr(d_id_rank),
            self.PLACE_PYRAMID if pyramid else 0, _native.ptr(d_peak_rs), _native.ptr(d_peak_step),
            _native.ptr(d_valid), _native.ptr(d_peak_mem), _native.ptr(d_nviol),
            _native.ptr(d_addr), _native.ptr(d_has), _native.ptr(d_best_key), int(index_base),
            stream))

    def score_plans(self, graph: Graph, orders, pyramid: bool = True):
        """Host convenience over score_plans_d: returns dict of numpy arrays (peak_rs,
        peak_step, valid, peak_mem, nviol, addr, has_addr) and the best plan index
        (first minimum peak_mem over feasible plans, -1 if none)."""
        import torch
        dg = self.upload(graph)
        o = np.ascontiguousarray(orders, np.int32).reshape(-1, graph.n)
        c, E = o.shape[0], graph.E
        dev = torch.device("cuda", self.device)
        t = lambda shape, dt: torch.zeros(shape, dtype=dt, device=dev)  # noqa: E731
        d_o = torch.from_numpy(o).to(dev)
        rank = torch.from_numpy(graph.id_rank()[:max(E, 1)].copy()).to(dev)
        out = {"peak_rs": t(max(c, 1), torch.int64), "peak_step": t(max(c, 1), torch.int32),
               "valid": t(max(c, 1), torch.uint8), "peak_mem": t(max(c, 1), torch.int64),
               "nviol": t(max(c, 1), torch.int32), "addr": t((max(c, 1), max(E, 1)), torch.int64),
               "has_addr": t((max(c, 1), max(E, 1)), torch.uint8)}
        key = t(2, torch.int64)
        st = torch.cuda.current_stream(dev).cuda_stream
        self.key_reset_d(key, st)
        self.score_plans_d(dg, d_o, c, rank, pyramid, out["peak_rs"], out["peak_step"],
                           out["valid"], out["peak_mem"], out["nviol"], out["addr"],
                           out["has_addr"], key, 0, st)
        torch.cuda.synchronize(dev)
        res = {k: v.cpu().numpy()[:c] for k, v in out.items()}
        for k in ("peak_rs", "peak_mem", "addr"):
            res[k] = res[k].view(np.uint64)
        from . import dist as D
        kp = key.cpu().tolist()
        best = -1 if D.key_overflowed(kp) or kp[0] == D.NO_KEY else D.unpack_key(kp[0])[1]
        if D.key_overflowed(kp):    # a peak past the packed range: reduce on the host
            ok = [i for i in range(c) if res["valid"][i] and res["nviol"][i] == 0]
            best = min(ok, key=lambda i: (int(res["peak_mem"][i]), i)) if ok else -1
        return res, best

    def validate_plans_d(self, num_edges, num_plans, d_lo, d_hi, d_size, d_has, d_addr, d_valid,
                         d_nviol, stream: int | None = None):
        """mp_validate_plans_d: below_above pair count per caller-supplied plan."""
        _native.check(_native.lib().mp_validate_plans_d(
            self.ctx, int(num_edges), int(num_plans), _native.ptr(d_lo), _native.ptr(d_hi),
            _native.ptr(d_size), _native.ptr(d_has), _native.ptr(d_addr), _native.ptr(d_valid),
            _native.ptr(d_nviol), stream))

    def lifetimes_batch_d(self, dg: DeviceGraph, d_orders, num_orders, d_lo, d_hi, d_valid,
                          stream: int | None = None):
        _native.check(_native.lib().mp_lifetimes_batch_d(
            self.ctx, dg.handle, _native.ptr(d_orders), int(num_orders), _native.ptr(d_lo),
            _native.ptr(d_hi), _native.ptr(d_valid), stream))

    def argmin_key_d(self, d_peak, d_valid, num_orders, index_base, d_out3,
                     stream: int | None = None):
        _native.check(_native.lib().mp_argmin_key_d(
            self.ctx, _native.ptr(d_peak), _native.ptr(d_valid), int(num_orders),
            int(index_base), _native.ptr(d_out3), stream))

    # ---- (a6) overlap pairs -----------------------------------------------------
    def encode_address_pairs(self, graph: Graph, lo, hi, preplaced: Mapping[int, int] | None = None,
                             want_pairs: bool = True):
        """Pair set of encode_addresses (encode.cpp:347-367) in emission order.

        ``preplaced`` maps edge index -> offset; pairs of two preplaced edges are
        skipped (:351). Returns int32[P, 2] (or the count with want_pairs=False);
        the count equals constraint_counts["live_pair"].
        """
        lo, hi = _i32(lo), _i32(hi)
        pin = None
        if preplaced:
            pin = np.zeros(graph.E, np.uint8)
            pin[list(preplaced.keys())] = 1
        return self.overlap_pairs(lo, hi, graph.edge_size, pin, want_pairs)

    def overlap_pairs(self, lo, hi, size, pinned=None, want_pairs: bool = True):
        lo, hi = _i32(lo), _i32(hi)
        size = np.ascontiguousarray(size, np.uint64)
        pin = None if pinned is None else np.ascontiguousarray(pinned, np.uint8)
        E = lo.size
        cnt = C.c_int64()
        L = _native.lib()
        _native.check(L.mp_overlap_pairs(self.ctx, E, lo.ctypes.data, hi.ctypes.data,
                                         size.ctypes.data, _native.ptr(pin), None, 0,
                                         C.byref(cnt)))
        if not want_pairs:
            return cnt.value
        out = np.zeros((max(cnt.value, 1), 2), np.int32)
        _native.check(L.mp_overlap_pairs(self.ctx, E, lo.ctypes.data, hi.ctypes.data,
                                         size.ctypes.data, _native.ptr(pin), out.ctypes.data,
                                         cnt.value, C.byref(cnt)))
        return out[:cnt.value]

    def overlap_pairs_d(self, num_edges, d_lo, d_hi, d_size, d_pinned, row_begin, row_end,
                        d_row_off, d_pairs, cap, stream: int | None = None) -> int:
        cnt = C.c_int64()
        _native.check(_native.lib().mp_overlap_pairs_d(
            self.ctx, int(num_edges), _native.ptr(d_lo), _native.ptr(d_hi), _native.ptr(d_size),
            _native.ptr(d_pinned), int(row_begin), int(row_end), _native.ptr(d_row_off),
            _native.ptr(d_pairs), int(cap), C.byref(cnt), stream))
        return cnt.value

    def overlap_pairs_rows_d(self, d_lo, d_hi, d_size, d_pinned, row_begin: int, row_end: int,
                             stream: int | None = None):
        """K2 over rows [row_begin, row_end) of device-resident lifetimes: count pass,
        then a fill into a fresh int32 [k, 2] device tensor (the shard function of
        dist.sharded_overlap_pairs)."""
        import torch
        E = int(d_lo.numel())
        rows = max(0, int(row_end) - int(row_begin))
        off = torch.empty(rows + 1, dtype=torch.int64, device=d_lo.device)
        k = self.overlap_pairs_d(E, d_lo, d_hi, d_size, d_pinned, row_begin, row_end, off, None,
                                 0, stream)
        out = torch.empty((max(k, 1), 2), dtype=torch.int32, device=d_lo.device)
        if k:
            self.overlap_pairs_d(E, d_lo, d_hi, d_size, d_pinned, row_begin, row_end, off, out, k,
                                 stream)
        return out[:k]

    # ---- (a11/a12/a13) validation -----------------------------------------------
    def conflicting_pairs(self, lo, hi, size, has_addr, addr) -> np.ndarray:
        """Pairwise part of validate_plan (plan.cpp:390-404), in (i, j) order."""
        lo, hi = _i32(lo), _i32(hi)
        size = np.ascontiguousarray(size, np.uint64)
        has = np.ascontiguousarray(has_addr, np.uint8)
        ad = np.ascontiguousarray(addr, np.uint64)
        E = lo.size
        cnt = C.c_int64()
        L = _native.lib()
        _native.check(L.mp_validate_pairs(self.ctx, E, lo.ctypes.data, hi.ctypes.data,
                                          size.ctypes.data, has.ctypes.data, ad.ctypes.data, None,
                                          0, C.byref(cnt)))
        out = np.zeros((max(cnt.value, 1), 2), np.int32)
        if cnt.value:
            _native.check(L.mp_validate_pairs(self.ctx, E, lo.ctypes.data, hi.ctypes.data,
                                              size.ctypes.data, has.ctypes.data, ad.ctypes.data,
                                              out.ctypes.data, cnt.value, C.byref(cnt)))
        return out[:cnt.value]

    def validate_pairs_d(self, num_edges, d_lo, d_hi, d_size, d_has, d_addr, row_begin, row_end,
                         d_row_off, d_viol, cap, stream: int | None = None) -> int:
        cnt = C.c_int64()
        _native.check(_native.lib().mp_validate_pairs_d(
            self.ctx, int(num_edges), _native.ptr(d_lo), _native.ptr(d_hi), _native.ptr(d_size),
            _native.ptr(d_has), _native.ptr(d_addr), int(row_begin), int(row_end),
            _native.ptr(d_row_off), _native.ptr(d_viol), int(cap), C.byref(cnt), stream))
        return cnt.value

    def conflicting_pairs_rows_d(self, d_lo, d_hi, d_size, d_has, d_addr, row_begin: int,
                                 row_end: int, stream: int | None = None):
        """K4 over rows [row_begin, row_end): violating pairs as an int32 [k, 2]
        device tensor (the shard function of dist.sharded_conflicts)."""
        import torch
        E = int(d_lo.numel())
        rows = max(0, int(row_end) - int(row_begin))
        off = torch.empty(rows + 1, dtype=torch.int64, device=d_lo.device)
        k = self.validate_pairs_d(E, d_lo, d_hi, d_size, d_has, d_addr, row_begin, row_end, off,
                                  None, 0, stream)
        out = torch.empty((max(k, 1), 2), dtype=torch.int32, device=d_lo.device)
        if k:
            self.validate_pairs_d(E, d_lo, d_hi, d_size, d_has, d_addr, row_begin, row_end, off,
                                  out, k, stream)
        return out[:k]

    def addresses_feasible(self, graph: Graph, lo, hi, addresses: Mapping[int, int]) -> bool:
        """pipeline.cpp:146-160 (addresses keyed by edge index)."""
        has, ad = self._addr_arrays(graph, addresses)
        f = C.c_int32()
        lo, hi = _i32(lo), _i32(hi)
        _native.check(_native.lib().mp_addresses_feasible(
            self.ctx, graph.E, lo.ctypes.data, hi.ctypes.data, graph.edge_size.ctypes.data,
            has.ctypes.data, ad.ctypes.data, C.byref(f)))
        return bool(f.value)

    def peak_mem(self, graph: Graph, addresses: Mapping[int, int]) -> int:
        """max(addr + size) over placed edges (pipeline.cpp:270-275)."""
        has, ad = self._addr_arrays(graph, addresses)
        out = C.c_uint64()
        _native.check(_native.lib().mp_peak_mem(self.ctx, graph.E, graph.edge_size.ctypes.data,
                                                has.ctypes.data, ad.ctypes.data, C.byref(out)))
        return int(out.value)

    # ---- joint-mode pair set (K8, k_joint.cu) -----------------------------------------
    def joint_pairs(self, graph: Graph, filter_pairs: bool = True) -> np.ndarray:
        """The pair loop of encode_joint (encode.cpp:401-408) -> int32[P][2] in (i, j) order:
        data-edge pairs not ordered by the graph (edge_precedes, analysis.cpp:94-113)."""
        dg = self.upload(graph)
        cnt = C.c_int64()
        _native.check(_native.lib().mp_joint_pairs(self.ctx, dg.handle, int(filter_pairs), None,
                                                   0, C.byref(cnt)))
        out = np.zeros((max(cnt.value, 1), 2), np.int32)
        _native.check(_native.lib().mp_joint_pairs(self.ctx, dg.handle, int(filter_pairs),
                                                   out.ctypes.data, cnt.value, C.byref(cnt)))
        return out[: cnt.value]

    # ---- non-overlap rows as LP text (K7, k_lp.cu) ------------------------------------
    def encode_addresses_lp(self, graph: Graph, lo, hi,
                            preplaced: Optional[Mapping[int, int]] = None,
                            want_counts: bool = False):
        """write_lp(encode_addresses(graph, lifetimes, preplaced)) (lp_format.cpp:88-121,
        encode.cpp:320-377): the external-ILP placement model as text, its pair rows
        built on the GPU from the K2 pair list. With want_counts also returns the
        constraint_counts of the model."""
        lo, hi = _i32(lo), _i32(hi)
        ids = [s.encode() for s in graph.edge_ids]
        blob = b"".join(ids) or b"\0"
        off = np.zeros(graph.E + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in ids]) if ids else []
        pin = pa = None
        if preplaced:
            pin, pa = self._addr_arrays(graph, preplaced)
        n = C.c_int64()
        counts = np.zeros(4, np.int64)
        args = [self.ctx, graph.E, lo.ctypes.data, hi.ctypes.data, graph.edge_size.ctypes.data,
                None if pin is None else pin.ctypes.data, None if pa is None else pa.ctypes.data,
                blob, off.ctypes.data]
        _native.check(_native.lib().mp_encode_addresses_lp(*args, None, 0, C.byref(n),
                                                           counts.ctypes.data))
        buf = C.create_string_buffer(n.value + 1)
        _native.check(_native.lib().mp_encode_addresses_lp(*args, buf, n.value + 1, C.byref(n),
                                                           None))
        text = buf.raw[: n.value].decode()
        if want_counts:
            return text, {"live_pair": int(counts[0]), "below": int(counts[1]),
                          "above": int(counts[2]), "peak_address": int(counts[3])}
        return text

    # ---- arena baseline (K6, k_arena.cu) ----------------------------------------------
    def run_baseline_batch(self, graph: Graph, orders, best_fit: bool = False):
        """run_baseline (placement.cpp:150-180) over many orders at once ->
        (mr_peak u64[B], rs_at_peak u64[B], fragmentation f64[B], valid u8[B])."""
        dg = self.upload(graph)
        o = _i32(orders)
        if o.ndim == 1:
            o = o.reshape(1, -1)
        c = o.shape[0]
        mr = np.zeros(max(c, 1), np.uint64)
        rs = np.zeros(max(c, 1), np.uint64)
        fr = np.zeros(max(c, 1), np.float64)
        valid = np.zeros(max(c, 1), np.uint8)
        if o.shape[1] != graph.n:  # wrong length: not a topological order (graph.cpp:241)
            return mr[:c], rs[:c], fr[:c], valid[:c]
        _native.check(_native.lib().mp_run_baseline(self.ctx, dg.handle, o.ctypes.data, c,
                                                    int(best_fit), mr.ctypes.data, rs.ctypes.data,
                                                    fr.ctypes.data, valid.ctypes.data))
        return mr[:c], rs[:c], fr[:c], valid[:c]

    def run_baseline(self, graph: Graph, order: Sequence[int],
                     policy: str = "first_fit") -> "BaselineResult":
        """run_baseline (placement.cpp:150-180); InvalidOrder for a non-topological order."""
        if policy not in ("first_fit", "best_fit"):
            raise ValueError("policy is 'first_fit' or 'best_fit' (FitPolicy, placement.hpp:40)")
        mr, rs, fr, valid = self.run_baseline_batch(graph, [list(order)] if len(order) else
                                                    np.zeros((1, 0), np.int32),
                                                    best_fit=policy == "best_fit")
        if not valid[0]:
            raise errors.InvalidOrder("sequence is not a topological order of the graph")
        return BaselineResult(int(mr[0]), int(rs[0]), float(fr[0]))

    def run_baseline_d(self, dg: "DeviceGraph", d_orders, num_orders, best_fit, d_mr, d_rs,
                       d_frag, d_valid, stream: int | None = None) -> None:
        _native.check(_native.lib().mp_run_baseline_d(
            self.ctx, dg.handle, _native.ptr(d_orders), int(num_orders), int(best_fit),
            _native.ptr(d_mr), _native.ptr(d_rs), _native.ptr(d_frag), _native.ptr(d_valid),
            stream))

    # ---- placement heuristics (K5, k_place.cu) ---------------------------------------
    PLACE_PYRAMID = 1
    PLACE_PYRAMID_ONLY = 2

    def place_batch(self, graph: Graph, lo, hi, pyramid: bool = True, pyramid_only: bool = False,
                    preplaced: Optional[Mapping[int, int]] = None):
        """Batched placement over B lifetime vectors (lo/hi [B][E]): the
        preplaced map (preallocate_pyramid's when ``pyramid``) then greedy_pack
        (placement.cpp:25-62, 182-204). Returns (addr u64[B][E], has u8[B][E],
        peak_mem u64[B], pyramid_base u64[B])."""
        lo = np.ascontiguousarray(np.atleast_2d(lo), np.int32)
        hi = np.ascontiguousarray(np.atleast_2d(hi), np.int32)
        B, E = lo.shape[0], graph.E
        if lo.shape != (B, E) or hi.shape != (B, E):
            raise ValueError("lo/hi must be [B][num_edges]")
        flags = (self.PLACE_PYRAMID if pyramid else 0) | (self.PLACE_PYRAMID_ONLY if pyramid_only
                                                           else 0)
        fx = fa = None
        if preplaced:
            fx, fa = self._addr_arrays(graph, preplaced)
        addr = np.zeros((B, max(E, 1)), np.uint64)
        has = np.zeros((B, max(E, 1)), np.uint8)
        peak = np.zeros(max(B, 1), np.uint64)
        base = np.zeros(max(B, 1), np.uint64)
        _native.check(_native.lib().mp_place(
            self.ctx, E, B, lo.ctypes.data, hi.ctypes.data, graph.edge_size.ctypes.data,
            graph.id_rank().ctypes.data, None if fx is None else fx.ctypes.data,
            None if fa is None else fa.ctypes.data, flags, addr.ctypes.data, has.ctypes.data,
            peak.ctypes.data, base.ctypes.data))
        return addr[:, :E], has[:, :E], peak[:B], base[:B]

    def place_batch_d(self, num_edges, num_problems, d_lo, d_hi, d_size, d_id_rank, flags,
                      d_addr, d_has, d_peak=None, d_base=None, d_fixed=None, d_fixed_addr=None,
                      stream: int | None = None) -> None:
        """Device-pointer form of place_batch (mp_place_d), stream-ordered."""
        _native.check(_native.lib().mp_place_d(
            self.ctx, int(num_edges), int(num_problems), _native.ptr(d_lo), _native.ptr(d_hi),
            _native.ptr(d_size), _native.ptr(d_id_rank), _native.ptr(d_fixed),
            _native.ptr(d_fixed_addr), int(flags), _native.ptr(d_addr), _native.ptr(d_has),
            _native.ptr(d_peak), _native.ptr(d_base), stream))

    def preallocate_pyramid(self, graph: Graph, lo, hi) -> "PrePlacement":
        """preallocate_pyramid (placement.cpp:25-62) -> PrePlacement."""
        addr, has, _, base = self.place_batch(graph, lo, hi, pyramid=True, pyramid_only=True)
        assigned = {int(e): int(addr[0, e]) for e in np.nonzero(has[0])[0]}
        remaining = [e for e in range(graph.E) if graph.edge_size[e] > 0 and e not in assigned]
        return PrePlacement(assigned, remaining, int(base[0]))

    def greedy_pack(self, graph: Graph, lo, hi,
                    preplaced: Optional[Mapping[int, int]] = None) -> dict:
        """greedy_pack (placement.cpp:182-204): {edge index: address} incl. preplaced."""
        addr, has, _, _ = self.place_batch(graph, lo, hi, pyramid=False, preplaced=preplaced or {})
        return {int(e): int(addr[0, e]) for e in np.nonzero(has[0])[0]}

    @staticmethod
    def _addr_arrays(graph: Graph, addresses: Mapping[int, int]):
        has = np.zeros(max(graph.E, 1), np.uint8)
        ad = np.zeros(max(graph.E, 1), np.uint64)
        for e, a in addresses.items():
            has[e] = 1
            ad[e] = a
        return has, ad

    def validate_plan(self, plan: MemoryPlan, graph: Graph) -> list[tuple[str, str]]:
        """validate_plan (plan.cpp:315-419): the same violations in the same order.

        Coverage / ordering / address-bound bookkeeping is host-side report
        assembly over ids; realized lifetimes, the O(E^2) pairwise check and
        the peak resident bytes run on the device.
        """
        out: list[tuple[str, str]] = []
        fail = lambda tag, detail: out.append((tag, detail))  # noqa: E731
        seen: dict[str, int] = {}
        for sid in plan.sequence.steps:
            if not graph.has_node(sid):
                fail("create_once", f"sequence names unknown node '{sid}'")
                continue
            seen[sid] = seen.get(sid, 0) + 1
            if seen[sid] == 2:
                fail("create_once", f"node '{sid}' appears more than once")
        for nid in graph.node_ids:
            if nid not in seen:
                fail("create_once", f"node '{nid}' is missing from the sequence")
        horizon = graph.n
        ts = plan.sequence.timestep_of
        step_of = lambda k: ts.get(k, 0)  # noqa: E731
        for sid in plan.sequence.steps:
            t = step_of(sid)
            if t <= 0:
                fail("create_once", f"node '{sid}' has no timestep")
            else:
                horizon = max(horizon, t)
        order_ok = True
        node_ids = graph.node_ids
        for e in range(graph.E):
            src_id = node_ids[graph.source_of(e)]
            t_src = step_of(src_id)
            for w in graph.sinks_of(e):
                t_sink = step_of(node_ids[w])
                if t_src <= 0 or t_sink <= 0:
                    continue
                if t_sink <= t_src:
                    fail("fanin_in_memory", f"edge '{graph.edge_ids[e]}': consumer '{node_ids[w]}'"
                         f" does not run after producer '{src_id}'")
                    order_ok = False
        mask64 = (1 << 64) - 1
        for aid in sorted(plan.addresses):
            addr = plan.addresses[aid]
            if not graph.has_edge(aid):
                fail("peak_address", f"address for unknown tensor '{aid}'")
                continue
            end = (addr + int(graph.edge_size[graph.edge_index(aid)])) & mask64
            if end > plan.peak_mem:
                fail("peak_address", f"tensor '{aid}' ends at {end}, above peak_mem {plan.peak_mem}")
        for e in range(graph.E):
            if graph.edge_size[e] > 0 and graph.edge_ids[e] not in plan.addresses:
                fail("peak_address", f"tensor '{graph.edge_ids[e]}' has no address")
        if not order_ok:
            return out
        for nid in node_ids:
            if step_of(nid) <= 0:
                return out
        lo, hi = self.realized_lifetimes(graph, ts, horizon)
        has = np.zeros(max(graph.E, 1), np.uint8)
        ad = np.zeros(max(graph.E, 1), np.uint64)
        for e, eid in enumerate(graph.edge_ids):
            if eid in plan.addresses:
                has[e] = 1
                ad[e] = plan.addresses[eid] & mask64
        for i, j in self.conflicting_pairs(lo, hi, graph.edge_size, has[:graph.E],
                                           ad[:graph.E]).tolist():
            fail("below_above", f"tensors '{graph.edge_ids[i]}' and '{graph.edge_ids[j]}' are "
                 "live together and overlap in memory")
        peak_rs = self.timeline_from_lifetimes(graph, lo, hi, horizon).peak_rs
        if plan.peak_mem < peak_rs:
            fail("peak_mem", f"peak_mem {plan.peak_mem} is below the peak resident bytes {peak_rs}")
        if plan.peak_rs != peak_rs:
            fail("peak_mem", f"stored peak_rs {plan.peak_rs} differs from the recomputed {peak_rs}")
        return out


def format_report(violations: list[tuple[str, str]]) -> str:
    """plan.cpp:421-427."""
    if not violations:
        return "ok\n"
    return "".join(f"{tag}  {detail}\n" for tag, detail in violations)


def random_topo_orders(graph: Graph, num_orders: int, seed: int = 0,
                       threads: int = 0) -> np.ndarray:
    """Seeded random topological orders (host C++ workload helper)."""
    out = np.zeros((max(num_orders, 1), max(graph.n, 1)), np.int32)
    csr = graph.mp_csr()
    _native.check(_native.lib().mp_random_topo_orders(C.byref(csr), int(num_orders), int(seed),
                                                      int(threads), out.ctypes.data))
    return out[:num_orders, :graph.n]


def parts_plan_info(graph: Graph, max_chunks: int = 0, smem_budget: int = 232448) -> dict:
    """Host-only: the node partition the large-graph scorer plans for `graph`
    (mp_parts_plan_host; no device needed)."""
    info = np.zeros(7, np.int64)
    csr = graph.mp_csr()
    _native.check(_native.lib().mp_parts_plan_host(C.byref(csr), int(max_chunks),
                                                   int(smem_budget), info.ctypes.data))
    keys = ("parts", "slots_per_part", "stash_slots", "cross_pairs", "cross_multi_consumer",
            "smem_bytes", "tiny4")
    return {k: int(v) for k, v in zip(keys, info)}


def prep_info(graph: Graph, with_pairs: bool = False):
    """Host-only: the scorer's derived tables for `graph` (mp_prep_host; no device):
    reduced validity pairs, order-dependent frees, which reachability was used.
    With with_pairs, also the reduced pairs as an int32 [m, 2] array (u before w)."""
    info = np.zeros(7, np.int64)
    csr = graph.mp_csr()
    _native.check(_native.lib().mp_prep_host(C.byref(csr), info.ctypes.data, None, 0))
    keys = ("reduced_pairs", "multi_consumer", "exact_reach", "tiny4", "tiny8", "narrow",
            "mid32")
    out = {k: int(v) for k, v in zip(keys, info)}
    if with_pairs:
        pairs = np.zeros((max(out["reduced_pairs"], 1), 2), np.int32)
        _native.check(_native.lib().mp_prep_host(C.byref(csr), info.ctypes.data,
                                                 pairs.ctypes.data, out["reduced_pairs"]))
        return out, pairs[:out["reduced_pairs"]]
    return out
