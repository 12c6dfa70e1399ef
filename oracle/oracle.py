"""TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.

ctypes access to
  * ``oracle/_build/liboracle.so``  — the plain-C restatement (memplan_oracle.c),
  * ``oracle/_ref/libmemplan_ref.so`` — the unmodified reference planner compiled
    from /root/reference/proj/src (oracle/Makefile) plus the ref_capi.cpp harness.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmemplan_ref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p


def build(quiet: bool = True) -> None:
    """Compile the C restatement and (when /root/reference exists) the reference."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _c(a, dt):
    return np.ascontiguousarray(a, dt)


def _opt_ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# C restatement
# ---------------------------------------------------------------------------
class OrGraph(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("num_edges", C.c_int32),
        ("edge_src", C.c_void_p),
        ("sink_off", C.c_void_p),
        ("sinks", C.c_void_p),
        ("edge_size", C.c_void_p),
    ]


_olib = None


def olib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        gp = C.POINTER(OrGraph)
        lib.or_is_topological_order.argtypes = [gp, _i32p, C.c_int64]
        lib.or_lifetimes_from_order.argtypes = [gp, _i32p, C.c_int64, _i32p, _i32p]
        lib.or_resident_bytes_per_step.argtypes = [gp, _i32p, C.c_int64, _u64p]
        lib.or_peak_resident_bytes.argtypes = [gp, _i32p, C.c_int64, C.POINTER(C.c_uint64)]
        lib.or_timeline_from_lifetimes.argtypes = [gp, _i32p, _i32p, C.c_int32, _vp,
                                                   C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]
        lib.or_realized_lifetimes.argtypes = [gp, _i32p, C.c_int32, _i32p, _i32p,
                                              C.POINTER(C.c_int32)]
        lib.or_overlap_pairs.argtypes = [C.c_int32, _i32p, _i32p, _u64p, _vp, _vp, C.c_int64]
        lib.or_overlap_pairs.restype = C.c_int64
        lib.or_overlap_row_stats.argtypes = [C.c_int32, _i32p, _i32p, _u64p, _vp,
                                             C.c_int64, C.c_int64, _i64p, _u64p]
        lib.or_validate_pairs.argtypes = [C.c_int32, _i32p, _i32p, _u64p, _u8p, _u64p,
                                          _vp, C.c_int64]
        lib.or_validate_pairs.restype = C.c_int64
        lib.or_addresses_feasible.argtypes = [C.c_int32, _i32p, _i32p, _u64p, _u8p, _u64p]
        lib.or_fragmentation.argtypes = [C.c_uint64, C.c_uint64]
        lib.or_fragmentation.restype = C.c_double
        lib.or_peak_mem.argtypes = [C.c_int32, _u64p, _u8p, _u64p]
        lib.or_peak_mem.restype = C.c_uint64
        lib.or_preallocate_pyramid.argtypes = [C.c_int32, _i32p, _i32p, _u64p, _i32p, _u8p, _u64p]
        lib.or_preallocate_pyramid.restype = C.c_uint64
        lib.or_greedy_pack.argtypes = [C.c_int32, _i32p, _i32p, _u64p, _vp, _u64p, _u8p]
        lib.or_joint_pairs.argtypes = [gp, C.c_int, _vp, C.c_int64]
        lib.or_joint_pairs.restype = C.c_int64
        lib.or_run_baseline.argtypes = [gp, _i32p, C.c_int64, C.c_int, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        _olib = lib
    return _olib


class Oracle:
    """C restatement bound to one CSR graph (arrays kept alive here)."""

    def __init__(self, n, edge_src, sink_off, sinks, edge_size):
        self.n = int(n)
        self.src = np.ascontiguousarray(edge_src, np.int32)
        self.sink_off = np.ascontiguousarray(sink_off, np.int64)
        self.sinks = np.ascontiguousarray(sinks, np.int32)
        self.size = np.ascontiguousarray(edge_size, np.uint64)
        self.E = int(self.src.shape[0])
        self._g = OrGraph(self.n, self.E, self.src.ctypes.data, self.sink_off.ctypes.data,
                          self.sinks.ctypes.data, self.size.ctypes.data)

    @classmethod
    def from_csr(cls, csr):
        return cls(csr["n"], csr["edge_src"], csr["sink_off"], csr["sinks"], csr["edge_size"])

    def is_topological_order(self, order):
        o = np.ascontiguousarray(order, np.int32)
        return bool(olib().or_is_topological_order(C.byref(self._g), o, o.size))

    def lifetimes_from_order(self, order):
        o = np.ascontiguousarray(order, np.int32)
        lo = np.zeros(self.E, np.int32)
        hi = np.zeros(self.E, np.int32)
        if olib().or_lifetimes_from_order(C.byref(self._g), o, o.size, lo, hi):
            return None
        return lo, hi

    def resident_bytes_per_step(self, order):
        o = np.ascontiguousarray(order, np.int32)
        out = np.zeros(max(self.n, 1), np.uint64)
        if olib().or_resident_bytes_per_step(C.byref(self._g), o, o.size, out):
            return None
        return out[: self.n]

    def peak_resident_bytes(self, order):
        o = np.ascontiguousarray(order, np.int32)
        p = C.c_uint64()
        if olib().or_peak_resident_bytes(C.byref(self._g), o, o.size, C.byref(p)):
            return None
        return int(p.value)

    def timeline_from_lifetimes(self, lo, hi, horizon, want_bytes=True):
        lo = np.ascontiguousarray(lo, np.int32)
        hi = np.ascontiguousarray(hi, np.int32)
        b = np.zeros(max(horizon, 1), np.uint64) if want_bytes else None
        pr, ps = C.c_uint64(), C.c_int32()
        olib().or_timeline_from_lifetimes(C.byref(self._g), lo, hi, int(horizon), _opt_ptr(b),
                                          C.byref(pr), C.byref(ps))
        return (b[:horizon] if want_bytes else None), int(pr.value), int(ps.value)

    def joint_pairs(self, filter_pairs=True):
        """encode_joint's pair set (encode.cpp:401-408) -> int32[P][2]."""
        cnt = olib().or_joint_pairs(C.byref(self._g), int(filter_pairs), None, 0)
        out = np.zeros((max(cnt, 1), 2), np.int32)
        olib().or_joint_pairs(C.byref(self._g), int(filter_pairs), out.ctypes.data, cnt)
        return out[:cnt]

    def run_baseline(self, order, best_fit=False):
        """placement.cpp:150-180 -> (mr_peak, rs_at_peak, fragmentation) or None (invalid)."""
        mr, rs, fr = C.c_uint64(), C.c_uint64(), C.c_double()
        o = _c(order, np.int32)
        if olib().or_run_baseline(C.byref(self._g), o, len(o), int(best_fit), C.byref(mr), C.byref(rs),
                                  C.byref(fr)):
            return None
        return mr.value, rs.value, fr.value

    def realized_lifetimes(self, timestep_of, horizon):
        ts = np.ascontiguousarray(timestep_of, np.int32)
        lo = np.zeros(self.E, np.int32)
        hi = np.zeros(self.E, np.int32)
        miss = C.c_int32(-1)
        if olib().or_realized_lifetimes(C.byref(self._g), ts, int(horizon), lo, hi, C.byref(miss)):
            return ("missing", int(miss.value))
        return lo, hi


def timeline_peak(lo, hi, size, horizon):
    """(peak_rs, peak_step) of timeline_from_lifetimes (plan.cpp:122-143) in O(E + h):
    RS(t) = sum of size over lo <= t <= hi as a difference array + prefix sum, then
    the first strict maximum (1 when all zero and horizon > 0, 0 when horizon == 0).
    Same definition as or_timeline_from_lifetimes (its literal O(h*E) loop is too
    slow at 100k tensors); tests/test_oracle_golden.py checks the two agree."""
    if horizon <= 0:
        return 0, 0
    lo = np.asarray(lo, np.int64)
    hi = np.asarray(hi, np.int64)
    sz = np.asarray(size, np.uint64).astype(np.int64)   # totals < 2^62 (graph.cpp:122-128)
    d = np.zeros(horizon + 2, np.int64)
    a = np.clip(lo, 1, horizon + 1)
    b = np.clip(hi + 1, 1, horizon + 1)
    keep = (lo <= hi) & (sz > 0) & (lo <= horizon)
    np.add.at(d, a[keep], sz[keep])
    np.add.at(d, b[keep], -sz[keep])
    rs = np.cumsum(d)[1:horizon + 1]
    best = int(rs.max())
    return best, (int(np.argmax(rs)) + 1 if best > 0 else 1)


def overlap_pairs(lo, hi, size, pinned=None, want_pairs=True):
    lo = np.ascontiguousarray(lo, np.int32)
    hi = np.ascontiguousarray(hi, np.int32)
    size = np.ascontiguousarray(size, np.uint64)
    pin = None if pinned is None else np.ascontiguousarray(pinned, np.uint8)
    E = lo.size
    cnt = olib().or_overlap_pairs(E, lo, hi, size, _opt_ptr(pin), None, 0)
    if not want_pairs:
        return cnt
    out = np.zeros((max(cnt, 1), 2), np.int32)
    olib().or_overlap_pairs(E, lo, hi, size, _opt_ptr(pin), out.ctypes.data_as(C.c_void_p), cnt)
    return out[:cnt]


def overlap_row_stats(lo, hi, size, pinned=None, rows=None):
    lo = np.ascontiguousarray(lo, np.int32)
    hi = np.ascontiguousarray(hi, np.int32)
    size = np.ascontiguousarray(size, np.uint64)
    pin = None if pinned is None else np.ascontiguousarray(pinned, np.uint8)
    E = lo.size
    r0, r1 = (0, E) if rows is None else rows
    cnt = np.zeros(max(r1 - r0, 1), np.int64)
    hsh = np.zeros(max(r1 - r0, 1), np.uint64)
    olib().or_overlap_row_stats(E, lo, hi, size, _opt_ptr(pin), r0, r1, cnt, hsh)
    return cnt[: r1 - r0], hsh[: r1 - r0]


def validate_pairs(lo, hi, size, has_addr, addr):
    lo = np.ascontiguousarray(lo, np.int32)
    hi = np.ascontiguousarray(hi, np.int32)
    size = np.ascontiguousarray(size, np.uint64)
    has = np.ascontiguousarray(has_addr, np.uint8)
    addr = np.ascontiguousarray(addr, np.uint64)
    E = lo.size
    cnt = olib().or_validate_pairs(E, lo, hi, size, has, addr, None, 0)
    out = np.zeros((max(cnt, 1), 2), np.int32)
    olib().or_validate_pairs(E, lo, hi, size, has, addr, out.ctypes.data_as(C.c_void_p), cnt)
    return out[:cnt]


def addresses_feasible(lo, hi, size, has_addr, addr):
    return bool(olib().or_addresses_feasible(
        len(lo), np.ascontiguousarray(lo, np.int32), np.ascontiguousarray(hi, np.int32),
        np.ascontiguousarray(size, np.uint64), np.ascontiguousarray(has_addr, np.uint8),
        np.ascontiguousarray(addr, np.uint64)))


def preallocate_pyramid(lo, hi, size, id_rank):
    """placement.cpp:25-62 -> (taken u8[E], addr u64[E], reserved_base)."""
    E = len(size)
    taken = np.zeros(max(E, 1), np.uint8)
    addr = np.zeros(max(E, 1), np.uint64)
    base = olib().or_preallocate_pyramid(E, _c(lo, np.int32), _c(hi, np.int32),
                                         _c(size, np.uint64), _c(id_rank, np.int32), taken, addr)
    return taken[:E], addr[:E], int(base)


def greedy_pack(lo, hi, size, fixed=None, fixed_addr=None):
    """placement.cpp:182-204 -> (addr u64[E], has u8[E]); fixed = preplaced map."""
    E = len(size)
    addr = np.zeros(max(E, 1), np.uint64)
    has = np.zeros(max(E, 1), np.uint8)
    if fixed is not None:
        addr[:E] = fixed_addr
    fx = None if fixed is None else _c(fixed, np.uint8)
    olib().or_greedy_pack(E, _c(lo, np.int32), _c(hi, np.int32), _c(size, np.uint64),
                          _opt_ptr(fx), addr, has)
    return addr[:E], has[:E]


def fragmentation(mr, rs):
    return float(olib().or_fragmentation(int(mr), int(rs)))


def peak_mem(size, has_addr, addr):
    return int(olib().or_peak_mem(len(size), np.ascontiguousarray(size, np.uint64),
                                  np.ascontiguousarray(has_addr, np.uint8),
                                  np.ascontiguousarray(addr, np.uint64)))


# ---------------------------------------------------------------------------
# The reference itself
# ---------------------------------------------------------------------------
REF_OK, REF_INVALID_ORDER, REF_ERROR, REF_CAPACITY, REF_UNKNOWN = range(5)
KIND = {"chain": 0, "fork_join": 1, "training_like": 2}

_rlib = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def rlib():
    global _rlib
    if _rlib is None:
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise RuntimeError("reference library unavailable (no /root/reference and no prebuilt "
                               "oracle/_ref/libmemplan_ref.so)")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_load_graph.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        lib.ref_generate_graph.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                           C.POINTER(C.c_void_p)]
        lib.ref_graph_free.argtypes = [_vp]
        lib.ref_save_graph.argtypes = [_vp, _vp, C.c_int64, C.POINTER(C.c_int64)]
        lib.ref_graph_dims.argtypes = [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int64)]
        lib.ref_graph_csr.argtypes = [_vp, _i32p, _i64p, _i32p, _u64p, _u8p]
        lib.ref_is_topological_order.argtypes = [_vp, _i32p, C.c_int64]
        lib.ref_topological_order.argtypes = [_vp, _i32p]
        lib.ref_lifetimes_from_order.argtypes = [_vp, _i32p, C.c_int64, _i32p, _i32p]
        lib.ref_resident_bytes_per_step.argtypes = [_vp, _i32p, C.c_int64, _u64p]
        lib.ref_peak_resident_bytes.argtypes = [_vp, _i32p, C.c_int64, C.POINTER(C.c_uint64)]
        lib.ref_score_orders.argtypes = [_vp, _i32p, C.c_int64, C.c_int64, _u64p, _u8p, C.c_int,
                                         C.POINTER(C.c_int64)]
        lib.ref_random_topo_orders.argtypes = [_vp, C.c_int64, C.c_uint64, C.c_int, _i32p]
        lib.ref_timeline_from_lifetimes.argtypes = [_vp, _i32p, _i32p, C.c_int32, _vp,
                                                    C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]
        lib.ref_realized_lifetimes.argtypes = [_vp, _i32p, C.c_int32, _i32p, _i32p]
        lib.ref_encode_address_pairs.argtypes = [_vp, _i32p, _i32p, _vp, _vp, C.c_int, _vp,
                                                 C.c_int64, C.POINTER(C.c_int64)]
        lib.ref_validate_plan.argtypes = [_vp, _i32p, C.c_int64, _i32p, _u8p, _u64p, C.c_uint64,
                                          C.c_uint64, C.c_int32, _vp, C.c_int64,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        lib.ref_greedy_pack.argtypes = [_vp, _i32p, _i32p, _u64p]
        lib.ref_joint_pairs.argtypes = [_vp, C.c_int, _vp, C.c_int64, C.POINTER(C.c_int64)]
        lib.ref_encode_addresses_lp.argtypes = [_vp, _i32p, _i32p, _vp, _vp, C.c_int, _vp,
                                                C.c_int64, C.POINTER(C.c_int64)]
        lib.ref_preallocate_pyramid.argtypes = [_vp, _i32p, _i32p, _u8p, _u64p,
                                                C.POINTER(C.c_uint64)]
        lib.ref_greedy_pack_fixed.argtypes = [_vp, _i32p, _i32p, _vp, _vp, _u64p, _u8p]
        lib.ref_run_baseline.argtypes = [_vp, _i32p, C.c_int64, C.c_int, C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        lib.ref_fragmentation.argtypes = [C.c_uint64, C.c_uint64]
        lib.ref_fragmentation.restype = C.c_double
        lib.ref_enumerate_min_peak.argtypes = [_vp, C.POINTER(C.c_uint64), _i32p]
        lib.ref_plan_graph.argtypes = [_vp, _vp, C.c_int64, C.POINTER(C.c_int64)]
        _rlib = lib
    return _rlib


class RefError(Exception):
    """A memplan::Error raised inside the reference; ``str`` is its what()."""

    def __init__(self, status, text):
        super().__init__(text)
        self.status = status
        self.text = text


def _check(status):
    if status != REF_OK:
        raise RefError(status, rlib().ref_last_error().decode())


def _text_call(fn, *args):
    n = C.c_int64()
    _check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


class RefGraph:
    """A memplan::Graph living inside the reference library."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        n, e, s = C.c_int32(), C.c_int32(), C.c_int64()
        rlib().ref_graph_dims(self._h, C.byref(n), C.byref(e), C.byref(s))
        self.n, self.E, self.S = n.value, e.value, s.value

    def __del__(self):
        if getattr(self, "_h", None) and _rlib is not None:
            _rlib.ref_graph_free(self._h)
            self._h = None

    @classmethod
    def load(cls, text: str):
        h = C.c_void_p()
        _check(rlib().ref_load_graph(text.encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def load_file(cls, path: str):
        with open(path) as f:
            return cls.load(f.read())

    @classmethod
    def generate(cls, kind: str, layers: int, size: int = 8, seed: int = 0):
        h = C.c_void_p()
        _check(rlib().ref_generate_graph(KIND[kind], layers, size, seed, C.byref(h)))
        return cls(h.value)

    def save(self) -> str:
        return _text_call(rlib().ref_save_graph, self._h)

    def csr(self):
        src = np.zeros(self.E, np.int32)
        off = np.zeros(self.E + 1, np.int64)
        sinks = np.zeros(max(self.S, 1), np.int32)
        size = np.zeros(self.E, np.uint64)
        ctrl = np.zeros(self.E, np.uint8)
        rlib().ref_graph_csr(self._h, src, off, sinks, size, ctrl)
        return {"n": self.n, "edge_src": src, "sink_off": off, "sinks": sinks[: self.S],
                "edge_size": size, "is_control": ctrl}

    def is_topological_order(self, order):
        o = np.ascontiguousarray(order, np.int32)
        return bool(rlib().ref_is_topological_order(self._h, o, o.size))

    def topological_order(self):
        out = np.zeros(max(self.n, 1), np.int32)
        k = rlib().ref_topological_order(self._h, out)
        return out[:k]

    def lifetimes_from_order(self, order):
        o = np.ascontiguousarray(order, np.int32)
        lo = np.zeros(max(self.E, 1), np.int32)
        hi = np.zeros(max(self.E, 1), np.int32)
        _check(rlib().ref_lifetimes_from_order(self._h, o, o.size, lo, hi))
        return lo[: self.E], hi[: self.E]

    def resident_bytes_per_step(self, order):
        o = np.ascontiguousarray(order, np.int32)
        out = np.zeros(max(self.n, 1), np.uint64)
        _check(rlib().ref_resident_bytes_per_step(self._h, o, o.size, out))
        return out[: self.n]

    def peak_resident_bytes(self, order):
        o = np.ascontiguousarray(order, np.int32)
        p = C.c_uint64()
        _check(rlib().ref_peak_resident_bytes(self._h, o, o.size, C.byref(p)))
        return int(p.value)

    def random_topo_orders(self, num_orders, seed=0, threads=1):
        """Seeded randomised-Kahn candidates (input preparation for the reference arm;
        the same draws as paper_2210_12924_b200.random_topo_orders)."""
        out = np.zeros((num_orders, self.n), np.int32)
        _check(rlib().ref_random_topo_orders(self._h, num_orders, seed, threads, out))
        return out

    def score_orders(self, orders, threads=1):
        orders = np.ascontiguousarray(orders, np.int32)
        c, n = orders.shape
        peak = np.zeros(max(c, 1), np.uint64)
        valid = np.zeros(max(c, 1), np.uint8)
        best = C.c_int64()
        _check(rlib().ref_score_orders(self._h, orders, c, n, peak, valid, threads, C.byref(best)))
        return peak[:c], valid[:c], int(best.value)

    def timeline_from_lifetimes(self, lo, hi, horizon):
        lo = np.ascontiguousarray(lo, np.int32)
        hi = np.ascontiguousarray(hi, np.int32)
        b = np.zeros(max(horizon, 1), np.uint64)
        pr, ps = C.c_uint64(), C.c_int32()
        _check(rlib().ref_timeline_from_lifetimes(self._h, lo, hi, int(horizon),
                                                  b.ctypes.data_as(C.c_void_p), C.byref(pr),
                                                  C.byref(ps)))
        return b[:horizon], int(pr.value), int(ps.value)

    def joint_pairs(self, filter_pairs=True):
        """encode_joint's pair set (encode.cpp:401-408) -> int32[P][2]."""
        cnt = olib().or_joint_pairs(C.byref(self._g), int(filter_pairs), None, 0)
        out = np.zeros((max(cnt, 1), 2), np.int32)
        olib().or_joint_pairs(C.byref(self._g), int(filter_pairs), out.ctypes.data, cnt)
        return out[:cnt]

    def run_baseline(self, order, best_fit=False):
        """placement.cpp:150-180 -> (mr_peak, rs_at_peak, fragmentation) or None (invalid)."""
        mr, rs, fr = C.c_uint64(), C.c_uint64(), C.c_double()
        o = _c(order, np.int32)
        if olib().or_run_baseline(C.byref(self._g), o, len(o), int(best_fit), C.byref(mr), C.byref(rs),
                                  C.byref(fr)):
            return None
        return mr.value, rs.value, fr.value

    def realized_lifetimes(self, timestep_of, horizon):
        ts = np.ascontiguousarray(timestep_of, np.int32)
        lo = np.zeros(max(self.E, 1), np.int32)
        hi = np.zeros(max(self.E, 1), np.int32)
        _check(rlib().ref_realized_lifetimes(self._h, ts, int(horizon), lo, hi))
        return lo[: self.E], hi[: self.E]

    def encode_address_pairs(self, lo, hi, pinned=None, pinned_addr=None, filter_pairs=True,
                             want_pairs=True):
        lo = np.ascontiguousarray(lo, np.int32)
        hi = np.ascontiguousarray(hi, np.int32)
        pin = None if pinned is None else np.ascontiguousarray(pinned, np.uint8)
        pa = None if pinned_addr is None else np.ascontiguousarray(pinned_addr, np.uint64)
        cnt = C.c_int64()
        _check(rlib().ref_encode_address_pairs(self._h, lo, hi, _opt_ptr(pin), _opt_ptr(pa),
                                               int(filter_pairs), None, 0, C.byref(cnt)))
        if not want_pairs:
            return cnt.value
        out = np.zeros((max(cnt.value, 1), 2), np.int32)
        _check(rlib().ref_encode_address_pairs(self._h, lo, hi, _opt_ptr(pin), _opt_ptr(pa),
                                               int(filter_pairs), out.ctypes.data_as(C.c_void_p),
                                               cnt.value, C.byref(cnt)))
        return out[: cnt.value]

    def joint_pairs(self, filter_pairs=True):
        """encode_joint's pair set (encode.cpp:401-408) from the reference -> int32[P][2]."""
        cnt = C.c_int64()
        _check(rlib().ref_joint_pairs(self._h, int(filter_pairs), None, 0, C.byref(cnt)))
        out = np.zeros((max(cnt.value, 1), 2), np.int32)
        _check(rlib().ref_joint_pairs(self._h, int(filter_pairs), out.ctypes.data_as(C.c_void_p),
                                      cnt.value, C.byref(cnt)))
        return out[: cnt.value]

    def encode_addresses_lp(self, lo, hi, pinned=None, pinned_addr=None, filter_pairs=True):
        """write_lp(encode_addresses(...)) from the reference, as text."""
        pin = None if pinned is None else _c(pinned, np.uint8)
        pa = None if pinned_addr is None else _c(pinned_addr, np.uint64)
        return _text_call(rlib().ref_encode_addresses_lp, self._h, _c(lo, np.int32),
                          _c(hi, np.int32), _opt_ptr(pin), _opt_ptr(pa), int(filter_pairs))

    def validate_plan(self, sequence, timestep_of, has_addr, addr, peak_mem, stored_peak_rs,
                      stored_peak_step=0):
        seq = np.ascontiguousarray(sequence, np.int32)
        ts = np.ascontiguousarray(timestep_of, np.int32)
        has = np.ascontiguousarray(has_addr, np.uint8)
        ad = np.ascontiguousarray(addr, np.uint64)
        n = C.c_int64()
        nv = C.c_int32()
        lib = rlib()
        _check(lib.ref_validate_plan(self._h, seq, seq.size, ts, has, ad, int(peak_mem),
                                     int(stored_peak_rs), int(stored_peak_step), None, 0,
                                     C.byref(n), C.byref(nv)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib.ref_validate_plan(self._h, seq, seq.size, ts, has, ad, int(peak_mem),
                                     int(stored_peak_rs), int(stored_peak_step), buf,
                                     n.value + 1, C.byref(n), C.byref(nv)))
        lines = [ln for ln in buf.value.decode().split("\n") if ln]
        return [tuple(ln.split("\t", 1)) for ln in lines]

    def greedy_pack(self, lo, hi):
        out = np.zeros(max(self.E, 1), np.uint64)
        _check(rlib().ref_greedy_pack(self._h, np.ascontiguousarray(lo, np.int32),
                                      np.ascontiguousarray(hi, np.int32), out))
        return out[: self.E]

    def preallocate_pyramid(self, lo, hi):
        """-> (taken u8[E], addr u64[E], reserved_base) from the reference."""
        taken = np.zeros(max(self.E, 1), np.uint8)
        addr = np.zeros(max(self.E, 1), np.uint64)
        base = C.c_uint64()
        _check(rlib().ref_preallocate_pyramid(self._h, _c(lo, np.int32), _c(hi, np.int32), taken,
                                              addr, C.byref(base)))
        return taken[: self.E], addr[: self.E], base.value

    def greedy_pack_fixed(self, lo, hi, fixed=None, fixed_addr=None):
        """greedy_pack with a preplaced map -> (addr u64[E], has u8[E])."""
        addr = np.zeros(max(self.E, 1), np.uint64)
        has = np.zeros(max(self.E, 1), np.uint8)
        fx = None if fixed is None else _c(fixed, np.uint8)
        fa = None if fixed is None else _c(fixed_addr, np.uint64)
        _check(rlib().ref_greedy_pack_fixed(self._h, _c(lo, np.int32), _c(hi, np.int32),
                                            _opt_ptr(fx), _opt_ptr(fa), addr, has))
        return addr[: self.E], has[: self.E]

    def run_baseline(self, order, best_fit=False):
        """run_baseline (placement.cpp:150-180) -> (mr_peak, rs_at_peak, fragmentation)."""
        mr, rs, fr = C.c_uint64(), C.c_uint64(), C.c_double()
        o = _c(order, np.int32)
        _check(rlib().ref_run_baseline(self._h, o, len(o), int(best_fit), C.byref(mr),
                                       C.byref(rs), C.byref(fr)))
        return mr.value, rs.value, fr.value

    def enumerate_min_peak(self):
        p = C.c_uint64()
        out = np.zeros(max(self.n, 1), np.int32)
        _check(rlib().ref_enumerate_min_peak(self._h, C.byref(p), out))
        return int(p.value), out[: self.n]

    def plan_graph(self) -> str:
        return _text_call(rlib().ref_plan_graph, self._h)


def ref_fragmentation(mr, rs):
    return float(rlib().ref_fragmentation(int(mr), int(rs)))


# ---- LP text of the address model (pure Python restatement, small graphs) -----------
def _sanitize(name: str) -> str:
    """lp_format.cpp:30-36: every non-alphanumeric byte becomes '_'."""
    return "".join(c if c.isascii() and c.isalnum() else "_" for c in name)


def address_model_lp(edge_ids, lo, hi, size, pinned=None, pinned_addr=None) -> str:
    """write_lp(encode_addresses(graph, lifetimes, preplaced)) restated:
    encode.cpp:320-377 (variables, the pair loop, the below/above/live_pair rows with
    pinned addresses folded into the constant, encode.cpp:40-97 Row::emit) and
    lp_format.cpp:75-121 (lp_names with "_2" suffixes, the section layout)."""
    E = len(size)
    M = int(sum(int(s) for s in size))                      # Graph::total_bytes
    data = [e for e in range(E) if int(size[e]) > 0]
    pin = {e: int(pinned_addr[e]) for e in data if pinned is not None and pinned[e]}
    vars_ = [("peak_mem", "int", 0, M)]                     # objective first
    addr = {}
    for e in data:
        if e not in pin:
            addr[e] = len(vars_)
            vars_.append((f"addr({edge_ids[e]})", "int", 0, M))
    rows = []

    def emit(tag, rel, rhs, terms):                          # terms: (coef, var or pinned edge)
        const, out = 0, []
        for coef, v in terms:
            if isinstance(v, tuple):                         # ("pin", e)
                const += coef * pin[v[1]]
            else:
                out.append((coef, v))
        rows.append((tag, out, rel, rhs - const))

    def slot(e):
        return ("pin", e) if e in pin else addr[e]

    for a in range(len(data)):
        for b in range(a + 1, len(data)):
            i, j = data[a], data[b]
            if i in pin and j in pin:
                continue
            if lo[i] > hi[i] or lo[j] > hi[j] or hi[i] < lo[j] or hi[j] < lo[i]:
                continue                                     # intervals_disjoint
            below = len(vars_)
            vars_.append((f"below({edge_ids[i]},{edge_ids[j]})", "bin", 0, 1))
            above = len(vars_)
            vars_.append((f"above({edge_ids[i]},{edge_ids[j]})", "bin", 0, 1))
            emit("live_pair", "=", 1, [(1, below), (1, above)])
            emit("below", "<=", M - int(size[i]), [(1, slot(i)), (-1, slot(j)), (M, below)])
            emit("above", ">=", int(size[j]) - M, [(1, slot(i)), (-1, slot(j)), (-M, above)])
    for e in data:
        emit("peak_address", "<=", -int(size[e]), [(1, slot(e)), (-1, 0)])
    names, seen = [], set()
    for name, _, _, _ in vars_:                              # lp_names
        base = cand = _sanitize(name)
        k = 2
        while cand in seen:
            cand = f"{base}_{k}"
            k += 1
        seen.add(cand)
        names.append(cand)
    out = [f"Minimize\n obj: {names[0]}\nSubject To\n"]
    for r, (tag, terms, rel, rhs) in enumerate(rows):
        t = "".join(f" {'-' if c < 0 else '+'}{abs(c)} {names[v]}" for c, v in terms)
        out.append(f" c{r}_{tag}:{t} {rel} {rhs}\n")
    out.append("Bounds\n")
    out += [f" {lo_} <= {names[k]} <= {hi_}\n" for k, (_, kind, lo_, hi_) in enumerate(vars_)
            if kind == "int"]
    out.append("Generals\n")
    out += [f" {names[k]}\n" for k, v in enumerate(vars_) if v[1] == "int"]
    out.append("Binaries\n")
    out += [f" {names[k]}\n" for k, v in enumerate(vars_) if v[1] == "bin"]
    out.append("End\n")
    return "".join(out)
