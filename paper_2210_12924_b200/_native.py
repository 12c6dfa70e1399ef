"""ctypes binding of the C ABI in include/memplan_b200.h.

The in-tree library ``paper_2210_12924_b200/lib/libmemplan_b200.so`` is the only
compute path. If it is missing this module raises on import of any compute
function — there is deliberately no pure-Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libmemplan_b200.so")
# MP_LIB selects a tuning build of the same sources (tools/gpu/variants.sh); never a fallback
LIB_PATH = os.environ.get("MP_LIB", LIB_PATH)

MP_OK = 0
MP_E_INVALID_ORDER = 1
MP_E_BAD_GRAPH = 2
MP_E_INVALID_ARG = 3
MP_E_CUDA = 4
MP_E_OOM = 5
MP_E_CAPACITY = 6
MP_E_NO_DEVICE = 7

# Every symbol include/memplan_b200.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "mp_abi_version", "mp_status_string", "mp_last_error",
    "mp_ctx_create", "mp_ctx_destroy", "mp_ctx_set_stream", "mp_ctx_synchronize",
    "mp_graph_upload", "mp_graph_free", "mp_graph_get_info",
    "mp_lifetimes", "mp_lifetimes_d", "mp_realized_lifetimes",
    "mp_resident_bytes", "mp_peak_resident_bytes", "mp_timeline",
    "mp_score_orders", "mp_score_orders_d", "mp_score_orders_best", "mp_score_orders_argmin_d",
    "mp_argmin", "mp_argmin_key_d", "mp_key_reset_d",
    "mp_overlap_pairs", "mp_overlap_pairs_d",
    "mp_validate_pairs", "mp_validate_pairs_d", "mp_addresses_feasible", "mp_peak_mem",
    "mp_fragmentation", "mp_generate_graph", "mp_random_topo_orders",
    "mp_place", "mp_place_d", "mp_run_baseline", "mp_run_baseline_d", "mp_encode_addresses_lp",
    "mp_joint_pairs", "mp_multi_create", "mp_multi_destroy", "mp_multi_upload",
    "mp_score_orders_multi", "mp_parts_plan_host", "mp_prep_host", "mp_score_plans_d", "mp_lifetimes_batch_d",
    "mp_validate_plans_d", "mp_multi_nccl",
]


class MpCsr(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int32),
        ("num_edges", C.c_int32),
        ("edge_src", C.c_void_p),
        ("sink_off", C.c_void_p),
        ("sinks", C.c_void_p),
        ("edge_size", C.c_void_p),
    ]


class MpGraphInfo(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int32),
        ("num_edges", C.c_int32),
        ("num_sinks", C.c_int64),
        ("num_pred_pairs", C.c_int64),
        ("num_multi_sink", C.c_int32),
        ("smem_resident", C.c_int32),
        ("total_bytes", C.c_uint64),
        ("orders16", C.c_int32),
        ("score_variant", C.c_int32),
    ]


_lib = None
_lock = threading.Lock()
vp = C.c_void_p
i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64
P = C.POINTER


def lib():
    """The loaded native library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise errors.DeviceError(
                f"memplan_b200 native library missing at {LIB_PATH}; run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        sig = {
            "mp_abi_version": (C.c_int, []),
            "mp_status_string": (C.c_char_p, [C.c_int]),
            "mp_last_error": (C.c_char_p, []),
            "mp_ctx_create": (C.c_int, [C.c_int, P(vp)]),
            "mp_ctx_destroy": (C.c_int, [vp]),
            "mp_ctx_set_stream": (C.c_int, [vp, vp]),
            "mp_ctx_synchronize": (C.c_int, [vp]),
            "mp_graph_upload": (C.c_int, [vp, P(MpCsr), P(vp)]),
            "mp_graph_free": (C.c_int, [vp]),
            "mp_graph_get_info": (C.c_int, [vp, P(MpGraphInfo)]),
            "mp_lifetimes": (C.c_int, [vp, vp, vp, i64, vp, vp]),
            "mp_lifetimes_d": (C.c_int, [vp, vp, vp, i64, vp, vp, vp, vp]),
            "mp_realized_lifetimes": (C.c_int, [vp, vp, vp, i32, vp, vp, P(i32)]),
            "mp_resident_bytes": (C.c_int, [vp, vp, vp, i64, vp]),
            "mp_peak_resident_bytes": (C.c_int, [vp, vp, vp, i64, P(u64)]),
            "mp_timeline": (C.c_int, [vp, vp, vp, vp, i32, vp, P(u64), P(i32)]),
            "mp_score_orders": (C.c_int, [vp, vp, vp, i64, vp, vp, vp]),
            "mp_score_orders_d": (C.c_int, [vp, vp, vp, i64, vp, vp, vp, vp]),
            "mp_score_orders_best": (C.c_int, [vp, vp, vp, i64, vp, vp, vp, P(i64)]),
            "mp_score_orders_argmin_d": (C.c_int, [vp, vp, vp, i64, vp, vp, vp, vp, i64, vp]),
            "mp_argmin": (C.c_int, [vp, vp, vp, i64, P(i64)]),
            "mp_argmin_key_d": (C.c_int, [vp, vp, vp, i64, i64, vp, vp]),
            "mp_key_reset_d": (C.c_int, [vp, vp, vp]),
            "mp_overlap_pairs": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, i64, P(i64)]),
            "mp_overlap_pairs_d": (C.c_int, [vp, i32, vp, vp, vp, vp, i64, i64, vp, vp, i64,
                                             P(i64), vp]),
            "mp_validate_pairs": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, vp, i64, P(i64)]),
            "mp_validate_pairs_d": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, i64, i64, vp, vp,
                                              i64, P(i64), vp]),
            "mp_addresses_feasible": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, P(i32)]),
            "mp_peak_mem": (C.c_int, [vp, i32, vp, vp, vp, P(u64)]),
            "mp_fragmentation": (C.c_double, [u64, u64]),
            "mp_multi_create": (C.c_int, [vp, C.c_int, P(vp)]),
            "mp_multi_destroy": (C.c_int, [vp]),
            "mp_multi_nccl": (C.c_int, [vp]),
            "mp_multi_upload": (C.c_int, [vp, P(MpCsr)]),
            "mp_score_orders_multi": (C.c_int, [vp, vp, i64, vp, vp, vp, P(i64)]),
            "mp_joint_pairs": (C.c_int, [vp, vp, C.c_int, vp, i64, P(i64)]),
            "mp_encode_addresses_lp": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, i64,
                                                 P(i64), vp]),
            "mp_run_baseline": (C.c_int, [vp, vp, vp, i64, C.c_int, vp, vp, vp, vp]),
            "mp_run_baseline_d": (C.c_int, [vp, vp, vp, i64, C.c_int, vp, vp, vp, vp, vp]),
            "mp_place": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, vp, vp, C.c_uint32, vp, vp,
                                   vp, vp]),
            "mp_place_d": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, vp, vp, C.c_uint32, vp, vp,
                                     vp, vp, vp]),
            "mp_generate_graph": (C.c_int, [C.c_int, i32, u64, u64, P(i32), P(i32), P(i64), vp,
                                            vp, vp, vp, vp]),
            "mp_random_topo_orders": (C.c_int, [P(MpCsr), i64, u64, i32, vp]),
            "mp_parts_plan_host": (C.c_int, [P(MpCsr), i32, i64, vp]),
            "mp_prep_host": (C.c_int, [P(MpCsr), vp, vp, i64]),
            "mp_score_plans_d": (C.c_int, [vp, vp, vp, i64, vp, C.c_uint32, vp, vp, vp, vp, vp,
                                           vp, vp, vp, i64, vp]),
            "mp_lifetimes_batch_d": (C.c_int, [vp, vp, vp, i64, vp, vp, vp, vp]),
            "mp_validate_plans_d": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return _lib


def last_error() -> str:
    return lib().mp_last_error().decode()


def check(status: int) -> None:
    """Raise the reference-style exception for a non-OK status."""
    if status == MP_OK:
        return
    msg = last_error()
    if status == MP_E_INVALID_ORDER:
        raise errors.InvalidOrder(msg)
    if status == MP_E_BAD_GRAPH:
        name = msg.split(":", 1)[0]
        cls = getattr(errors, name, errors.InvalidStructure)
        raise cls(msg)
    if status == MP_E_INVALID_ARG:
        raise ValueError(msg)
    if status == MP_E_CAPACITY:
        raise errors.Capacity(msg)
    raise errors.DeviceError(msg or lib().mp_status_string(status).decode())


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
