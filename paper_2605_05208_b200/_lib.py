"""ctypes binding of libmdr_sm100.so (include/mdr_sm100.h).

The library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_2605_05208_b200/csrc`).  There is no CPU fallback: if the
library is missing or no CUDA device is present, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MDR_LIB") or os.path.join(_HERE, "libmdr_sm100.so")

MDR_OK, MDR_ERR_ARG, MDR_ERR_CONFLICT, MDR_ERR_CAPACITY, MDR_ERR_CUDA, MDR_ERR_PERMS = range(6)

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)


class CapacityError(RuntimeError):
    """A population capacity (routes, positions, followers) was exceeded."""


class InstanceDesc(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_depots", C.c_int32),
                ("dist", f64p), ("time", f64p), ("demand", f64p), ("service", f64p),
                ("tw_early", f64p), ("tw_late", f64p),
                ("capacity", C.c_double), ("max_duration", C.c_double), ("fleet_per_depot", C.c_double),
                ("open_routes", C.c_int32), ("has_windows", C.c_int32),
                ("gamma", C.c_double), ("theta", C.c_double),
                ("lists", i32p), ("width", C.c_int32)]


class Cands(C.Structure):
    _fields_ = [("n", C.c_int64)] + [(f, i64p) for f in
                                    ("r1", "p1", "r2", "p2", "len1", "len2", "depot", "mode")] + \
               [("rev1", u8p), ("rev2", u8p)]


class Deltas(C.Structure):
    _fields_ = [(f, f64p) for f in ("dD", "dV1", "dV2", "dV3", "dV4", "dF")] + [("fleet_neutral", u8p)]


class LsCfg(C.Structure):
    _fields_ = [("depth", C.c_int32), ("multi_move", C.c_int32), ("kappa", C.c_double),
                ("lam_min", C.c_double), ("lam_max", C.c_double), ("max_passes", C.c_int32),
                ("n_ops", C.c_int32), ("perms", u8p), ("deadline_s", C.c_double),
                ("rounds_per_sync", C.c_int32), ("use_graph", C.c_int32), ("snapshot_best", C.c_int32),
                ("trace", C.c_int32)]


class LsStats(C.Structure):
    _fields_ = [("passes", C.c_int32), ("accepted", C.c_int32), ("op_evals", C.c_int32),
                ("status", C.c_int32), ("cands", C.c_int64 * 6), ("moves_applied", C.c_int64),
                ("n_feasible", C.c_int32), ("n_improving", C.c_int32), ("best_feasible_D", C.c_double),
                ("need_followers", C.c_int32), ("need_queue", C.c_int32), ("need_routes", C.c_int32),
                ("need_positions", C.c_int32)]


class RepairStats(C.Structure):
    _fields_ = [("status", C.c_int32), ("inserted", C.c_int32), ("need_j", C.c_int32), ("need_k", C.c_int32),
                ("slot_evals", C.c_int64), ("ref_slot_evals", C.c_int64)]


class Timing(C.Structure):
    _fields_ = [("eval_ms", C.c_double), ("select_ms", C.c_double), ("plan_ms", C.c_double),
                ("total_ms", C.c_double), ("eval_launches", C.c_int64), ("rounds", C.c_int64),
                ("cands_total", C.c_int64), ("geval_ms", C.c_double), ("kern_ms", C.c_double * 6),
                ("kern_rounds", C.c_int64)]


_L = None


def lib():
    """Load the sm_100a library; raises if it was not built."""
    global _L
    if _L is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(the CUDA library has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.mdr_last_error.restype = C.c_char_p
        L.mdr_build_info.restype = C.c_char_p
        L.mdr_device_count.restype = C.c_int
        L.mdr_instance_create.argtypes = [C.POINTER(InstanceDesc), C.c_int32, C.POINTER(vp)]
        L.mdr_instance_destroy.argtypes = [vp]
        L.mdr_instance_destroy.restype = None
        L.mdr_pop_create.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp)]
        L.mdr_pop_destroy.argtypes = [vp]
        L.mdr_pop_destroy.restype = None
        L.mdr_pop_upload.argtypes = [vp, C.c_int32, i32p, i32p, i32p, i32p, i32p, f64p, vp]
        L.mdr_pop_download.argtypes = [vp, i32p, i32p, i32p, i32p, i32p, f64p, i32p, i32p, vp]
        L.mdr_pop_download_best.argtypes = [vp, i32p, i32p, i32p, i32p, i32p, f64p, i32p, i32p, vp]
        L.mdr_count.argtypes = [vp, C.c_int32, C.c_int32]
        L.mdr_count.restype = C.c_int64
        L.mdr_enumerate.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(Cands)]
        L.mdr_evaluate.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(Cands), f64p, C.POINTER(Deltas)]
        L.mdr_leader_followers.argtypes = [vp, C.POINTER(Cands), C.POINTER(Deltas), C.c_int32, i64p, i64p, i64p]
        L.mdr_totals.argtypes = [vp, C.c_int32, f64p]
        L.mdr_local_search.argtypes = [vp, C.POINTER(LsCfg), C.POINTER(LsStats), vp]
        L.mdr_get_timing.argtypes = [vp, C.POINTER(Timing)]
        L.mdr_set_profiling.argtypes = [vp, C.c_int32]
        L.mdr_pop_info.argtypes = [vp, i32p]
        L.mdr_shuffle_stream.argtypes = [C.POINTER(C.c_uint32), C.c_int32, u8p, C.c_int32, u8p]
        L.mdr_probe_l2_gbs.argtypes = [C.c_int32, C.c_int64, C.c_int32, f64p]
        L.mdr_probe_fp64_gops.argtypes = [C.c_int32, C.c_int32, f64p]
        L.mdr_pop_download_range.argtypes = [vp, C.c_int32, C.c_int32, i32p, i32p, i32p, i32p, i32p,
                                             C.POINTER(C.c_int32), C.POINTER(C.c_int32), vp]
        L.mdr_pop_breakdown.argtypes = [vp, f64p, f64p, vp]
        L.mdr_repair.argtypes = [vp, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(RepairStats),
                                 vp]
        L.mdr_neighbor_build.argtypes = [C.c_int32, C.c_int32, C.c_int32, f64p, f64p, f64p, f64p, f64p, C.c_double,
                                         C.c_double, C.c_double, C.c_int32, C.POINTER(C.c_int32), u8p,
                                         C.POINTER(C.c_float)]
        L.mdr_population_select.argtypes = [C.c_int32, C.c_int32, C.c_int32, i64p, i64p, f64p, C.c_int32,
                                            C.c_double, f64p, i64p, i32p]
        L.mdr_pop_trace.argtypes = [vp, C.c_int32, C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_int64)]
        L.mdr_pop_route_attrs.argtypes = [vp, C.c_int32, C.c_int32, f64p, vp]
        L.mdr_route_exchange.argtypes = [vp, C.c_int32, i32p, i32p, i32p, i32p, i32p, C.c_int32, i32p, i32p,
                                         C.POINTER(C.c_uint32), f64p, C.c_int32, C.c_int32, i32p, i32p, i32p, i32p,
                                         i32p, f64p]
        L.mdr_construct.argtypes = [vp, C.c_int32, i32p, i32p, i32p, i32p, vp]
        L.mdr_route_sim.argtypes = [vp, C.c_int32, i32p, i32p, C.c_int32, f64p]
        _L = L
    return _L


def check(rc: int, what: str = "") -> None:
    if rc == MDR_OK:
        return
    msg = lib().mdr_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == MDR_ERR_ARG:
        raise ValueError(text)
    if rc == MDR_ERR_CONFLICT:
        raise ValueError(text)
    if rc == MDR_ERR_CAPACITY:
        raise CapacityError(text)
    raise RuntimeError(f"libmdr_sm100 status {rc}: {text}")


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def device_count() -> int:
    return int(lib().mdr_device_count())


EXPORTED = ("mdr_last_error", "mdr_device_count", "mdr_build_info", "mdr_instance_create",
            "mdr_instance_destroy", "mdr_pop_create", "mdr_pop_destroy", "mdr_pop_upload",
            "mdr_pop_download", "mdr_pop_download_best", "mdr_count", "mdr_enumerate", "mdr_evaluate",
            "mdr_leader_followers", "mdr_totals", "mdr_local_search", "mdr_get_timing",
            "mdr_set_profiling", "mdr_shuffle_stream", "mdr_probe_l2_gbs",
            "mdr_probe_fp64_gops", "mdr_neighbor_build", "mdr_repair", "mdr_pop_download_range",
            "mdr_population_select", "mdr_route_sim", "mdr_construct", "mdr_pop_trace", "mdr_pop_route_attrs", "mdr_route_exchange",
            "mdr_pop_breakdown", "mdr_pop_info")
