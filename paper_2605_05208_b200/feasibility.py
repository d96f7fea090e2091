"""Feasibility check by forward simulation, on the device (SURVEY.md 8(a) row
a48; drop-in for model.simulate_route / minimal_duration / check_feasible,
model.py:242-392).

The structural and coverage checks are set bookkeeping over the host route
lists; every route's simulation -- distance, load, time warp, late arrivals,
duration and the minimal duration over warp-minimal departure times -- runs in
one batched launch (mdr_route_sim, csrc/mdr_feasibility.cu).  The report's
sums accumulate the per-route values in route order, as the reference's loop
does, so the report is bit-identical (tests/test_scalar_oracles.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .model import INF


@dataclass
class RouteSim:
    distance: float = 0.0
    load: float = 0.0
    duration: float = 0.0
    time_warp: float = 0.0
    late_count: int = 0


@dataclass
class FeasibilityReport:
    structural_error: Optional[str] = None
    missing: list = field(default_factory=list)
    duplicated: list = field(default_factory=list)
    capacity_excess: float = 0.0
    duration_excess: float = 0.0
    time_warp: float = 0.0
    late_count: int = 0
    closure_violations: int = 0
    fleet_excess: int = 0

    @property
    def coverage_ok(self) -> bool:
        return not (self.missing or self.duplicated)

    @property
    def all_ok(self) -> bool:
        tol = 1e-9
        return (self.structural_error is None and self.coverage_ok and self.capacity_excess <= tol
                and self.duration_excess <= tol and self.time_warp <= tol and self.closure_violations == 0
                and self.fleet_excess == 0)


def _simulate(routes, inst, want_min: bool, device: int = 0) -> np.ndarray:
    """[len(routes), 6] {distance, load, duration, time_warp, late, min duration} from the device."""
    from .session import session_for
    seqs = [r.sequence(inst.open_routes) for r in routes]
    off = np.zeros(len(seqs) + 1, np.int32)
    off[1:] = np.cumsum([len(s) for s in seqs])
    flat = np.ascontiguousarray(np.concatenate(seqs) if seqs else np.zeros(0), np.int32)
    out = np.zeros((max(len(seqs), 1), 6), np.float64)
    if seqs:
        sess = session_for(inst, None, None, device)
        _lib.check(_lib.lib().mdr_route_sim(sess.dinst.handle, len(seqs), _lib.ptr(off, _lib.i32p),
                                            _lib.ptr(flat, _lib.i32p), int(want_min), _lib.ptr(out, _lib.f64p)),
                   "mdr_route_sim")
    return out[:len(seqs)]


def _sim(row) -> RouteSim:
    return RouteSim(float(row[0]), float(row[1]), float(row[2]), float(row[3]), int(row[4]))


def simulate_route(route, inst, device: int = 0) -> RouteSim:
    """Earliest-departure forward simulation of one route (model.py:285-288)."""
    return _sim(_simulate([route], inst, False, device)[0])


def minimal_duration(route, inst, device: int = 0) -> float:
    """Minimal duration over warp-minimal departure times (model.py:291-314)."""
    return float(_simulate([route], inst, True, device)[0, 5])


def _structure_error(sol, inst) -> Optional[str]:
    n = inst.n_nodes
    for r in sol.routes:
        for x in (r.depart, r.arrive):
            if not 0 <= x < n:
                return f"unknown depot id on route {r!r}"
        if not (inst.is_depot(r.depart) and inst.is_depot(r.arrive)):
            return f"route endpoint is not a depot: {r!r}"
        for c in r.customers:
            if not 0 <= c < n:
                return f"unknown node id {c}"
            if inst.is_depot(c):
                return f"depot {c} appears as a customer"
        if len(r.customers) != len(set(r.customers)):
            return f"repeated customer within route {r!r}"
    return None


def check_feasible(sol, inst, device: int = 0) -> FeasibilityReport:
    """Coverage, structure and every violation magnitude (model.py:349-392)."""
    rep = FeasibilityReport(structural_error=_structure_error(sol, inst))
    if rep.structural_error is not None:
        return rep
    count = np.bincount(np.asarray(sol.customer_list(), np.int64), minlength=inst.n_nodes)
    cust = np.arange(inst.n_depots, inst.n_nodes)
    rep.missing = [int(c) for c in cust[count[inst.n_depots:] == 0]]
    rep.duplicated = [int(c) for c in np.nonzero(count > 1)[0]]
    live = [r for r in sol.routes if r.customers]
    sims = _simulate(live, inst, inst.max_duration != INF, device)
    per_depot = np.zeros(inst.n_depots, np.int64)
    for r, row in zip(live, sims):
        rep.capacity_excess += max(float(row[1]) - inst.capacity, 0.0)
        if inst.max_duration != INF:
            rep.duration_excess += max(float(row[5]) - inst.max_duration, 0.0)
        rep.time_warp += float(row[3])
        rep.late_count += int(row[4])
        rep.closure_violations += int(not inst.open_routes and r.depart != r.arrive)
        per_depot[r.depart] += 1
    if inst.fleet_per_depot != INF:
        rep.fleet_excess = int(np.maximum(per_depot - inst.fleet_per_depot, 0).sum())
    return rep
