"""Forward-simulation feasibility oracle -- TEST INFRASTRUCTURE ONLY: a scalar
restatement of `mdroute.model`, model.py:232-392 (SURVEY.md sec. 8(a) row
a48), the checker of the device simulation (csrc/mdr_feasibility.cu) and
pinned to the reference by tests/golden/scalar.json.

Independent of the concat algebra: every route is simulated node by node
(wait for early windows, clamp late arrivals and accumulate the overshoot as
time warp), and `check_feasible` reports coverage, structure and every
violation magnitude.  `minimal_duration` scans the finitely many departure
times that align an arrival with a window bound.  Host-side test/validation
utility, used to cross-check the device results (F = D <=> feasible).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

INF = float("inf")


@dataclass
class RouteSim:
    distance: float = 0.0
    load: float = 0.0
    duration: float = 0.0   # travel + service + waiting, warps excluded by clamping
    time_warp: float = 0.0
    late_count: int = 0


def simulate_from(route, inst, t0: float) -> RouteSim:
    """Simulate a route whose first node is reached at time t0 (model.py:242-282)."""
    seq = route.sequence(inst.open_routes)
    c, t = inst.dist, inst.time
    e, l, s, q = inst.tw_early, inst.tw_late, inst.service, inst.demand
    sim = RouteSim()
    first = seq[0]
    start = max(t0, e[first])
    if start > l[first]:
        sim.time_warp += start - l[first]
        sim.late_count += 1
        start = l[first]
    now = start + s[first]
    for a, b in zip(seq, seq[1:]):
        sim.distance += c[a, b]
        arrive = now + t[a, b]
        if arrive < e[b]:
            arrive = e[b]
        elif arrive > l[b]:
            sim.time_warp += arrive - l[b]
            sim.late_count += 1
            arrive = l[b]
        now = arrive + s[b]
        sim.load += q[b]
    sim.duration = float(now - start + sim.time_warp)
    sim.distance, sim.load, sim.time_warp = float(sim.distance), float(sim.load), float(sim.time_warp)
    return sim


def simulate_route(route, inst) -> RouteSim:
    """Earliest-departure simulation."""
    return simulate_from(route, inst, float(inst.tw_early[route.sequence(inst.open_routes)[0]]))


def minimal_duration(route, inst) -> float:
    """Minimal duration over warp-minimal departure times (model.py:285-315)."""
    if not inst.has_windows:
        return simulate_route(route, inst).duration
    seq = route.sequence(inst.open_routes)
    e, l, s, t = inst.tw_early, inst.tw_late, inst.service, inst.time
    first = seq[0]
    starts = {float(e[first])}
    if math.isfinite(l[first]):
        starts.add(float(l[first]))
    raw = 0.0  # travel + service from the first service start, no waiting
    for a, b in zip(seq, seq[1:]):
        raw += s[a] + t[a, b]
        for bound in (e[b], l[b]):
            if math.isfinite(bound):
                starts.add(float(bound - raw))
    base = simulate_route(route, inst)
    best = base.duration
    for t0 in starts:
        if t0 < e[first]:
            continue
        sim = simulate_from(route, inst, t0)
        if sim.time_warp <= base.time_warp + 1e-9:
            best = min(best, sim.duration)
    return best


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
        return not self.missing and not self.duplicated

    @property
    def all_ok(self) -> bool:
        tol = 1e-9
        return (self.structural_error is None and self.coverage_ok and self.capacity_excess <= tol
                and self.duration_excess <= tol and self.time_warp <= tol and self.closure_violations == 0
                and self.fleet_excess == 0)


def _structure_error(sol, inst) -> Optional[str]:
    n = inst.n_nodes
    for r in sol.routes:
        if not (0 <= r.depart < n) or not (0 <= r.arrive < n):
            return f"unknown depot id on route {r!r}"
        if not inst.is_depot(r.depart) or not inst.is_depot(r.arrive):
            return f"route endpoint is not a depot: {r!r}"
        for c in r.customers:
            if not (0 <= c < n):
                return f"unknown node id {c}"
            if inst.is_depot(c):
                return f"depot {c} appears as a customer"
        if len(set(r.customers)) != len(r.customers):
            return f"repeated customer within route {r!r}"
    return None


def check_feasible(sol, inst) -> FeasibilityReport:
    """Oracle feasibility check by direct forward simulation (model.py:349-392)."""
    rep = FeasibilityReport()
    rep.structural_error = _structure_error(sol, inst)
    if rep.structural_error is not None:
        return rep
    seen: dict = {}
    for c in sol.customer_list():
        seen[c] = seen.get(c, 0) + 1
    rep.missing = sorted(c for c in inst.customers() if c not in seen)
    rep.duplicated = sorted(c for c, k in seen.items() if k > 1)
    per_depot = [0] * inst.n_depots
    for r in sol.routes:
        if not r.customers:
            continue
        sim = simulate_route(r, inst)
        rep.capacity_excess += max(sim.load - inst.capacity, 0.0)
        if inst.max_duration != INF:
            rep.duration_excess += max(minimal_duration(r, inst) - inst.max_duration, 0.0)
        rep.time_warp += sim.time_warp
        rep.late_count += sim.late_count
        if not inst.open_routes and r.depart != r.arrive:
            rep.closure_violations += 1
        per_depot[r.depart] += 1
    if inst.fleet_per_depot != INF:
        rep.fleet_excess = int(sum(max(k - inst.fleet_per_depot, 0) for k in per_depot))
    return rep
