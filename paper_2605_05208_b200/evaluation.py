"""Penalty scaling constants, adaptive penalty state and the scalar evaluation
(mirrors `mdroute.evaluation`).

`ScalingConstants.from_instance` restates evaluation.py:117-132, `PenaltyState`
evaluation.py:135-150 and `adapt_penalties` evaluation.py:153-161.  The device
local search applies the same update on the GPU (csrc/mdr_kernels.cu); this
host copy is used by the operator-level API and for argument checking.

The scalar sequence algebra (`single_attr`, `concat`, `fold_attrs`,
`route_attr`, evaluation.py:22-106) and the from-scratch `evaluate`
(evaluation.py:164-224) are what the generation loop (engine.py) scores each
offspring with; they keep Python's `max`/`min` semantics (first argument unless
the second compares strictly larger / smaller).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

LAMBDA_MIN = 0.01
LAMBDA_MAX = 10000.0


@dataclass(frozen=True)
class ScalingConstants:
    gamma: float
    theta: float

    @staticmethod
    def from_instance(inst) -> "ScalingConstants":
        n = inst.n_nodes
        iu, ju = np.triu_indices(n, 1)  # row-major i<j, the order of evaluation.py:121-124
        c = np.asarray(inst.dist)[iu, ju]
        t = np.asarray(inst.time)[iu, ju]
        if float(c.max(initial=0.0)) <= 0.0:
            raise ValueError("degenerate instance: all arc distances are zero")
        t_sum = float(t.sum())
        gamma = float(c.sum()) / t_sum if t_sum > 0 else 1.0
        theta = 2.0 * float(c.max()) - float(c.min())
        return ScalingConstants(gamma, theta)


class PenaltyState:
    __slots__ = ("lam", "kappa", "lam_min", "lam_max")

    def __init__(self, kappa: float = 0.5, lam: Optional[Sequence[float]] = None,
                 lam_min: float = LAMBDA_MIN, lam_max: float = LAMBDA_MAX):
        if not (0.0 < kappa < 1.0):
            raise ValueError("kappa must lie in (0, 1)")
        self.kappa = kappa
        self.lam = list(lam) if lam is not None else [1.0, 1.0, 1.0, 1.0]
        self.lam_min = lam_min
        self.lam_max = lam_max

    def clone(self) -> "PenaltyState":
        return PenaltyState(self.kappa, self.lam, self.lam_min, self.lam_max)


def adapt_penalties(penalties, violated):
    for i in range(4):
        if violated[i]:
            penalties.lam[i] /= penalties.kappa
        else:
            penalties.lam[i] *= penalties.kappa
        penalties.lam[i] = min(max(penalties.lam[i], penalties.lam_min), penalties.lam_max)
    return penalties


INF = float("inf")


class SeqAttr:
    """dist, load, T, E, L, TW of a node sequence plus its end nodes (evaluation.py:22-57)."""

    __slots__ = ("dist", "load", "T", "E", "L", "TW", "first", "last")

    def __init__(self, dist=0.0, load=0.0, T=0.0, E=0.0, L=INF, TW=0.0, first=-1, last=-1):
        self.dist, self.load, self.T, self.E, self.L, self.TW = dist, load, T, E, L, TW
        self.first, self.last = first, last

    def is_empty(self) -> bool:
        return self.first < 0


def single_attr(node: int, inst) -> SeqAttr:
    return SeqAttr(0.0, float(inst.demand[node]), float(inst.service[node]), float(inst.tw_early[node]),
                   float(inst.tw_late[node]), 0.0, node, node)


def concat(a: SeqAttr, b: SeqAttr, inst) -> SeqAttr:
    if b.first < 0:
        return a
    if a.first < 0:
        return b
    t = float(inst.time[a.last, b.first])
    c = float(inst.dist[a.last, b.first])
    delta = a.T - a.TW + t
    wait = max(b.E - delta - a.L, 0.0)
    warp = max(a.E + delta - b.L, 0.0)
    return SeqAttr(a.dist + c + b.dist, a.load + b.load, a.T + b.T + t + wait,
                   max(b.E - delta, a.E) - wait, min(b.L - delta, a.L) + warp,
                   a.TW + b.TW + warp, a.first, b.last)


def fold_attrs(seq, inst) -> SeqAttr:
    acc = single_attr(seq[0], inst)
    for node in seq[1:]:
        acc = concat(acc, single_attr(node, inst), inst)
    return acc


def route_attr(route, inst) -> SeqAttr:
    return fold_attrs(route.sequence(inst.open_routes), inst)


class EvalBreakdown:
    """D, the four unweighted violation terms and the penalised total (evaluation.py:164-176)."""

    __slots__ = ("D", "V1", "V2", "V3", "V4", "F")

    def __init__(self, D=0.0, V1=0.0, V2=0.0, V3=0.0, V4=0.0, F=0.0):
        self.D, self.V1, self.V2, self.V3, self.V4, self.F = D, V1, V2, V3, V4, F

    def violations(self):
        return [self.V1, self.V2, self.V3, self.V4]


def route_contributions(attr: SeqAttr, depart: int, arrive: int, consts, inst):
    v1 = consts.gamma * attr.TW if inst.has_windows else 0.0
    v2 = consts.theta * max(attr.load - inst.capacity, 0.0) / inst.capacity
    v3 = 0.0
    if inst.max_duration != INF:
        v3 = consts.theta * max(attr.T - inst.max_duration, 0.0) / inst.max_duration
    closure = 0 if inst.open_routes else int(depart != arrive)
    return attr.dist, v1, v2, v3, closure


def depot_counts(sol, inst) -> list:
    counts = [0] * inst.n_depots
    for r in sol.routes:
        if r.customers:
            counts[r.depart] += 1
    return counts


def fleet_excess(counts, inst) -> int:
    if inst.fleet_per_depot == INF:
        return 0
    return int(sum(max(k - inst.fleet_per_depot, 0) for k in counts))


def evaluate(sol, penalties, consts, inst) -> EvalBreakdown:
    """Full penalised evaluation of a solution from scratch (evaluation.py:206-224)."""
    out = EvalBreakdown()
    closures = 0
    for r in sol.routes:
        if not r.customers:
            continue
        d, v1, v2, v3, clo = route_contributions(route_attr(r, inst), r.depart, r.arrive, consts, inst)
        out.D += d
        out.V1 += v1
        out.V2 += v2
        out.V3 += v3
        closures += clo
    out.V4 = consts.theta * (closures + fleet_excess(depot_counts(sol, inst), inst))
    lam = penalties.lam
    out.F = out.D + lam[0] * out.V1 + lam[1] * out.V2 + lam[2] * out.V3 + lam[3] * out.V4
    return out


def move_delta(sol, move, penalties, consts, inst) -> EvalBreakdown:
    """Recompute-from-scratch delta of one move over the affected routes only
    (evaluation.py:227-275): the scalar cross-check of the batched evaluator
    (agrees with it to ~1e-6, not bit for bit -- SURVEY.md 8(c))."""
    from .moves import move_plan
    from .model import Route
    delta = EvalBreakdown()
    closure_delta = 0
    changes: dict = {}
    for plan in move_plan(sol, move, inst):
        if plan.route_index is not None:
            old = sol.routes[plan.route_index]
            attr = old.attr if getattr(old, "attr", None) is not None else route_attr(old, inst)
            d, v1, v2, v3, clo = route_contributions(attr, old.depart, old.arrive, consts, inst)
            delta.D -= d
            delta.V1 -= v1
            delta.V2 -= v2
            delta.V3 -= v3
            closure_delta -= clo
            changes[old.depart] = changes.get(old.depart, 0) - 1
        if plan.customers:
            d, v1, v2, v3, clo = route_contributions(route_attr(Route(plan.depart, plan.arrive, plan.customers), inst),
                                                     plan.depart, plan.arrive, consts, inst)
            delta.D += d
            delta.V1 += v1
            delta.V2 += v2
            delta.V3 += v3
            closure_delta += clo
            changes[plan.depart] = changes.get(plan.depart, 0) + 1
    fleet_delta = 0
    if inst.fleet_per_depot != INF and changes:
        counts = depot_counts(sol, inst)
        nv = inst.fleet_per_depot
        for dep, chg in changes.items():
            fleet_delta += max(counts[dep] + chg - nv, 0) - max(counts[dep] - nv, 0)
    delta.V4 = consts.theta * (closure_delta + fleet_delta)
    lam = penalties.lam
    delta.F = delta.D + lam[0] * delta.V1 + lam[1] * delta.V2 + lam[2] * delta.V3 + lam[3] * delta.V4
    return delta
