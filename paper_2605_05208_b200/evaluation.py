"""Penalty scaling constants, adaptive penalty state and the solution
evaluation (the API types of `mdroute.evaluation`).

`ScalingConstants.from_instance` restates evaluation.py:117-132 with numpy,
`PenaltyState` evaluation.py:135-150 and `adapt_penalties` evaluation.py:153-161
(the device local search applies the same update on the GPU, csrc/
mdr_kernels.cu).  `evaluate` (evaluation.py:206-224) runs on the device
(mdr_pop_breakdown: route folds, contributions and the ordered sums of the
reference, bit-identical); `RouteAttr` is the record of a route's cached
sequence attributes (`Route.attr`) the local search refreshes from the device
tables.  The scalar host algebra lives in oracle/scalar_ref.py as a test
checker only.
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


class EvalBreakdown:
    """D, the four unweighted violation terms and the penalised total (evaluation.py:164-176)."""

    __slots__ = ("D", "V1", "V2", "V3", "V4", "F")

    def __init__(self, D=0.0, V1=0.0, V2=0.0, V3=0.0, V4=0.0, F=0.0):
        self.D, self.V1, self.V2, self.V3, self.V4, self.F = D, V1, V2, V3, V4, F

    def violations(self):
        return [self.V1, self.V2, self.V3, self.V4]


class RouteAttr:
    """Sequence attributes of a whole route (the reference's SeqAttr of
    route_attr, evaluation.py:22-57, 97-106): the left fold the device keeps in
    its prefix table at the last sequence position."""

    __slots__ = ("dist", "load", "T", "E", "L", "TW", "first", "last")

    def __init__(self, dist=0.0, load=0.0, T=0.0, E=0.0, L=INF, TW=0.0, first=-1, last=-1):
        self.dist, self.load, self.T, self.E, self.L, self.TW = dist, load, T, E, L, TW
        self.first, self.last = first, last

    def is_empty(self) -> bool:
        return self.first < 0

    def __repr__(self):
        return (f"RouteAttr(dist={self.dist!r}, load={self.load!r}, T={self.T!r}, E={self.E!r}, L={self.L!r}, "
                f"TW={self.TW!r}, first={self.first}, last={self.last})")


def evaluate(sol, penalties, consts, inst, device: int = 0) -> EvalBreakdown:
    """Full penalised evaluation of one solution (evaluation.py:206-224), on the device."""
    from .session import session_for
    sess = session_for(inst, consts, None, device)
    row = sess.single(sol, penalties.lam).breakdowns([penalties.lam])[0]
    return EvalBreakdown(*(float(x) for x in row))
