"""Penalty scaling constants and adaptive penalty state (mirrors `mdroute.evaluation`).

`ScalingConstants.from_instance` restates evaluation.py:117-132, `PenaltyState`
evaluation.py:135-150 and `adapt_penalties` evaluation.py:153-161.  The device
local search applies the same update on the GPU (csrc/mdr_ls.cu); this host
copy is used by the operator-level API and for argument checking.
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
