"""Operator-level ETGA contract on the GPU (mirrors `mdroute.batch`).

    SolutionCache(sol, inst, consts)                      batch.py:48-170
    evaluate_candidates(cache, cs, penalties)             batch.py:365-553
    leader_and_followers(cache, cs, deltas, multi_move)   batch.py:578-614

The cache is the device-resident subsequence tables of one individual; the
deltas are computed by the sm_100a evaluator (csrc/mdr_device.cuh eval_cand)
bit-for-bit equal to the reference's numpy arithmetic; the leader/follower
extraction is a device reduction + stable radix sort on (dF, key, index).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .moves import CandidateSet, Move, Op
from .session import session_for

EPS = 1e-9


@dataclass
class DeltaArrays:
    dD: np.ndarray
    dV1: np.ndarray
    dV2: np.ndarray
    dV3: np.ndarray
    dV4: np.ndarray
    dF: np.ndarray
    fleet_neutral: np.ndarray


class _Snap:
    __slots__ = ("depart", "arrive", "customers")

    def __init__(self, r):
        self.depart, self.arrive, self.customers = r.depart, r.arrive, list(r.customers)


class _SnapSol:
    __slots__ = ("routes",)

    def __init__(self, sol):
        self.routes = [_Snap(r) for r in sol.routes]


class SolutionCache:
    """Device-resident subsequence tables of one solution (a snapshot, like
    the reference cache)."""

    def __init__(self, sol, inst, consts):
        self.inst = inst
        self.consts = consts
        self.windows = inst.has_windows
        self._sol = _SnapSol(sol)
        self.m = len(sol.routes)
        self.k = np.array([len(r.customers) for r in sol.routes], dtype=np.int64)
        self.depart = np.array([r.depart for r in sol.routes], dtype=np.int64)
        self.arrive = np.array([r.arrive for r in sol.routes], dtype=np.int64)
        self._session = session_for(inst, consts, None)
        self.pop()

    def pop(self):
        return self._session.single(self._sol, [1.0, 1.0, 1.0, 1.0])

    def totals(self):
        """Solution-level (D, V1, V2, V3, V4) with numpy's pairwise summation."""
        return self.pop().totals(0)

    def penalized(self, penalties) -> float:
        d, v1, v2, v3, v4 = self.totals()
        lam = penalties.lam
        return d + lam[0] * v1 + lam[1] * v2 + lam[2] * v3 + lam[3] * v4


def evaluate_candidates(cache: SolutionCache, cs, penalties) -> DeltaArrays:
    op = Op(int(cs.op))
    n = len(cs)
    if n == 0:
        z = np.zeros(0)
        return DeltaArrays(z, z, z, z, z, z, np.zeros(0, bool))
    d = cache.pop().evaluate(0, int(op), cs, penalties.lam)
    return DeltaArrays(d["dD"], d["dV1"], d["dV2"], d["dV3"], d["dV4"], d["dF"], d["fleet_neutral"])


def _materialize(cs, deltas, i: int) -> Move:
    mv = CandidateSet.move(cs, i) if not hasattr(cs, "move") else cs.move(i)
    if not isinstance(mv, Move):
        mv = Move(Op(int(mv.op)), mv.r1, mv.p1, mv.r2, mv.p2, mv.len1, mv.len2, mv.rev1, mv.rev2, mv.depot, mv.mode)
    mv.dD = float(deltas.dD[i])
    mv.dV = (float(deltas.dV1[i]), float(deltas.dV2[i]), float(deltas.dV3[i]), float(deltas.dV4[i]))
    mv.dF = float(deltas.dF[i])
    return mv


def leader_and_followers(cache: SolutionCache, cs, deltas, multi_move: bool):
    if len(cs) == 0:
        return None, []
    d = {f: getattr(deltas, f) for f in ("dD", "dV1", "dV2", "dV3", "dV4", "dF", "fleet_neutral")}
    best, fol = cache.pop().leader_followers(cs, d, multi_move)
    if best < 0:
        return None, []
    leader = _materialize(cs, deltas, best)
    followers = [_materialize(cs, deltas, int(i)) for i in fol] if multi_move else []
    return leader, followers
