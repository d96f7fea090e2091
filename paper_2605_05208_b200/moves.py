"""Move types and candidate enumeration (mirrors `mdroute.moves`, moves.py:24-464).

`enumerate_candidates` runs on the GPU: the candidate index spaces of the six
operators are enumerated implicitly by the device (mdr_enumerate) in the
reference's emission order, so the returned `CandidateSet` equals the
reference's array for array.  `move_plan` / `SolutionIndex` are the host-side
bookkeeping twins used by the operator-level API and the tests.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional

import numpy as np


class Op(IntEnum):
    RELOCATE = 0
    SWAP = 1
    TWO_OPT_STAR = 2
    TWO_OPT = 3
    DEPOT_INSERT = 4
    DEPOT_REPLACE = 5


MODE_DEPART = 0
MODE_ARRIVE = 1
MODE_BOTH = 2
ALL_OPS = tuple(Op)


@dataclass
class Move:
    op: Op
    r1: int
    p1: int
    r2: int = -1
    p2: int = -1
    len1: int = 0
    len2: int = 0
    rev1: bool = False
    rev2: bool = False
    depot: int = -1
    mode: int = -1
    dD: float = 0.0
    dV: tuple = (0.0, 0.0, 0.0, 0.0)
    dF: float = 0.0

    def routes_touched(self) -> set:
        out = {self.r1}
        if self.r2 >= 0:
            out.add(self.r2)
        return out

    def key(self) -> tuple:
        return (int(self.op), self.r1, self.r2, self.p1, self.p2, self.len1, self.len2,
                int(self.rev1), int(self.rev2), self.depot, self.mode)


@dataclass
class RoutePlan:
    route_index: Optional[int]
    depart: int
    arrive: int
    customers: list


_FIELDS = ("r1", "p1", "r2", "p2", "len1", "len2", "rev1", "rev2", "depot", "mode")


@dataclass
class CandidateSet:
    op: Op
    r1: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    p1: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    r2: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    p2: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    len1: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    len2: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    rev1: np.ndarray = field(default_factory=lambda: np.zeros(0, bool))
    rev2: np.ndarray = field(default_factory=lambda: np.zeros(0, bool))
    depot: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    mode: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))

    def __len__(self) -> int:
        return len(self.r1)

    def move(self, i: int) -> Move:
        return Move(Op(int(self.op)), int(self.r1[i]), int(self.p1[i]), int(self.r2[i]), int(self.p2[i]),
                    int(self.len1[i]), int(self.len2[i]), bool(self.rev1[i]), bool(self.rev2[i]),
                    int(self.depot[i]), int(self.mode[i]))

    def moves(self) -> list:
        return [self.move(i) for i in range(len(self))]

    def key_arrays(self) -> tuple:
        return (self.mode, self.depot, self.rev2, self.rev1, self.len2, self.len1,
                self.p2, self.p1, self.r2, self.r1)


class SolutionIndex:
    """Array views of a solution (moves.py:151-171)."""

    def __init__(self, sol, inst):
        n = inst.n_nodes
        self.route_of = np.full(n, -1, dtype=np.int64)
        self.idx_of = np.full(n, -1, dtype=np.int64)
        self.n_routes = len(sol.routes)
        self.k = np.array([len(r.customers) for r in sol.routes], dtype=np.int64)
        self.depart = np.array([r.depart for r in sol.routes], dtype=np.int64)
        self.arrive = np.array([r.arrive for r in sol.routes], dtype=np.int64)
        routed = []
        for ri, r in enumerate(sol.routes):
            routed.extend(r.customers)
            for pi, c in enumerate(r.customers):
                self.route_of[c] = ri
                self.idx_of[c] = pi
        self.routed = np.array(sorted(routed), dtype=np.int64)


def _seg(route, p, length, rev):
    seg = route.customers[p:p + length]
    return seg[::-1] if rev else seg


def move_plan(sol, move, inst) -> list:
    """New contents of every route a move touches (moves.py:88-148)."""
    op = Op(int(move.op))
    ra = sol.routes[move.r1]
    if op == Op.RELOCATE:
        seg = _seg(ra, move.p1, move.len1, move.rev1)
        rest = ra.customers[:move.p1] + ra.customers[move.p1 + move.len1:]
        if move.r1 == move.r2:
            at = move.p2 - move.len1 if move.p2 > move.p1 else move.p2
            return [RoutePlan(move.r1, ra.depart, ra.arrive, rest[:at] + seg + rest[at:])]
        rb = sol.routes[move.r2]
        return [RoutePlan(move.r1, ra.depart, ra.arrive, rest),
                RoutePlan(move.r2, rb.depart, rb.arrive, rb.customers[:move.p2] + seg + rb.customers[move.p2:])]
    if op == Op.SWAP:
        s1 = _seg(ra, move.p1, move.len1, move.rev1)
        if move.r1 == move.r2:
            s2 = _seg(ra, move.p2, move.len2, move.rev2)
            c = ra.customers
            return [RoutePlan(move.r1, ra.depart, ra.arrive,
                              c[:move.p1] + s2 + c[move.p1 + move.len1:move.p2] + s1 + c[move.p2 + move.len2:])]
        rb = sol.routes[move.r2]
        s2 = _seg(rb, move.p2, move.len2, move.rev2)
        return [RoutePlan(move.r1, ra.depart, ra.arrive,
                          ra.customers[:move.p1] + s2 + ra.customers[move.p1 + move.len1:]),
                RoutePlan(move.r2, rb.depart, rb.arrive,
                          rb.customers[:move.p2] + s1 + rb.customers[move.p2 + move.len2:])]
    if op == Op.TWO_OPT:
        c = ra.customers
        return [RoutePlan(move.r1, ra.depart, ra.arrive,
                          c[:move.p1] + c[move.p1:move.p2 + 1][::-1] + c[move.p2 + 1:])]
    if op == Op.TWO_OPT_STAR:
        rb = sol.routes[move.r2]
        return [RoutePlan(move.r1, ra.depart, rb.arrive, ra.customers[:move.p1] + rb.customers[move.p2:]),
                RoutePlan(move.r2, rb.depart, ra.arrive, rb.customers[:move.p2] + ra.customers[move.p1:])]
    if op == Op.DEPOT_INSERT:
        return [RoutePlan(move.r1, ra.depart, ra.arrive, ra.customers[:move.p1]),
                RoutePlan(None, move.depot, move.depot, ra.customers[move.p1:])]
    if op == Op.DEPOT_REPLACE:
        dep = move.depot if move.mode in (MODE_DEPART, MODE_BOTH) else ra.depart
        arr = move.depot if move.mode in (MODE_ARRIVE, MODE_BOTH) else ra.arrive
        return [RoutePlan(move.r1, dep, arr, list(ra.customers))]
    raise ValueError(f"unknown operator {op}")


def candidate_set_from_arrays(op, arrs: dict) -> CandidateSet:
    cs = CandidateSet(Op(int(op)))
    for f in _FIELDS:
        a = np.asarray(arrs[f])
        setattr(cs, f, a.astype(bool) if f.startswith("rev") else a.astype(np.int64))
    return cs


def enumerate_candidates(sol, op, nbr, inst, sidx=None) -> CandidateSet:
    """All structurally valid candidates of one operator, enumerated on the GPU."""
    from .session import session_for
    op = Op(int(op))  # ValueError for unknown operators, as moves.py:464
    if op == Op.TWO_OPT and inst.has_windows:
        return CandidateSet(op)
    sess = session_for(inst, None, nbr)
    pop = sess.single(sol, [1.0, 1.0, 1.0, 1.0])
    return candidate_set_from_arrays(op, pop.enumerate(0, int(op)))
