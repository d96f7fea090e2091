"""Loader for tests/golden/repair.{npz,json} (made by make_repair_golden.py)."""
from __future__ import annotations

import hashlib
import json
import os
from functools import lru_cache

import numpy as np

from paper_2605_05208_b200.evaluation import PenaltyState, ScalingConstants
from paper_2605_05208_b200.model import Instance, Route, Solution

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(None)
def _load():
    S = dict(np.load(os.path.join(GOLD, "repair.npz")))
    with open(os.path.join(GOLD, "repair.json")) as f:
        return S, json.load(f)


def tags():
    return sorted(_load()[1])


def _sol(S, tag, pfx):
    off, cust, dep, arr = (S[f"{tag}_{pfx}_{k}"] for k in ("off", "cust", "dep", "arr"))
    return Solution([Route(int(dep[r]), int(arr[r]), [int(c) for c in cust[off[r]:off[r + 1]]])
                     for r in range(len(dep))])


class RepairCase:
    def __init__(self, tag):
        S, man = _load()
        m = man[tag]
        self.tag, self.meta = tag, m
        nodes, nd = S[f"{tag}_nodes"], m["n_depots"]
        windows = m["variant"] == "mdvrptw"
        depots = [tuple(nodes[d, :2]) for d in range(nd)]
        cust = [(x, y, q, s, e, l) if windows else (x, y, q, s) for x, y, q, s, e, l in nodes[nd:]]
        dw = [(float(nodes[d, 4]), float(nodes[d, 5])) for d in range(nd)] if windows else None
        self.inst = Instance.from_coords(m["variant"], depots, cust, fleet_per_depot=m["fleet"],
                                         capacity=m["capacity"], max_duration=m["max_duration"],
                                         depot_windows=dw)
        sha = hashlib.sha256(np.ascontiguousarray(self.inst.dist).tobytes()).hexdigest()
        assert sha == m["dist_sha"], tag
        self.consts = ScalingConstants(float.fromhex(m["gamma"]), float.fromhex(m["theta"]))
        self.sol = _sol(S, tag, "in")
        self.want = _sol(S, tag, "out")
        self.unrouted = [int(c) for c in S[f"{tag}_unrouted"]]
        self.op = m["op"]
        self.lam = list(m["lam"])
        self.seed = m["seed"]

    def penalties(self):
        return PenaltyState(lam=list(self.lam))


def routes_of(sol):
    return [(r.depart, r.arrive, list(r.customers)) for r in sol.routes]
