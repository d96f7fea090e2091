"""Loader for the committed golden fixtures (tests/golden/, made by make_golden.py)."""
from __future__ import annotations

import hashlib
import json
import os
from functools import lru_cache

import numpy as np

from paper_2605_05208_b200.evaluation import PenaltyState, ScalingConstants
from paper_2605_05208_b200.model import Instance, Route, Solution
from paper_2605_05208_b200.neighborhood import NeighborLists

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIELDS = ("r1", "p1", "r2", "p2", "len1", "len2", "rev1", "rev2", "depot", "mode")
DFIELDS = ("dD", "dV1", "dV2", "dV3", "dV4", "dF")


@lru_cache(None)
def manifest():
    with open(os.path.join(GOLD, "manifest.json")) as f:
        return json.load(f)


@lru_cache(None)
def store(name):
    return dict(np.load(os.path.join(GOLD, f"{name}.npz")))


class Case:
    def __init__(self, group, npz, tag):
        self.tag = tag
        self.meta = manifest()[group][tag]
        S = store(npz)
        self.S = S
        m = self.meta
        nodes = S[f"{tag}_nodes"]
        nd = m["n_depots"]
        depots = [tuple(nodes[d, :2]) for d in range(nd)]
        windows = m["variant"] == "mdvrptw"
        cust = []
        for row in nodes[nd:]:
            x, y, q, s, e, l = (float(v) for v in row)
            cust.append((x, y, q, s, e, l) if windows else (x, y, q, s))
        dw = [(float(nodes[d, 4]), float(nodes[d, 5])) for d in range(nd)] if windows else None
        self.inst = Instance.from_coords(m["variant"], depots, cust, fleet_per_depot=m["fleet"],
                                         capacity=m["capacity"], max_duration=m["max_duration"],
                                         depot_windows=dw)
        sha = hashlib.sha256(np.ascontiguousarray(self.inst.dist).tobytes()).hexdigest()
        assert sha == m["dist_sha"], f"{tag}: rebuilt distance matrix differs from the reference"
        self.consts = ScalingConstants(float.fromhex(m["gamma"]), float.fromhex(m["theta"]))
        lists = S[f"{tag}_lists"]
        mask = np.zeros((self.inst.n_nodes, self.inst.n_nodes), bool)
        for i in range(lists.shape[0]):
            row = lists[i][lists[i] >= 0]
            mask[i, row] = True
        self.nbr = NeighborLists(lists, mask, lists.shape[1])
        self.sol = self._sol("")
        self.lam = [float(x) for x in S[f"{tag}_lam"]]

    def _sol(self, pfx):
        S, t = self.S, self.tag
        off, cust = S[f"{t}_{pfx}off"], S[f"{t}_{pfx}cust"]
        dep, arr = S[f"{t}_{pfx}dep"], S[f"{t}_{pfx}arr"]
        return Solution([Route(int(dep[r]), int(arr[r]), [int(c) for c in cust[off[r]:off[r + 1]]])
                         for r in range(len(dep))])

    def penalties(self):
        return PenaltyState(lam=self.lam)

    def op_full(self, op):
        S, t = self.S, self.tag
        if f"{t}_op{op}_c" not in S:
            return None
        cm, dm, fn = S[f"{t}_op{op}_c"], S[f"{t}_op{op}_d"], S[f"{t}_op{op}_fn"]
        cands = {f: cm[i] for i, f in enumerate(FIELDS)}
        cands["rev1"] = cands["rev1"].astype(bool)
        cands["rev2"] = cands["rev2"].astype(bool)
        deltas = {f: dm[i] for i, f in enumerate(DFIELDS)}
        deltas["fleet_neutral"] = fn.astype(bool)
        return cands, deltas

    def op_sample(self, op):
        S, t = self.S, self.tag
        if f"{t}_op{op}_si" not in S:
            return None
        return S[f"{t}_op{op}_si"], S[f"{t}_op{op}_sc"], S[f"{t}_op{op}_sd"], S[f"{t}_op{op}_sfn"]

    def final_routes(self):
        s = self._sol("fin_")
        return [(r.depart, r.arrive, list(r.customers)) for r in s.routes]


def canon_sha(cm, dm, fn):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(cm, np.int64).tobytes())
    h.update((np.ascontiguousarray(dm, np.float64) + 0.0).tobytes())
    h.update(np.ascontiguousarray(fn, np.uint8).tobytes())
    return h.hexdigest()


def cases(group):
    npz = {"small": "ops_small", "medium": "ops_medium", "traj": "ls_traj"}[group]
    return [Case(group, npz, t) for t in sorted(manifest()[group])]


def routes_of(sol):
    return [(r.depart, r.arrive, list(r.customers)) for r in sol.routes]
