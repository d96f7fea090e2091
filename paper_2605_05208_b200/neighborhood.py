"""Granular neighbour lists (input of the hot path; mirrors `mdroute.neighborhood`).

The lists are built once per instance on the host and uploaded with the
instance (`mdr_instance_create`).  Semantics follow neighborhood.py:60-101:
correlation eta_ij = c_ij + Gamma*(alpha*early + beta*late), arcs with
e_i + s_i + t_ij > l_j pruned, customer targets only, no self arcs, rows sorted
ascending by eta with ties broken by smaller node id, first theta kept.
Moving this build to the GPU is a SURVEY.md sec. 8(f) "next" row.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class NeighborConfig:
    theta: int = 50
    alpha: float = 1.0
    beta: float = 10.0

    def __post_init__(self):
        if self.theta < 1:
            raise ValueError("theta must be >= 1")


class NeighborLists:
    def __init__(self, lists: np.ndarray, mask: np.ndarray, theta: int):
        self.lists = lists  # (n_nodes, theta) int32, -1 padded
        self.mask = mask    # (n_nodes, n_nodes) bool
        self.theta = theta

    def neighbors(self, i: int) -> np.ndarray:
        row = self.lists[i]
        return row[row >= 0]


def build(inst, cfg: NeighborConfig, consts) -> NeighborLists:
    n = inst.n_nodes
    c = np.asarray(inst.dist)
    t = np.asarray(inst.time)
    e = np.asarray(inst.tw_early)
    l = np.asarray(inst.tw_late)
    s = np.asarray(inst.service)
    finish = (l[:, None] + s[:, None]) + t          # latest finish of i plus travel
    early = np.maximum(e[None, :] - finish, 0.0)
    with np.errstate(invalid="ignore"):
        late = np.maximum(finish - l[None, :], 0.0)
    late[:, np.isinf(l)] = 0.0
    late = np.nan_to_num(late, nan=0.0)
    eta = c + consts.gamma * (cfg.alpha * early + cfg.beta * late)
    allowed = ((e[:, None] + s[:, None]) + t) <= l[None, :]
    allowed[:, :inst.n_depots] = False
    np.fill_diagonal(allowed, False)
    theta = int(cfg.theta)
    lists = np.full((n, theta), -1, dtype=np.int32)
    mask = np.zeros((n, n), dtype=bool)
    for i in range(n):
        cand = np.flatnonzero(allowed[i])          # ascending ids
        if cand.size == 0:
            continue
        keep = cand[np.argsort(eta[i, cand], kind="stable")[:theta]]
        lists[i, :keep.size] = keep
        mask[i, keep] = True
    return NeighborLists(lists, mask, theta)
