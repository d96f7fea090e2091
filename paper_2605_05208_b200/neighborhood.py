"""Granular neighbour lists (input of the hot path; mirrors `mdroute.neighborhood`).

The lists are built once per instance on the host and uploaded with the
instance (`mdr_instance_create`).  Semantics follow neighborhood.py:60-101:
correlation eta_ij = c_ij + Gamma*(alpha*early + beta*late), arcs with
e_i + s_i + t_ij > l_j pruned, customer targets only, no self arcs, rows sorted
ascending by eta with ties broken by smaller node id, first theta kept.
`build` is the host restatement used to prepare inputs; `build_device` is the
B200 build: one CTA per source node computes the
correlation row, prunes it and selects the first theta by (eta, id) with a
shared-memory bitonic sorter (csrc/mdr_neighbors.cu, C-ABI mdr_neighbor_build).
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


def build_device(inst, cfg: NeighborConfig, consts, device: int = 0, with_mask: bool = True) -> NeighborLists:
    """`build` on the GPU (bit-identical lists and mask).  The kernel's device
    time is left in `NeighborLists.kernel_ms`."""
    import ctypes as C

    from . import _lib
    n = inst.n_nodes
    dist = np.ascontiguousarray(inst.dist, dtype=np.float64)
    tm = None if inst.time is inst.dist else np.ascontiguousarray(inst.time, dtype=np.float64)
    e = np.ascontiguousarray(inst.tw_early, dtype=np.float64)
    l = np.ascontiguousarray(inst.tw_late, dtype=np.float64)
    s = np.ascontiguousarray(inst.service, dtype=np.float64)
    theta = int(cfg.theta)
    lists = np.empty((n, theta), np.int32)
    mask = np.empty((n, n), np.uint8) if with_mask else None
    ms = C.c_float(0.0)
    f64 = lambda a: _lib.ptr(a, _lib.f64p)  # noqa: E731
    _lib.check(_lib.lib().mdr_neighbor_build(
        device, n, inst.n_depots, f64(dist), None if tm is None else f64(tm), f64(e), f64(l), f64(s),
        float(consts.gamma), float(cfg.alpha), float(cfg.beta), theta, _lib.ptr(lists, C.POINTER(C.c_int32)),
        None if mask is None else _lib.ptr(mask, _lib.u8p), C.byref(ms)), "mdr_neighbor_build")
    out = NeighborLists(lists, mask.view(bool) if mask is not None else None, theta)
    out.kernel_ms = float(ms.value)
    return out
