"""Granular neighbour lists: the host restatement and the
device build (mdr_neighbor_build) against the reference's own lists
(tests/golden/nbr_edge.npz from make_nbr_golden.py, plus every golden case)."""
import hashlib
import json
import math
import os
from functools import lru_cache

import numpy as np
import pytest

import golden_io as G
from paper_2605_05208_b200.evaluation import ScalingConstants
from paper_2605_05208_b200.model import Instance
from paper_2605_05208_b200.neighborhood import NeighborConfig, build, build_device

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(None)
def _edge():
    S = dict(np.load(os.path.join(GOLD, "nbr_edge.npz")))
    with open(os.path.join(GOLD, "nbr_edge.json")) as f:
        return S, json.load(f)


def _edge_case(tag):
    S, man = _edge()
    m = man[tag]
    nodes, nd = S[f"{tag}_nodes"], m["n_depots"]
    depots = [tuple(nodes[d, :2]) for d in range(nd)]
    cust = []
    for x, y, q, s, e, l in nodes[nd:]:
        cust.append((x, y, q, s) if math.isinf(l) and e == 0.0 else (x, y, q, s, e, l))
    dw = [(float(nodes[d, 4]), float(nodes[d, 5])) for d in range(nd)] if m["variant"] == "mdvrptw" else None
    inst = Instance.from_coords(m["variant"], depots, cust, fleet_per_depot=4, capacity=200,
                                max_duration=float("inf"), depot_windows=dw)
    assert hashlib.sha256(np.ascontiguousarray(inst.dist).tobytes()).hexdigest() == m["dist_sha"]
    consts = ScalingConstants.from_instance(inst)
    assert consts.gamma.hex() == m["gamma"]
    return inst, consts, m["theta"], S[f"{tag}_lists"], S[f"{tag}_masksum"]


EDGE = ["ties", "ties_tw", "mixed_inf", "all_inf_tw", "tight", "theta_gt", "theta1", "open", "chunked",
        "chunked_tw"]
SMALL_EDGE = [t for t in EDGE if not t.startswith("chunked")]


def _mask_of(lists, n):
    mask = np.zeros((n, n), bool)
    for i in range(lists.shape[0]):
        mask[i, lists[i][lists[i] >= 0]] = True
    return mask


@pytest.mark.parametrize("tag", SMALL_EDGE)
def test_host_build_equals_reference_edge_cases(tag):
    inst, consts, theta, want, msum = _edge_case(tag)
    with np.errstate(over="ignore"):
        nbr = build(inst, NeighborConfig(theta), consts)
    assert np.array_equal(nbr.lists, want)
    assert np.array_equal(nbr.mask.sum(axis=1), msum)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", EDGE)
def test_device_build_equals_reference_edge_cases(tag):
    inst, consts, theta, want, msum = _edge_case(tag)
    nbr = build_device(inst, NeighborConfig(theta), consts)
    assert nbr.lists.dtype == np.int32 and nbr.lists.shape == want.shape
    assert np.array_equal(nbr.lists, want)
    assert np.array_equal(nbr.mask, _mask_of(want, inst.n_nodes))
    assert np.array_equal(nbr.mask.sum(axis=1), msum)


@pytest.mark.gpu
@pytest.mark.parametrize("group", ["small", "medium", "traj"])
def test_device_build_equals_reference_on_golden_cases(group):
    for case in G.cases(group):
        width = case.nbr.lists.shape[1]
        nbr = build_device(case.inst, NeighborConfig(width), case.consts, with_mask=False)
        assert np.array_equal(nbr.lists, case.nbr.lists), case.tag


@pytest.mark.gpu
def test_device_build_distinct_time_matrix():
    """time is a separate array (not the dist alias): the kernel reads it, not dist."""
    inst, consts, theta, _, _ = _edge_case("tight")
    inst.time = np.ascontiguousarray(inst.dist * 1.25)
    want = build(inst, NeighborConfig(theta), consts)
    got = build_device(inst, NeighborConfig(theta), consts)
    assert np.array_equal(got.lists, want.lists) and np.array_equal(got.mask, want.mask)
