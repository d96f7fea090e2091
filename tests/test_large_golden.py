"""Reference goldens at the benchmark shapes (tests/golden/large.json, made by
tests/golden/make_golden_large.py from the real reference package).

BASELINE.json configs[3] (C4: MDVRPTW 1000x10) and configs[4] (C5: MDVRP
4000x20, theta 40), Appendix-A instances (seed 2026):
* the rebuilt instance, constants and neighbour lists equal the reference's;
* workload.initial_solution reproduces the reference's start states;
* the oracle's operator-level results at individual 0's start state equal the
  reference's (candidate/delta array SHA, leader, followers, select_moves), and
  the device's do too (GPU);
* the oracle's complete C4 descent of individual 0 equals the reference's
  (final routes, lambda, passes, per-operator candidate counts); the device's
  C4 descents are checked against both reference descents inside the
  population-256 run of tests/test_gpu_shapes.py.
"""
import hashlib
import json
import os
import random
from functools import lru_cache

import numpy as np
import pytest

import golden_io as G
import paper_2605_05208_b200 as P
from paper_2605_05208_b200 import workload as W
from paper_2605_05208_b200.localsearch import draw_permutations
from oracle import oracle as O

GOLD = json.load(open(os.path.join(G.GOLD, "large.json")))


@lru_cache(None)
def built(name):
    spec = W.CONFIGS[name]
    inst, _ = W.appendix_a_instance(spec)
    consts = P.ScalingConstants.from_instance(inst)
    nbr = P.build_neighbors(inst, P.NeighborConfig(spec.theta), consts)
    return inst, consts, nbr


def start(name, i):
    g = GOLD[name]["starts"][i]
    return P.Solution([P.Route(d, a, list(c)) for d, a, c in g])


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_large_instance_constants_lists_equal_reference(name):
    inst, consts, nbr = built(name)
    g = GOLD[name]
    assert _sha(np.ascontiguousarray(inst.dist, np.float64)) == g["dist_sha"]
    assert (inst.time is inst.dist) == g["time_is_dist"]
    assert consts.gamma.hex() == g["gamma"] and consts.theta.hex() == g["theta"]
    assert _sha(np.ascontiguousarray(nbr.lists, np.int32)) == g["lists_sha"]


@pytest.mark.parametrize("impl", [pytest.param("oracle"), pytest.param("device", marks=pytest.mark.gpu)])
@pytest.mark.parametrize("name,i", [("C4", 0), ("C4", 1), ("C4", 2), ("C4", 3), ("C5", 0), ("C5", 3)])
def test_start_states_equal_reference(name, i, impl):
    from oracle import initial_ref
    from paper_2605_05208_b200 import genetic
    inst, consts, _ = built(name)
    make = initial_ref.initial_solution if impl == "oracle" else genetic.initial_solution
    s = make(inst, consts, P.PenaltyState(), random.Random(100 + i))
    assert G.routes_of(s) == [(d, a, list(c)) for d, a, c in GOLD[name]["starts"][i]]


def _check_ops(name, enum, evaluate, leader_followers):
    inst, consts, nbr = built(name)
    g = GOLD[name]
    sol = start(name, 0)
    for op in range(6):
        rec = g["ops"][str(op)]
        if op == 3 and inst.has_windows:
            assert rec["n"] == 0
            continue
        cands = enum(sol, op)
        assert len(cands["r1"]) == rec["n"], f"{name} op {op}: candidate count"
        d = evaluate(sol, op, cands)
        cm = np.stack([np.asarray(cands[f]).astype(np.int64) for f in G.FIELDS])
        dm = np.stack([d[f] for f in G.DFIELDS])
        assert G.canon_sha(cm, dm, np.asarray(d["fleet_neutral"]).astype(np.uint8)) == rec["sha"], f"{name} op {op}"
        best, fol = leader_followers(cands, d)
        if rec["leader"] is None:
            assert best < 0
        else:
            assert [int(cands[f][best]) for f in ("r1", "r2", "p1", "p2", "len1", "len2", "rev1", "rev2", "depot",
                                                  "mode")] == rec["leader"][1:]
            assert len(fol) == rec["n_followers"]
        del cands, d, cm, dm


def test_oracle_c4_operator_level_equals_reference():
    inst, consts, nbr = built("C4")
    oi = O.OracleInstance(inst, consts, nbr)
    _check_ops("C4", lambda s, op: O.enumerate_op(oi, s, op),
               lambda s, op, c: O.evaluate(oi, s, op, c, [1.0] * 4),
               lambda c, d: O.leader_followers(c, d, True))
    assert [x.hex() for x in O.totals(oi, start("C4", 0))] == GOLD["C4"]["totals"]


def test_oracle_c4_complete_descent_equals_reference():
    inst, consts, nbr = built("C4")
    oi = O.OracleInstance(inst, consts, nbr)
    g = GOLD["C4"]["descents"]["0"]
    perms = draw_permutations(random.Random(0), P.enabled_operators(inst), 501)
    routes, lam, st, _ = O.local_search(oi, start("C4", 0), [1.0] * 4, 500, True, 0.5, 0.01, 1e4, perms)
    assert routes == [(d, a, list(c)) for d, a, c in g["final"]]
    assert [x.hex() for x in lam] == g["lam"]
    assert st["passes"] == g["passes"] and st["accepted"] == g["accepted"]
    assert st["cands"] == g["cands"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C4", "C5"])
def test_device_operator_level_equals_reference(name):
    from paper_2605_05208_b200.device import DeviceInstance, Population
    inst, consts, nbr = built(name)
    sol = start(name, 0)
    dinst = DeviceInstance(inst, consts, nbr)
    J, K = Population.caps_for([sol], inst)
    pop = Population(dinst, 1, J, K, 1 << 14)
    pop.upload([sol], [[1.0] * 4])
    _check_ops(name, lambda s, op: pop.enumerate(0, op), lambda s, op, c: pop.evaluate(0, op, c, [1.0] * 4),
               lambda c, d: pop.leader_followers(c, d, True))
    assert [x.hex() for x in pop.totals(0)] == GOLD[name]["totals"]
