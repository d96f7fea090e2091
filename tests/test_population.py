"""Population management (reference population.py:19-122).

CPU: the scalar restatement in oracle/ against the reference's own survivor
selections and distance matrices (tests/golden/population.json).  GPU: the
device distances and selection (mdr_population_select) against the same
goldens and against the restatement on larger random populations."""
import json
import os
import random

import numpy as np
import pytest

from oracle import population_ref as PR
from paper_2605_05208_b200 import workload as W
from paper_2605_05208_b200.evaluation import EvalBreakdown, PenaltyState
from paper_2605_05208_b200.model import Route, Solution
from paper_2605_05208_b200.population import Population, edge_keys

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "population.json")))


def _inst(spec):
    variant, nc, nd, seed = spec
    return W.make_instance(random.Random(seed), variant, n_customers=nc, n_depots=nd)


def _members(case, inst):
    out = []
    for m in case["members"]:
        sol = Solution([Route(d, a, list(c)) for d, a, c in m["routes"]])
        bd = EvalBreakdown(*[float.fromhex(x) for x in m["bd"]])
        out.append((sol, bd, m["feasible"]))
    return out


def _cost(bd, lam):
    return bd.D + lam[0] * bd.V1 + lam[1] * bd.V2 + lam[2] * bd.V3 + lam[3] * bd.V4


@pytest.mark.parametrize("k", range(len(GOLD)))
def test_restatement_equals_reference(k):
    case = GOLD[k]
    inst = _inst(case["spec"])
    mem = _members(case, inst)
    edges = [edge_keys(s, inst.n_nodes, inst.open_routes) for s, _, _ in mem]
    rows = PR.distance_rows(edges)
    assert [[x.hex() for x in r] for r in rows] == case["dist"]
    births = [m["birth"] for m in case["members"]]
    gone = PR.removal_order(edges, [_cost(bd, case["lam"]) for _, bd, _ in mem], births, case["mu"], case["xi"])
    assert [b for i, b in enumerate(births) if i not in set(gone)] == case["survivors"]


def test_edge_keys_are_the_reference_edge_sets():
    case = GOLD[2]  # open routes
    inst = _inst(case["spec"])
    for s, _, _ in _members(case, inst):
        want = set()
        for r in s.routes:
            if r.customers:
                seq = r.sequence(inst.open_routes)
                want |= {(min(a, b), max(a, b)) for a, b in zip(seq, seq[1:])}
        got = {(int(k) // inst.n_nodes, int(k) % inst.n_nodes) for k in edge_keys(s, inst.n_nodes, True)}
        assert got == want


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(GOLD)))
def test_device_selection_equals_reference(k):
    case = GOLD[k]
    inst = _inst(case["spec"])
    pop = Population(case["mu"], case["xi"])
    for s, bd, f in _members(case, inst):
        pop.add(s, bd, f, inst)
    assert [[x.hex() for x in r] for r in pop.distance_matrix()] == case["dist"]
    pop.survivor_selection(PenaltyState(lam=case["lam"]))
    assert [m.birth for m in pop.members] == case["survivors"]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_device_selection_incremental_vs_restatement(seed):
    """Generations of adds and selections (the distance cache carried across
    them) against the restatement recomputing everything each time."""
    rng = random.Random(seed)
    inst = W.make_instance(random.Random(seed), "mdvrp", n_customers=120, n_depots=4)
    mu, xi = 40, 0.7
    pop = Population(mu, xi)
    ref = []  # (edges, cost, birth)
    birth = 0
    pen = PenaltyState()
    for gen in range(6):
        for _ in range(rng.randint(10, 70)):
            if ref and rng.random() < 0.15:
                src = rng.choice(pop.members)
                s, bd = src.sol.clone(), EvalBreakdown(src.breakdown.D, 0.0, 0.0, 0.0, 0.0)
            else:
                s = W.random_solution(random.Random(rng.randrange(1 << 30)), inst)
                bd = EvalBreakdown(float(rng.randint(0, 50)), 0.0, 0.0, 0.0, 0.0)  # many equal costs
            pop.add(s, bd, True, inst)
            ref.append((edge_keys(s, inst.n_nodes, False), bd.D, birth))
            birth += 1
        if len(pop) > mu:
            gone = set(PR.removal_order([e for e, _, _ in ref], [c for _, c, _ in ref], [b for _, _, b in ref], mu, xi))
            ref = [x for i, x in enumerate(ref) if i not in gone]
            pop.survivor_selection(pen)
            assert [m.birth for m in pop.members] == [b for _, _, b in ref]
    rows = PR.distance_rows([e for e, _, _ in ref])
    assert np.array_equal(np.asarray(pop.distance_matrix()), np.asarray(rows))
