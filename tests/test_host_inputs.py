"""CPU tests of the host-side input preparation, pinned to the reference's outputs
in the golden fixtures: neighbour lists, scaling constants, Appendix A instances and
initial solutions, and the flat solution layout of the C-ABI."""
import random

import numpy as np
import pytest

import golden_io as G
from paper_2605_05208_b200 import workload as W
from paper_2605_05208_b200.device import Population, flatten_population
from paper_2605_05208_b200.evaluation import PenaltyState, ScalingConstants, adapt_penalties
from paper_2605_05208_b200.model import Route, flatten, unflatten
from paper_2605_05208_b200.neighborhood import NeighborConfig, build


@pytest.mark.parametrize("group", ["small", "medium", "traj"])
def test_neighbor_lists_and_constants_equal_reference(group):
    for case in G.cases(group):
        consts = ScalingConstants.from_instance(case.inst)
        assert consts.gamma.hex() == case.meta["gamma"] and consts.theta.hex() == case.meta["theta"]
        width = case.nbr.lists.shape[1]
        nbr = build(case.inst, NeighborConfig(width), consts)
        assert np.array_equal(nbr.lists, case.nbr.lists), case.tag


@pytest.mark.parametrize("impl", [pytest.param("oracle"), pytest.param("device", marks=pytest.mark.gpu)])
@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_appendix_a_initial_solution_equals_reference(name, impl):
    """medium golden '<name>_init' = reference genetic.initial_solution continuing the
    seed-2026 stream after the Appendix A instance draws.  oracle: the scalar
    restatement; device: genetic.initial_solution (mdr_construct + IBI repair)."""
    from oracle import initial_ref
    from paper_2605_05208_b200 import genetic
    case = [c for c in G.cases("medium") if c.tag == f"{name}_init"][0]
    inst, rng = W.appendix_a_instance(W.CONFIGS[name])
    assert np.array_equal(inst.dist, case.inst.dist)
    consts = ScalingConstants.from_instance(inst)
    make = initial_ref.initial_solution if impl == "oracle" else genetic.initial_solution
    sol = make(inst, consts, PenaltyState(), rng)
    assert G.routes_of(sol) == G.routes_of(case.sol)


def test_flat_layouts_round_trip():
    inst = W.make_instance(random.Random(2), "mdvrptw", n_customers=40, n_depots=3)
    sols = [W.random_solution(random.Random(i), inst) for i in range(5)]
    sols[2].routes.insert(0, Route(1, 1, []))
    off, cust, dep, arr = flatten(sols[0])
    back = unflatten(off, cust, dep, arr)
    assert [(r.depart, r.arrive, r.customers) for r in back] == G.routes_of(sols[0])
    rbase, coff, cust, dep, arr = flatten_population(sols)
    assert rbase[-1] == sum(len(s.routes) for s in sols)
    for b, s in enumerate(sols):
        got = [(int(dep[r]), int(arr[r]), cust[coff[r]:coff[r + 1]].tolist()) for r in range(rbase[b], rbase[b + 1])]
        assert got == G.routes_of(s)
    J, K = Population.caps_for(sols, inst)
    assert J >= 2 * max(len(s.routes) for s in sols) and K >= 32


def test_adapt_penalties_matches_reference_rule():
    p = PenaltyState(kappa=0.5, lam=[1.0, 0.015, 9000.0, 2.0])
    adapt_penalties(p, [True, False, True, False])
    assert p.lam == [2.0, 0.01, 10000.0, 1.0]
    with pytest.raises(ValueError):
        PenaltyState(kappa=1.0)
