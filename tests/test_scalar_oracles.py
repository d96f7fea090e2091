"""Scalar oracles of the reference test path:
evaluate, move_delta, check_feasible, simulate_route, minimal_duration -- against
the reference's own values (tests/golden/scalar.json, make_scalar_golden.py)."""
import json
import os
import random

import pytest

from paper_2605_05208_b200 import workload as W
from oracle import feasibility_ref as FR, scalar_ref as SR
from paper_2605_05208_b200 import evaluation as EV, feasibility as FD
from paper_2605_05208_b200.evaluation import PenaltyState, ScalingConstants
from paper_2605_05208_b200.moves import Move, Op

CASES = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scalar.json")))
H = lambda x: float(x).hex()  # noqa: E731


def _case(c):
    inst = W.make_instance(random.Random(c["iseed"]), c["variant"], n_customers=c["nc"], n_depots=c["nd"], **c["kw"])
    sol = W.random_solution(random.Random(c["sseed"]), inst)
    if c["emptied"] and sol.routes:
        sol.routes[0].customers = []
    return inst, sol


IMPLS = [pytest.param("oracle", id="oracle"), pytest.param("device", id="device", marks=pytest.mark.gpu)]


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("i", range(len(CASES)))
def test_evaluate_and_feasibility_equal_reference(i, impl):
    """oracle: the scalar restatements (test checkers); device: the product's
    evaluate (mdr_pop_breakdown) and check_feasible / simulate_route /
    minimal_duration (mdr_route_sim)."""
    evaluate = SR.evaluate if impl == "oracle" else EV.evaluate
    M = FR if impl == "oracle" else FD
    check_feasible, simulate_route, minimal_duration = M.check_feasible, M.simulate_route, M.minimal_duration
    c = CASES[i]
    inst, sol = _case(c)
    consts = ScalingConstants.from_instance(inst)
    bd = evaluate(sol, PenaltyState(lam=c["lam"]), consts, inst)
    assert [H(x) for x in (bd.D, bd.V1, bd.V2, bd.V3, bd.V4, bd.F)] == c["evaluate"]
    fr, want = check_feasible(sol, inst), c["report"]
    assert fr.structural_error == want["structural_error"]
    assert fr.missing == want["missing"] and fr.duplicated == want["duplicated"]
    assert [H(fr.capacity_excess), H(fr.duration_excess), H(fr.time_warp)] == \
        [want["capacity_excess"], want["duration_excess"], want["time_warp"]]
    assert (fr.late_count, fr.closure_violations, fr.fleet_excess, fr.all_ok) == \
        (want["late_count"], want["closure_violations"], want["fleet_excess"], want["all_ok"])
    sims = []
    for r in sol.routes:
        if r.customers:
            s = simulate_route(r, inst)
            sims.append([H(s.distance), H(s.load), H(s.duration), H(s.time_warp), s.late_count,
                         H(minimal_duration(r, inst))])
    assert sims == c["sims"]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_move_delta_equals_reference(i):
    c = CASES[i]
    inst, sol = _case(c)
    consts = ScalingConstants.from_instance(inst)
    pen = PenaltyState(lam=c["lam"])
    for key, want in c["move_deltas"]:
        op, r1, r2, p1, p2, l1, l2, v1, v2, dep, mode = key
        mv = Move(Op(op), r1, p1, r2, p2, l1, l2, bool(v1), bool(v2), dep, mode)
        d = SR.move_delta(sol, mv, pen, consts, inst)
        assert [H(x) for x in (d.D, d.V1, d.V2, d.V3, d.V4, d.F)] == want, key
