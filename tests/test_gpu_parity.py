"""GPU parity: the sm_100a path (through the C-ABI) against the reference's
golden outputs and the C oracle.  Bit-exact (`==`, -0.0 == +0.0) everywhere."""
import random

import numpy as np
import pytest

import golden_io as G
import paper_2605_05208_b200 as P
from paper_2605_05208_b200 import workload as W
from paper_2605_05208_b200.device import DeviceInstance, Population
from paper_2605_05208_b200.localsearch import draw_permutations
from oracle import oracle as O

pytestmark = pytest.mark.gpu

KEY_FIELDS = ("r1", "r2", "p1", "p2", "len1", "len2", "rev1", "rev2", "depot", "mode")


def _cm(c):
    return np.stack([np.asarray(c[f]).astype(np.int64) for f in G.FIELDS])


def _key(c, i):
    return [int(c[f][i]) for f in KEY_FIELDS]


def _pop_for(case, nbr=True):
    di = DeviceInstance(case.inst, case.consts, case.nbr if nbr else None)
    J, K = Population.caps_for([case.sol], case.inst)
    pop = Population(di, 1, J, K, 1 << 12)
    pop.upload([case.sol], [case.lam])
    return pop


@pytest.mark.parametrize("case", G.cases("small"), ids=lambda c: c.tag)
def test_ops_small_vs_reference_golden(case):
    pop = _pop_for(case)
    for op in range(6):
        cands, deltas = case.op_full(op)
        if op == 3 and case.inst.has_windows:
            assert len(cands["r1"]) == 0
        else:
            got = pop.enumerate(0, op)
            assert np.array_equal(_cm(got), _cm(cands)), f"op {op}: device enumeration differs"
        if len(cands["r1"]) == 0:
            continue
        d = pop.evaluate(0, op, cands, case.lam)
        for f in G.DFIELDS + ("fleet_neutral",):
            assert np.array_equal(d[f], deltas[f]), f"op {op} field {f}"
        rec = case.meta["ops"][str(op)]
        best, fol = pop.leader_followers(cands, deltas, True)
        if rec["leader"] is None:
            assert best < 0
        else:
            assert _key(cands, best) == rec["leader"][1:]
            assert len(fol) == rec["n_followers"]
            assert [_key(cands, i) for i in fol[:256]] == [k[1:] for k in rec["followers"]]
    assert [x.hex() for x in pop.totals(0)] == case.meta["totals"]


@pytest.mark.parametrize("case", G.cases("medium"), ids=lambda c: c.tag)
def test_ops_medium_vs_reference_golden(case):
    pop = _pop_for(case)
    for op in range(6):
        rec = case.meta["ops"][str(op)]
        if op == 3 and case.inst.has_windows:
            assert rec["n"] == 0
            continue
        got = pop.enumerate(0, op)
        assert len(got["r1"]) == rec["n"]
        d = pop.evaluate(0, op, got, case.lam)
        dm = np.stack([d[f] for f in G.DFIELDS])
        assert G.canon_sha(_cm(got), dm, d["fleet_neutral"].astype(np.uint8)) == rec["sha"], f"op {op}"
        if rec["n"]:
            best, fol = pop.leader_followers(got, d, True)
            if rec["leader"] is None:
                assert best < 0
            else:
                assert _key(got, best) == rec["leader"][1:]
                assert len(fol) == rec["n_followers"]


@pytest.mark.parametrize("case", G.cases("traj"), ids=lambda c: c.tag)
def test_local_search_api_vs_reference_trajectory(case):
    m = case.meta
    sol = case.sol.clone()
    pen = P.PenaltyState()
    rng = random.Random(m["ls_seed"])
    P.local_search(sol, pen, P.SearchConfig(depth=m["depth"], multi_move=m["multi_move"]), case.nbr,
                   case.consts, case.inst, rng)
    assert G.routes_of(sol) == case.final_routes()
    assert [x.hex() for x in pen.lam] == m["final_lam"]
    ref = random.Random(m["ls_seed"])
    for _ in range(m["passes"]):
        o = list(P.enabled_operators(case.inst))
        ref.shuffle(o)
    assert rng.getstate() == ref.getstate(), "rng not advanced by exactly one shuffle per pass"


def _synthetic_states(variant, n_customers, n_depots, seed, count, **kw):
    rng = random.Random(seed)
    inst = W.make_instance(rng, variant, n_customers=n_customers, n_depots=n_depots, **kw)
    consts = P.ScalingConstants.from_instance(inst)
    nbr = P.build_neighbors(inst, P.NeighborConfig(10), consts)
    sols = [W.random_solution(random.Random(seed * 1000 + i), inst) for i in range(count)]
    return inst, consts, nbr, sols


@pytest.mark.parametrize("variant,fleet,dur,mm", [
    ("mdvrp", None, None, True), ("mdvrp", 3, 250.0, False), ("mdvrptw", 4, 500.0, True),
    ("mdvrptw", None, None, False), ("mdovrp", 2, None, True), ("mdovrp", None, None, False)])
def test_population_descents_bit_exact_vs_oracle(variant, fleet, dur, mm):
    inst, consts, nbr, sols = _synthetic_states(variant, 60, 3, hash((variant, fleet, mm)) % 1000, 12,
                                                fleet=fleet, max_duration=dur)
    cfg = P.SearchConfig(depth=500, multi_move=mm)
    ops = P.enabled_operators(inst)
    oi = O.OracleInstance(inst, consts, nbr)
    want = []
    for i, s in enumerate(sols):
        perms = draw_permutations(random.Random(i), ops, cfg.depth + 1)
        want.append(O.local_search(oi, s, [1.0] * 4, cfg.depth, mm, 0.5, 0.01, 1e4, perms))
    work = [s.clone() for s in sols]
    pens = [P.PenaltyState() for _ in sols]
    stats = P.local_search_population(work, pens, cfg, nbr, consts, inst, [random.Random(i) for i in range(12)])
    for i in range(len(sols)):
        routes, lam, st, _ = want[i]
        assert G.routes_of(work[i]) == routes, f"individual {i}"
        assert pens[i].lam == lam
        assert stats[i]["passes"] == st["passes"] and stats[i]["accepted"] == st["accepted"]
        assert stats[i]["cands"] == st["cands"], "candidate counts per operator must equal the reference's"


def test_appendix_a_c2_shape_descents_vs_oracle():
    spec = W.CONFIGS["C2"]
    inst, _ = W.appendix_a_instance(spec)
    consts = P.ScalingConstants.from_instance(inst)
    nbr = P.build_neighbors(inst, P.NeighborConfig(spec.theta), consts)
    sols = [W.initial_solution(inst, consts, P.PenaltyState(), random.Random(100 + i)) for i in range(4)]
    cfg = P.SearchConfig(depth=40, multi_move=True)
    ops = P.enabled_operators(inst)
    oi = O.OracleInstance(inst, consts, nbr)
    work = [s.clone() for s in sols]
    pens = [P.PenaltyState() for _ in sols]
    stats = P.local_search_population(work, pens, cfg, nbr, consts, inst, [random.Random(i) for i in range(4)])
    for i, s in enumerate(sols):
        perms = draw_permutations(random.Random(i), ops, cfg.depth + 1)
        routes, lam, st, _ = O.local_search(oi, s, [1.0] * 4, cfg.depth, True, 0.5, 0.01, 1e4, perms)
        assert G.routes_of(work[i]) == routes
        assert pens[i].lam == lam
        assert stats[i]["cands"] == st["cands"]


def test_capacity_overflow_is_retried():
    inst, consts, nbr, sols = _synthetic_states("mdvrp", 40, 2, 5, 3)
    di = DeviceInstance(inst, consts, nbr)
    pop = Population(di, 3, len(max(sols, key=lambda s: len(s.routes)).routes) + 1, 6, 4)
    pop.upload(sols, [[1.0] * 4] * 3)
    ops = P.enabled_operators(inst)
    perms = np.stack([draw_permutations(random.Random(i), ops, 501) for i in range(3)])
    with pytest.raises(P._lib.CapacityError):
        pop.local_search(perms, 500, True, 0.5, 0.01, 1e4)
    # the public API re-creates the population with larger caps and gets the oracle answer
    work = [s.clone() for s in sols]
    pens = [P.PenaltyState() for _ in sols]
    P.local_search_population(work, pens, P.SearchConfig(500, True), nbr, consts, inst,
                              [random.Random(i) for i in range(3)])
    oi = O.OracleInstance(inst, consts, nbr)
    for i, s in enumerate(sols):
        routes, lam, _, _ = O.local_search(oi, s, [1.0] * 4, 500, True, 0.5, 0.01, 1e4, perms[i])
        assert G.routes_of(work[i]) == routes


def test_deadline_stops_early():
    inst, consts, nbr, sols = _synthetic_states("mdvrp", 60, 3, 9, 2)
    sol = sols[0].clone()
    pen = P.PenaltyState()
    import time
    P.local_search(sol, pen, P.SearchConfig(500, True), nbr, consts, inst, random.Random(1),
                   deadline=time.monotonic() - 1.0)
    assert sorted(sol.customer_list()) == sorted(sols[0].customer_list())


def test_on_feasible_reports_best_feasible_state():
    inst, consts, nbr, sols = _synthetic_states("mdvrp", 30, 2, 21, 1)
    sol = sols[0].clone()
    seen = []
    P.local_search(sol, P.PenaltyState(), P.SearchConfig(500, True), nbr, consts, inst, random.Random(3),
                   on_feasible=lambda D, s: seen.append((D, G.routes_of(s))))
    oi = O.OracleInstance(inst, consts, nbr)
    perms = draw_permutations(random.Random(3), P.enabled_operators(inst), 501)
    _, _, st, tr = O.local_search(oi, sols[0], [1.0] * 4, 500, True, 0.5, 0.01, 1e4, perms, trace_cap=501)
    if st["n_feasible"]:
        assert len(seen) == 1 and seen[0][0] == st["best_feasible_D"]
    else:
        assert not seen
