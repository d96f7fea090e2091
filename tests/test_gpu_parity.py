"""GPU parity: the sm_100a path (through the C-ABI) against the reference's
golden outputs and the C oracle.  Bit-exact (`==`, -0.0 == +0.0) everywhere."""
import os
import random
import zlib

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
    inst, consts, nbr, sols = _synthetic_states(variant, 60, 3, zlib.crc32(repr((variant, fleet, mm)).encode()) % 1000, 12,
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


FUZZ = list(range(int(os.environ.get("MDR_FUZZ_N", "64"))))  # more: MDR_FUZZ_N=500


@pytest.mark.parametrize("seed", FUZZ)
def test_fuzz_descents_bit_exact_vs_oracle(seed):
    """Randomised shapes: variant, 2-120 customers, 1-6 depots, fleet limits
    (incl. one vehicle per depot), tight or loose capacity and duration,
    theta 1-30, depth 1-300, single/multi-move, lambda != 1 starts."""
    r = random.Random(9000 + seed)
    variant = r.choice(["mdvrp", "mdvrptw", "mdovrp"])
    nc, nd = r.randint(2, 120), r.randint(1, 6)
    fleet = r.choice([None, None, 1, 2, 4])
    cap = r.choice([None, 15, 40, 1000])
    dur = r.choice([None, None, 150.0, 400.0]) if variant != "mdovrp" else None
    inst = W.make_instance(r, variant, n_customers=nc, n_depots=nd, capacity=cap, max_duration=dur, fleet=fleet)
    consts = P.ScalingConstants.from_instance(inst)
    nbr = P.build_neighbors(inst, P.NeighborConfig(r.choice([1, 3, 8, 30])), consts)
    count = r.randint(1, 6)
    sols = [W.random_solution(random.Random(seed * 100 + i), inst, scramble_depots=r.random() < 0.5)
            for i in range(count)]
    depth, mm = r.randint(1, 300), r.random() < 0.6
    lams = [[r.choice([0.01, 0.3, 1.0, 7.0]) for _ in range(4)] for _ in range(count)]
    cfg = P.SearchConfig(depth=depth, multi_move=mm)
    ops = P.enabled_operators(inst)
    oi = O.OracleInstance(inst, consts, nbr)
    want = []
    for i, s in enumerate(sols):
        perms = draw_permutations(random.Random(i), ops, depth + 1)
        want.append(O.local_search(oi, s, lams[i], depth, mm, 0.5, 0.01, 1e4, perms))
    work = [s.clone() for s in sols]
    pens = [P.PenaltyState(lam=list(l)) for l in lams]
    rngs = [random.Random(i) for i in range(count)]
    stats = P.local_search_population(work, pens, cfg, nbr, consts, inst, rngs)
    for i in range(count):
        routes, lam, st, _ = want[i]
        assert G.routes_of(work[i]) == routes, f"seed {seed} individual {i}"
        assert pens[i].lam == lam
        assert stats[i]["passes"] == st["passes"] and stats[i]["cands"] == st["cands"]
        ref_rng = random.Random(i)
        for _ in range(st["passes"]):
            ref_rng.shuffle(list(ops))
        assert rngs[i].getstate() == ref_rng.getstate()


def test_appendix_a_c2_shape_descents_vs_oracle():
    spec = W.CONFIGS["C2"]
    inst, _ = W.appendix_a_instance(spec)
    consts = P.ScalingConstants.from_instance(inst)
    nbr = P.build_neighbors(inst, P.NeighborConfig(spec.theta), consts)
    sols = P.initial_solutions(inst, consts, P.PenaltyState(), [random.Random(100 + i) for i in range(4)])
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


@pytest.mark.parametrize("seed", [3, 4, 5, 6])
def test_on_feasible_per_state_and_attrs(seed):
    """on_feasible(D, sol) fires on every feasible post-step state, in order
    (localsearch.py:133-134: D values hex-equal to the oracle's trace); with
    feasible_best_only once with the lowest D.  Routes are mutated in place and
    their attr caches equal the scalar route_attr of the final routes."""
    from oracle.scalar_ref import route_attr
    inst, consts, nbr, sols = _synthetic_states(["mdvrp", "mdvrptw", "mdovrp", "mdvrptw"][seed % 4], 30, 2, 21 + seed, 1)
    oi = O.OracleInstance(inst, consts, nbr)
    perms = draw_permutations(random.Random(seed), P.enabled_operators(inst), 501)
    want_routes, _, st, tr = O.local_search(oi, sols[0], [1.0] * 4, 500, True, 0.5, 0.01, 1e4, perms, trace_cap=501)
    sol = sols[0].clone()
    objs = list(sol.routes)
    seen = []
    P.local_search(sol, P.PenaltyState(), P.SearchConfig(500, True), nbr, consts, inst, random.Random(seed),
                   on_feasible=lambda D, s: seen.append((D.hex(), G.routes_of(s))))
    assert [d for d, _ in seen] == [float(x).hex() for x, f in zip(tr["D"], tr["feasible"]) if f]
    assert G.routes_of(sol) == want_routes
    assert any(r is o for r in sol.routes for o in objs)  # the caller's Route objects are mutated, not replaced
    for r in sol.routes:
        if r.attr is not None:
            w = route_attr(r, inst)
            assert [x.hex() for x in (r.attr.dist, r.attr.load, r.attr.T, r.attr.E, r.attr.L, r.attr.TW)] == \
                [float(x).hex() for x in (w.dist, w.load, w.T, w.E, w.L, w.TW)]
            assert (r.attr.first, r.attr.last) == (w.first, w.last)
    best = []
    P.local_search(sols[0].clone(), P.PenaltyState(), P.SearchConfig(500, True), nbr, consts, inst,
                   random.Random(seed), on_feasible=lambda D, s: best.append(D), feasible_best_only=True)
    if st["n_feasible"]:
        assert best == [st["best_feasible_D"]]
    else:
        assert not best and not seen


@pytest.mark.parametrize("name,pop,depth", [("C1", 6, 500), ("C3", 3, 60), ("C5", 1, 8)])
def test_appendix_a_configs_descents_vs_oracle(name, pop, depth):
    """BASELINE.json shapes (MDVRP 50x4, MDOVRP 360x9, MDVRP 4000x20 theta 40): short
    population descents bit-exact against the oracle, counts included."""
    spec = W.CONFIGS[name]
    inst, _ = W.appendix_a_instance(spec)
    consts = P.ScalingConstants.from_instance(inst)
    nbr = P.build_neighbors(inst, P.NeighborConfig(spec.theta), consts)
    sols = P.initial_solutions(inst, consts, P.PenaltyState(), [random.Random(100 + i) for i in range(pop)])
    cfg = P.SearchConfig(depth=depth, multi_move=True)
    ops = P.enabled_operators(inst)
    oi = O.OracleInstance(inst, consts, nbr)
    work = [s.clone() for s in sols]
    pens = [P.PenaltyState() for _ in sols]
    stats = P.local_search_population(work, pens, cfg, nbr, consts, inst, [random.Random(i) for i in range(pop)])
    for i, s in enumerate(sols):
        perms = draw_permutations(random.Random(i), ops, cfg.depth + 1)
        routes, lam, st, _ = O.local_search(oi, s, [1.0] * 4, cfg.depth, True, 0.5, 0.01, 1e4, perms)
        assert G.routes_of(work[i]) == routes, f"{name} individual {i}"
        assert pens[i].lam == lam
        assert stats[i]["cands"] == st["cands"]


def test_edge_cases_empty_routes_unrouted_and_single_move():
    """Input with empty routes and an unrouted customer, single-move mode, depth 1 and 3."""
    rng = random.Random(17)
    for variant in ("mdvrp", "mdvrptw", "mdovrp"):
        inst = W.make_instance(rng, variant, n_customers=25, n_depots=3, fleet=2,
                               max_duration=None if variant == "mdovrp" else 400.0)
        consts = P.ScalingConstants.from_instance(inst)
        nbr = P.build_neighbors(inst, P.NeighborConfig(8), consts)
        oi = O.OracleInstance(inst, consts, nbr)
        for depth, mm in ((1, False), (3, True), (500, False)):
            sol = W.random_solution(random.Random(depth), inst)
            sol.routes.insert(1, P.Route(0, 0, []))
            sol.routes.append(P.Route(1, 2 if variant != "mdovrp" else 1, []))
            sol.routes[0].customers.pop()  # one unrouted customer
            perms = draw_permutations(random.Random(5), P.enabled_operators(inst), depth + 1)
            routes, lam, st, _ = O.local_search(oi, sol, [1.0] * 4, depth, mm, 0.5, 0.01, 1e4, perms)
            work = sol.clone()
            pen = P.PenaltyState()
            P.local_search(work, pen, P.SearchConfig(depth, mm), nbr, consts, inst, random.Random(5))
            assert G.routes_of(work) == routes, (variant, depth, mm)
            assert pen.lam == lam


def test_operator_level_api_on_random_states_vs_oracle():
    """enumerate_candidates / evaluate_candidates / leader_and_followers through the
    reference-shaped API on larger random states."""
    rng = random.Random(99)
    for variant in ("mdvrp", "mdvrptw", "mdovrp"):
        inst = W.make_instance(rng, variant, n_customers=80, n_depots=4, fleet=5, max_duration=None)
        consts = P.ScalingConstants.from_instance(inst)
        nbr = P.build_neighbors(inst, P.NeighborConfig(15), consts)
        sol = W.random_solution(random.Random(3), inst)
        pen = P.PenaltyState(lam=[0.3, 2.0, 1.7, 0.9])
        oi = O.OracleInstance(inst, consts, nbr)
        cache = P.SolutionCache(sol, inst, consts)
        for op in P.enabled_operators(inst):
            cs = P.enumerate_candidates(sol, op, nbr, inst)
            want = O.enumerate_op(oi, sol, int(op))
            assert np.array_equal(_cm({f: getattr(cs, f) for f in G.FIELDS}), _cm(want))
            d = P.evaluate_candidates(cache, cs, pen)
            od = O.evaluate(oi, sol, int(op), want, pen.lam)
            for f in G.DFIELDS + ("fleet_neutral",):
                assert np.array_equal(getattr(d, f), od[f]), (variant, op, f)
            leader, fol = P.leader_and_followers(cache, cs, d, True)
            best, ofol = O.leader_followers(want, od, True)
            assert (leader is None) == (best < 0)
            if leader is not None:
                assert leader.key()[1:] == tuple(_key(want, best))
                assert [m.key()[1:] for m in fol] == [tuple(_key(want, i)) for i in ofol]
        assert [x.hex() for x in cache.totals()] == [x.hex() for x in O.totals(oi, sol)]


def test_many_routes_beyond_2046_capacity_path():
    """Random C5-shaped start (~1300 short routes): population caps grow to 4094 routes,
    the CTA-staging is disabled (too many routes for shared memory) and the warp-task
    path runs; trajectory bit-exact vs the oracle."""
    spec = W.CONFIGS["C5"]
    inst, _ = W.appendix_a_instance(spec)
    consts = P.ScalingConstants.from_instance(inst)
    nbr = P.build_neighbors(inst, P.NeighborConfig(spec.theta), consts)
    sol = W.random_solution(random.Random(301), inst)
    assert len(sol.routes) > 1100
    work = sol.clone()
    pen = P.PenaltyState()
    P.local_search(work, pen, P.SearchConfig(depth=3, multi_move=True), nbr, consts, inst, random.Random(0))
    oi = O.OracleInstance(inst, consts, nbr)
    perms = draw_permutations(random.Random(0), P.enabled_operators(inst), 4)
    routes, lam, st, _ = O.local_search(oi, sol, [1.0] * 4, 3, True, 0.5, 0.01, 1e4, perms)
    assert G.routes_of(work) == routes
    assert pen.lam == lam


def test_totals_pairwise_sum_many_routes():
    """SolutionCache.totals() uses numpy's pairwise summation; check the device
    restatement bit for bit on route lists far beyond one 128-element block."""
    rng = random.Random(8)
    for variant in ("mdvrptw", "mdvrp"):
        inst = W.make_instance(rng, variant, n_customers=1500, n_depots=5, max_duration=300.0, capacity=15)
        consts = P.ScalingConstants.from_instance(inst)
        nbr = P.build_neighbors(inst, P.NeighborConfig(5), consts)
        oi = O.OracleInstance(inst, consts, nbr)
        for seed in range(3):
            sol = W.random_solution(random.Random(seed), inst)
            assert len(sol.routes) > 300
            cache = P.SolutionCache(sol, inst, consts)
            assert [x.hex() for x in cache.totals()] == [x.hex() for x in O.totals(oi, sol)]


@pytest.mark.gpu
def test_download_range_matches_full_download():
    inst, consts, nbr, sols = _synthetic_states("mdvrptw", 40, 3, 77, 7)
    dinst = DeviceInstance(inst, consts, nbr)
    J, K = Population.caps_for(sols, inst)
    pop = Population(dinst, 7, J, K)
    pop.upload(sols, [[1.0] * 4] * 7)
    full, _ = pop.download()
    for b0, nb in ((0, 7), (3, 1), (6, 1), (2, 3), (4, 0)):
        assert pop.download_range(b0, nb) == full[b0:b0 + nb]
    with pytest.raises(ValueError):
        pop.download_range(5, 3)


@pytest.mark.gpu
def test_abi_argument_errors_raise():
    """Bad arguments fail loudly at the C-ABI (ValueError like the reference), never silently."""
    from paper_2605_05208_b200.model import Route, Solution
    inst, consts, nbr, sols = _synthetic_states("mdvrp", 20, 2, 5, 2)
    dinst = DeviceInstance(inst, consts, nbr)
    pop = Population(dinst, 2, 40, 32)
    with pytest.raises(ValueError):  # route endpoint is not a depot
        pop.upload([Solution([Route(5, 0, [6, 7])])], [[1.0] * 4])
    with pytest.raises(ValueError):  # a depot listed as a customer
        pop.upload([Solution([Route(0, 0, [1, 6])])], [[1.0] * 4])
    pop.upload(sols[:1], [[1.0] * 4])
    with pytest.raises(ValueError):  # unknown insertion operator
        pop.repair(7, [[]])
    with pytest.raises(ValueError):
        pop.download_range(0, 2)
    from paper_2605_05208_b200 import _lib
    with pytest.raises(ValueError):  # theta must be >= 1, buffers non-null
        _lib.check(_lib.lib().mdr_neighbor_build(0, inst.n_nodes, inst.n_depots, None, None, None, None, None,
                                                 1.0, 1.0, 10.0, 0, None, None, None), "mdr_neighbor_build")
