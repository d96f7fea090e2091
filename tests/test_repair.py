"""Repair insertion: the oracle restatement and the device
path (mdr_repair) against the reference's own repair_insert outputs
(tests/golden/repair.npz from make_repair_golden.py)."""
import os
import random
import zlib

import pytest

import repair_io as R
from oracle import oracle as O
from paper_2605_05208_b200 import workload as W
from paper_2605_05208_b200.evaluation import PenaltyState, ScalingConstants
from paper_2605_05208_b200.genetic import InsertionOperator, repair_insert, repair_population
from paper_2605_05208_b200.model import INF, Instance, Route, Solution
from paper_2605_05208_b200.neighborhood import NeighborConfig, build

TAGS = R.tags()
DET = [t for t in TAGS if R.RepairCase(t).op != "RI"]
RI = [t for t in TAGS if R.RepairCase(t).op == "RI"]


def _oi(inst, consts):
    return O.OracleInstance(inst, consts, build(inst, NeighborConfig(4), consts))


def test_golden_covers_every_operator_and_variant():
    cases = [R.RepairCase(t) for t in TAGS]
    assert {c.op for c in cases} == {"FBI", "IBI", "FRI", "IRI", "RI"}
    assert {c.meta["variant"] for c in cases} == {"mdvrp", "mdvrptw", "mdovrp"}
    assert any(not c.sol.routes for c in cases)  # every route removed
    assert any(any(not r.customers for r in c.sol.routes) for c in cases)  # emptied routes kept


@pytest.mark.parametrize("tag", DET)
def test_oracle_repair_equals_reference(tag):
    c = R.RepairCase(tag)
    got, _ = O.repair(_oi(c.inst, c.consts), c.sol, c.unrouted, O.REPAIR_OPS[c.op], c.lam)
    assert got == R.routes_of(c.want)


@pytest.mark.parametrize("tag", RI)
def test_random_insertion_equals_reference(tag):
    c = R.RepairCase(tag)
    sol = c.sol.clone()
    out = repair_insert(sol, list(c.unrouted), InsertionOperator.RI, c.inst, c.consts, c.penalties(),
                        random.Random(c.seed))
    assert out is sol and R.routes_of(sol) == R.routes_of(c.want)


# ------------------------------------------------------------------ GPU ----

@pytest.mark.gpu
@pytest.mark.parametrize("tag", DET)
def test_device_repair_equals_reference(tag):
    c = R.RepairCase(tag)
    sol = c.sol.clone()
    out = repair_insert(sol, list(c.unrouted), InsertionOperator[c.op], c.inst, c.consts, c.penalties(),
                        random.Random(c.seed))
    assert out is sol
    assert R.routes_of(sol) == R.routes_of(c.want)


def _partial(rng, sol, frac, drop_empty):
    s = sol.clone()
    cust = [x for r in s.routes for x in r.customers]
    removed = set(rng.sample(cust, max(1, int(len(cust) * frac))))
    for r in s.routes:
        r.customers = [x for x in r.customers if x not in removed]
    if drop_empty:
        s.drop_empty_routes()
    order = sorted(removed)
    rng.shuffle(order)
    return s, order


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["FBI", "IBI", "FRI", "IRI"])
@pytest.mark.parametrize("name", ["C2", "C3"])
def test_device_repair_population_matches_oracle(name, op):
    """16 offspring of an Appendix A start (25-40% removed), repaired together."""
    spec = W.CONFIGS[name]
    inst, _ = W.appendix_a_instance(spec)
    consts = ScalingConstants.from_instance(inst)
    rng = random.Random(zlib.crc32(f"{name}{op}".encode()))
    from paper_2605_05208_b200.genetic import initial_solutions
    base = initial_solutions(inst, consts, PenaltyState(), [random.Random(100 + i) for i in range(4)])
    sols, pend, pens = [], [], []
    for i in range(16):
        s, u = _partial(rng, base[i % 4], rng.choice([0.25, 0.4]), i % 2 == 0)
        sols.append(s)
        pend.append(u)
        pens.append(PenaltyState(lam=[rng.choice([0.5, 1.0, 10.0]) for _ in range(4)]))
    oi = _oi(inst, consts)
    want = [O.repair(oi, s, u, O.REPAIR_OPS[op], p.lam)[0] for s, u, p in zip(sols, pend, pens)]
    work = [s.clone() for s in sols]
    stats = repair_population(work, pend, InsertionOperator[op], inst, consts, pens)
    for b in range(16):
        assert R.routes_of(work[b]) == want[b], b
        assert stats[b]["inserted"] == len(pend[b])
        assert 0 < stats[b]["slot_evals"] <= stats[b]["ref_slot_evals"]


@pytest.mark.gpu
def test_device_repair_grows_route_capacity():
    """IBI with one vehicle per depot: every customer lands in one long route
    (beyond the initial K_cap) -- the capacity retry must reproduce the oracle."""
    rng = random.Random(9)
    depots = [(50.0, 50.0)]
    cust = [(rng.uniform(0, 100), rng.uniform(0, 100), 1, 0.0) for _ in range(70)]
    inst = Instance.from_coords("mdvrp", depots, cust, fleet_per_depot=1, capacity=INF)
    consts = ScalingConstants.from_instance(inst)
    sol = Solution([Route(0, 0, [1, 2])])
    pend = list(range(3, 71))
    want, _ = O.repair(_oi(inst, consts), sol, pend, 1, [1.0] * 4)
    out = repair_insert(sol, pend, InsertionOperator.IBI, inst, consts, PenaltyState(), random.Random(0))
    assert R.routes_of(out) == want and len(out.routes[0].customers) == 70


@pytest.mark.gpu
def test_device_repair_errors_and_noop():
    c = R.RepairCase(DET[0])
    routed = c.sol.routes[0].customers[0] if c.sol.routes and c.sol.routes[0].customers else None
    if routed is not None:
        with pytest.raises(ValueError):
            repair_insert(c.sol.clone(), [routed], InsertionOperator.FBI, c.inst, c.consts, c.penalties(), None)
    with pytest.raises(ValueError):
        repair_population([c.sol.clone()], [[c.unrouted[0], c.unrouted[0]]], InsertionOperator.IBI, c.inst,
                          c.consts, c.penalties())
    s = c.sol.clone()
    assert R.routes_of(repair_insert(s, [], InsertionOperator.FRI, c.inst, c.consts, c.penalties(), None)) == \
        R.routes_of(c.sol)


RFUZZ = list(range(int(os.environ.get("MDR_FUZZ_N", "32"))))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", RFUZZ)
def test_fuzz_device_repair_vs_oracle(seed):
    """Random shapes and partial solutions: every operator, a batch of 1-8
    individuals with different pending sets and lambdas, vs the oracle."""
    r = random.Random(5000 + seed)
    variant = r.choice(["mdvrp", "mdvrptw", "mdovrp"])
    inst = W.make_instance(r, variant, n_customers=r.randint(2, 90), n_depots=r.randint(1, 5),
                           capacity=r.choice([None, 10, 30, 500]), fleet=r.choice([None, 1, 2, 5]),
                           max_duration=r.choice([None, 300.0]) if variant != "mdovrp" else None)
    consts = ScalingConstants.from_instance(inst)
    oi = _oi(inst, consts)
    op = r.choice(["FBI", "IBI", "FRI", "IRI"])
    sols, pend, pens = [], [], []
    for i in range(r.randint(1, 8)):
        s, u = _partial(r, W.random_solution(random.Random(seed * 10 + i), inst), r.choice([0.05, 0.3, 0.7, 1.0]),
                        r.random() < 0.5)
        if r.random() < 0.15:
            s.routes = []  # everything unrouted
            u = list(inst.customers())
        sols.append(s)
        pend.append(u)
        pens.append(PenaltyState(lam=[r.choice([0.01, 1.0, 50.0]) for _ in range(4)]))
    want = [O.repair(oi, s, u, O.REPAIR_OPS[op], p.lam)[0] for s, u, p in zip(sols, pend, pens)]
    work = [s.clone() for s in sols]
    repair_population(work, pend, InsertionOperator[op], inst, consts, pens)
    for b in range(len(sols)):
        assert R.routes_of(work[b]) == want[b], (seed, b)
