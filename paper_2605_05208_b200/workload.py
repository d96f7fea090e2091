"""Synthetic workloads: the instance/solution generators the benchmark and the
parity tests use.

* `make_instance` / `random_solution` restate the reference test fixtures
  (pkg/tests/conftest.py:9-53), so seeded states equal the reference's.
* `appendix_a_instance` restates the SURVEY.md Appendix A generator behind the
  BASELINE.json configs C1-C5.
* `build_config` gives a config's start states through the device
  construction (genetic.initial_solutions: mdr_construct + mdr_repair IBI).
"""
from __future__ import annotations

import random
from dataclasses import dataclass

from .evaluation import PenaltyState, ScalingConstants
from .model import INF, Instance, Route, Solution, Variant
from .neighborhood import NeighborConfig, build


# --------------------------------------------------------------------------- #
# reference test fixtures (conftest.py:9-53)
# --------------------------------------------------------------------------- #
def make_instance(rng: random.Random, variant=Variant.MDVRP, n_customers=8, n_depots=2,
                  capacity=None, max_duration=None, fleet=None) -> Instance:
    variant = Variant(variant)
    depot_xy = [(rng.uniform(0, 100), rng.uniform(0, 100)) for _ in range(n_depots)]
    windows = variant is Variant.MDVRPTW
    customers = []
    for _ in range(n_customers):
        x, y = rng.uniform(0, 100), rng.uniform(0, 100)
        q = rng.randint(1, 10)
        if windows:
            s = rng.uniform(5, 15)
            e = rng.uniform(0, 600)
            customers.append((x, y, q, s, e, e + rng.uniform(80, 400)))
        else:
            customers.append((x, y, q, 0.0))
    if capacity is None:
        capacity = max(12, 10 * n_customers // (2 * n_depots))
    return Instance.from_coords(
        variant, depot_xy, customers,
        fleet_per_depot=INF if fleet is None else fleet, capacity=capacity,
        max_duration=INF if max_duration is None else max_duration,
        depot_windows=[(0.0, 1200.0)] * n_depots if windows else None)


def random_solution(rng: random.Random, inst, scramble_depots=True) -> Solution:
    cust = list(inst.customers())
    rng.shuffle(cust)
    routes = []
    i = 0
    while i < len(cust):
        size = rng.randint(1, min(5, len(cust) - i))
        chunk = cust[i:i + size]
        i += size
        depart = rng.randrange(inst.n_depots)
        if scramble_depots and not inst.open_routes and rng.random() < 0.3:
            arrive = rng.randrange(inst.n_depots)
        else:
            arrive = depart
        routes.append(Route(depart, arrive, chunk))
    return Solution(routes)


# --------------------------------------------------------------------------- #
# BASELINE.json configurations
# --------------------------------------------------------------------------- #
@dataclass(frozen=True)
class ConfigSpec:
    name: str
    variant: Variant
    n_customers: int
    n_depots: int
    fleet: float
    capacity: float
    max_duration: float
    theta: int
    population: int


CONFIGS = {
    "C1": ConfigSpec("C1", Variant.MDVRP, 50, 4, 4, 80, INF, 50, 1),
    "C2": ConfigSpec("C2", Variant.MDVRPTW, 288, 6, 12, 200, 450, 50, 64),
    "C3": ConfigSpec("C3", Variant.MDOVRP, 360, 9, INF, 200, INF, 50, 128),
    "C4": ConfigSpec("C4", Variant.MDVRPTW, 1000, 10, 30, 200, 450, 50, 256),
    "C5": ConfigSpec("C5", Variant.MDVRP, 4000, 20, INF, 200, INF, 40, 512),
}


def appendix_a_instance(spec: ConfigSpec, seed: int = 2026):
    """Returns (instance, rng) -- the rng continues the seed stream (Appendix A)."""
    rng = random.Random(seed)
    windows = spec.variant is Variant.MDVRPTW
    depots = [(rng.uniform(0, 100), rng.uniform(0, 100)) for _ in range(spec.n_depots)]
    customers = []
    for _ in range(spec.n_customers):
        x = rng.uniform(0, 100)
        y = rng.uniform(0, 100)
        q = rng.randint(1, 25)
        if windows:
            s = rng.uniform(1, 20)
            e = rng.uniform(0, 700)
            customers.append((x, y, q, s, e, e + rng.uniform(30, 200)))
        else:
            customers.append((x, y, q, rng.choice([0.0, 10.0])))
    inst = Instance.from_coords(spec.variant, depots, customers, fleet_per_depot=spec.fleet,
                                capacity=spec.capacity, max_duration=spec.max_duration,
                                depot_windows=[(0.0, 1000.0)] * spec.n_depots if windows else None,
                                name=spec.name)
    return inst, rng


def build_config(name: str, population: int | None = None, seed: int = 2026, start_seed: int = 100):
    """Instance, constants, neighbour lists and the BASELINE.md start states:
    individual i starts from initial_solution(..., random.Random(start_seed+i))."""
    spec = CONFIGS[name]
    inst, _ = appendix_a_instance(spec, seed)
    consts = ScalingConstants.from_instance(inst)
    nbr = build(inst, NeighborConfig(spec.theta), consts)
    pop = spec.population if population is None else population
    from .genetic import initial_solutions
    sols = initial_solutions(inst, consts, PenaltyState(), [random.Random(start_seed + i) for i in range(pop)])
    return spec, inst, consts, nbr, sols
