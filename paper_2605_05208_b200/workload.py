"""Synthetic workloads: the instance/solution generators the benchmark and the
parity tests use.

* `make_instance` / `random_solution` restate the reference test fixtures
  (pkg/tests/conftest.py:9-53), so seeded states equal the reference's.
* `appendix_a_instance` restates the SURVEY.md Appendix A generator behind the
  BASELINE.json configs C1-C5.
* `initial_solution` restates genetic.initial_solution (genetic.py:251-294)
  with its relaxed best-insertion repair (genetic.py:71-244, IBI branch): it
  produces the benchmark's starting states, not part of the hot path.
"""
from __future__ import annotations

import random
from dataclasses import dataclass

from .evaluation import PenaltyState, ScalingConstants, concat, single_attr
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
    sols = [initial_solution(inst, consts, PenaltyState(), random.Random(start_seed + i))
            for i in range(pop)]
    return spec, inst, consts, nbr, sols


# --------------------------------------------------------------------------- #
# initial_solution (genetic.py:251-294) and its IBI repair (genetic.py:71-244)
# --------------------------------------------------------------------------- #
_single = single_attr  # scalar algebra with Python max/min semantics (evaluation.py:60-94)
_concat = concat


class _RouteEval:
    def __init__(self, route, inst):
        self.route = route
        self.rebuild(inst)

    def rebuild(self, inst):
        seq = self.route.sequence(inst.open_routes)
        n = len(seq)
        pref = [_single(seq[0], inst)]
        for v in seq[1:]:
            pref.append(_concat(pref[-1], _single(v, inst), inst))
        suf = [None] * n
        suf[n - 1] = _single(seq[n - 1], inst)
        for i in range(n - 2, -1, -1):
            suf[i] = _concat(_single(seq[i], inst), suf[i + 1], inst)
        self.pref, self.suf, self.n = pref, suf, n

    def candidate_attr(self, pos, node, inst):
        mid = _concat(self.pref[pos], _single(node, inst), inst)
        return _concat(mid, self.suf[pos + 1], inst) if pos + 1 < self.n else mid


def _cost_terms(a, inst, consts):
    v1 = consts.gamma * a.TW if inst.has_windows else 0.0
    v2 = consts.theta * max(a.load - inst.capacity, 0.0) / inst.capacity
    v3 = 0.0
    if inst.max_duration != INF:
        v3 = consts.theta * max(a.T - inst.max_duration, 0.0) / inst.max_duration
    return a.dist, v1, v2, v3


def _feasible(a, inst):
    if a.load > inst.capacity + 1e-9:
        return False
    if inst.max_duration != INF and a.T > inst.max_duration + 1e-9:
        return False
    if inst.has_windows and a.TW > 1e-9:
        return False
    return True


def _repair_ibi(sol, unrouted, inst, consts, penalties):
    pending = sorted(unrouted)
    evals = [_RouteEval(r, inst) for r in sol.routes]
    lam = penalties.lam

    def open_route(node):
        counts = [0] * inst.n_depots
        for r in sol.routes:
            if r.customers:
                counts[r.depart] += 1
        best, best_key = None, None
        for d in range(inst.n_depots):
            cost = inst.dist[d, node] + (0.0 if inst.open_routes else inst.dist[node, d])
            free = inst.fleet_per_depot == INF or counts[d] < inst.fleet_per_depot
            key = (not free, cost, d)
            if best_key is None or key < best_key:
                best, best_key = d, key
        r = Route(best, best, [node])
        sol.routes.append(r)
        evals.append(_RouteEval(r, inst))

    if not sol.routes and pending:
        open_route(pending.pop(0))
    while pending:
        chosen_node, chosen_slot, best_cost = None, None, INF
        for node in pending:
            slot, c1 = None, INF
            for ri, ev in enumerate(evals):
                d0, v10, v20, v30 = _cost_terms(ev.pref[ev.n - 1], inst, consts)
                for pos in range(len(sol.routes[ri].customers) + 1):
                    a = ev.candidate_attr(pos, node, inst)
                    d1, v11, v21, v31 = _cost_terms(a, inst, consts)
                    df = (d1 - d0) + lam[0] * (v11 - v10) + lam[1] * (v21 - v20) + lam[2] * (v31 - v30)
                    if df < c1:
                        slot, c1 = (ri, pos), df
            if slot is not None and c1 < best_cost:
                best_cost, chosen_node, chosen_slot = c1, node, slot
        if chosen_node is None:
            chosen_node, chosen_slot = pending[0], None
        pending.remove(chosen_node)
        if chosen_slot is None:
            open_route(chosen_node)
        else:
            ri, pos = chosen_slot
            sol.routes[ri].customers.insert(pos, chosen_node)
            evals[ri].rebuild(inst)
    return sol


def initial_solution(inst, consts, penalties, rng) -> Solution:
    by_depot = {d: [] for d in inst.depots()}
    for cst in inst.customers():
        d = min(inst.depots(), key=lambda dd: (inst.dist[dd, cst], dd))
        by_depot[d].append(cst)
    sol = Solution()
    leftovers = []
    for d, members in by_depot.items():
        rng.shuffle(members)
        routes, evals = [], []
        for cst in members:
            best, best_cost = None, INF
            for ri, ev in enumerate(evals):
                base = ev.pref[ev.n - 1].dist
                for pos in range(len(routes[ri].customers) + 1):
                    a = ev.candidate_attr(pos, cst, inst)
                    if not _feasible(a, inst):
                        continue
                    cost = a.dist - base
                    if cost < best_cost:
                        best, best_cost = (ri, pos), cost
            if best is not None:
                ri, pos = best
                routes[ri].customers.insert(pos, cst)
                evals[ri].rebuild(inst)
            elif inst.fleet_per_depot == INF or len(routes) < inst.fleet_per_depot:
                r = Route(d, d, [cst])
                routes.append(r)
                evals.append(_RouteEval(r, inst))
            else:
                leftovers.append(cst)
        sol.routes.extend(routes)
    if leftovers:
        _repair_ibi(sol, leftovers, inst, consts, penalties)
    sol.drop_empty_routes()
    return sol
