"""Offspring construction: repair insertion on the GPU (mirrors
`mdroute.genetic.repair_insert`, genetic.py:174-244)
and the route-exchange crossover, bandits and population initialisation the
generation loop drives (genetic.py:25-66, 296-446; sec. 8(f) row 3).

`repair_insert` keeps the reference signature and semantics: `sol` is modified
in place (existing routes keep their order, new routes are appended), pending
customers are processed in ascending id order, FBI/IBI/FRI/IRI evaluate every
(pending customer x slot) under the scalar concat algebra and pick best or
regret insertions.  The evaluation runs in csrc/mdr_repair.cu (C-ABI
`mdr_repair`); RI only draws positions from the caller's rng and stays on the
host, like the reference's.

`repair_population` is the batched form: a GA generation's offspring are
repaired together (one CTA per individual) and can then be handed straight to
`local_search_population`.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

from ._lib import CapacityError
from .device import Population
from .model import INF, Route, Solution, route_edges, solution_edges
from .session import session_for

DIVERSITY_LEVELS = 20


class InsertionOperator(IntEnum):
    FBI = 0  # feasible best insertion (new route as fallback)
    IBI = 1  # relaxed best insertion
    FRI = 2  # feasible regret insertion
    IRI = 3  # relaxed regret insertion
    RI = 4   # uniformly random insertion


def _route_cls(sol):
    """The caller's Route class (the reference's when `sol` is a reference Solution)."""
    if sol.routes:
        return type(sol.routes[0])
    import sys
    return getattr(sys.modules.get(type(sol).__module__), "Route", Route)


def _open_route_host(sol, node, inst):
    """InsertState.open_route (genetic.py:148-166) for the RI operator."""
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
    sol.routes.append(_route_cls(sol)(best, best, [node]))


def _random_insert(sol, pending, inst, rng):
    """RI (genetic.py:200-208): the rng draws are the whole operator."""
    for node in pending:
        if not sol.routes:
            _open_route_host(sol, node, inst)
            continue
        ri = rng.randrange(len(sol.routes))
        pos = rng.randint(0, len(sol.routes[ri].customers))
        r = sol.routes[ri]
        r.customers.insert(pos, node)
        if hasattr(r, "attr"):
            r.attr = None


def _write_back(sol, routes):
    cls = _route_cls(sol)
    old = sol.routes
    for i, (d, a, c) in enumerate(routes):
        if i < len(old):
            r = old[i]
            r.depart, r.arrive, r.customers = d, a, list(c)
            if hasattr(r, "attr"):
                r.attr = None
        else:
            old.append(cls(d, a, list(c)))


def repair_population(sols, unrouteds, op, inst, consts, penalties, device: int = 0):
    """Repair every sols[b] with unrouteds[b] on the GPU (in place).  `penalties`
    is one PenaltyState per individual (or a single shared one).  Returns the
    per-individual stats (slot evaluations done / the reference's full re-scan count)."""
    op = InsertionOperator(op)
    if op == InsertionOperator.RI:
        raise ValueError("RI is rng-only; use repair_insert with an rng")
    if not isinstance(penalties, (list, tuple)):
        penalties = [penalties] * len(sols)
    sess = session_for(inst, consts, None, device)
    J, K = Population.caps_for(sols, inst)
    J = min(4094, J + max((len(u) for u in unrouteds), default=0))
    need = None
    for attempt in range(6):
        if need:
            J = min(4094, max(J * 2, need["J"] + 16))
            K = min(500, max(K * 2, need["K"] + 16))
        pop = getattr(sess, "_repair_pop", None)  # reused across calls while the caps fit
        if pop is None or pop.B_cap < len(sols) or pop.J_cap < J or pop.K_cap < K:
            if pop is not None:  # grow with headroom so a GA's varying offspring do not re-allocate
                J, K = min(4094, max(J, pop.J_cap * 3 // 2)), min(500, max(K, pop.K_cap * 3 // 2))
            sess._repair_pop = None
            pop = sess._repair_pop = Population(sess.dinst, max(len(sols), 1, pop.B_cap if pop else 0), J, K,
                                                1 << 10)
        pop.upload(sols, [p.lam for p in penalties])
        try:
            stats = pop.repair(int(op), unrouteds)
            break
        except CapacityError as e:
            need = getattr(e, "need", None) or dict(J=J, K=K)
            if attempt == 5 or (J >= 4094 and K >= 500):
                raise
    routes, _ = pop.download()
    for sol, rt in zip(sols, routes):
        _write_back(sol, rt)
    return stats


def repair_insert(sol, unrouted, op, inst, consts, penalties, rng):
    """Insert every unrouted customer using the selected insertion operator
    (genetic.py:193-244); returns `sol`, modified in place."""
    op = InsertionOperator(op)
    pending = sorted(unrouted)
    if not pending:
        return sol
    if op == InsertionOperator.RI:
        _random_insert(sol, pending, inst, rng)
        return sol
    repair_population([sol], [pending], op, inst, consts, [penalties])
    return sol


# --------------------------------------------------------------------------- #
# learning pieces (genetic.py:25-66)
# --------------------------------------------------------------------------- #

class DiscountedUCB1:
    """Discounted UCB1 over a fixed action set; unplayed actions first, in index order."""

    def __init__(self, n_actions: int, discount: float = 0.99):
        self.n_actions = n_actions
        self.discount = discount
        self.rewards = [0.0] * n_actions
        self.counts = [0.0] * n_actions

    def select(self) -> int:
        for i, c in enumerate(self.counts):
            if c == 0.0:
                return i
        total = sum(self.counts)
        best, best_val = 0, -INF
        for i in range(self.n_actions):
            val = self.rewards[i] / self.counts[i] + math.sqrt(2.0 * math.log(total) / self.counts[i])
            if val > best_val:
                best, best_val = i, val
        return best

    def update(self, action: int, reward: float) -> None:
        g = self.discount
        self.rewards = [x * g for x in self.rewards]
        self.counts = [x * g for x in self.counts]
        self.rewards[action] += reward
        self.counts[action] += 1.0


def improvement_reward(parent_value: float, offspring_value: float) -> float:
    """Percent improvement of the offspring over the main parent."""
    return 100.0 * (parent_value - offspring_value) / parent_value


def _construction_orders(inst, rngs):
    """The host half of initial_solution (genetic.py:255-266): nearest-depot
    membership (ties to the lower depot id) and each depot's rng.shuffle, drawn
    in the reference's order -- rngs[i] may repeat the same object, whose
    stream then continues across the individuals as a sequential caller's would."""
    nd = inst.n_depots
    near = np.argmin(np.asarray(inst.dist)[:nd, nd:], axis=0)  # first minimum = lowest id
    base = [[int(c) for c in np.nonzero(near == d)[0] + nd] for d in range(nd)]
    ooff, order = [0], []
    for rng in rngs:
        for d in range(nd):
            members = list(base[d])
            rng.shuffle(members)
            order.extend(members)
            ooff.append(len(order))
    return np.asarray(ooff, np.int32), np.asarray(order, np.int32)


def initial_solutions(inst, consts, penalties, rngs, device: int = 0) -> list:
    """genetic.initial_solution (genetic.py:251-294) for len(rngs) individuals at
    once: the shuffles on the host, the greedy per-depot construction
    (mdr_construct) and the relaxed best-insertion repair of the leftovers
    (mdr_repair, IBI) on the device, then drop_empty_routes."""
    B = len(rngs)
    if B == 0:
        return []
    ooff, order = _construction_orders(inst, rngs)
    nc, nd = inst.n_customers, inst.n_depots
    sess = session_for(inst, consts, None, device)
    demand = float(np.sum(np.asarray(inst.demand)[nd:]))
    est = nd + (int(math.ceil(demand / inst.capacity)) if inst.capacity != INF and inst.capacity > 0 else nd)
    J, K = min(4094, max(32, 2 * est)), min(500, max(32, 2 * -(-nc // max(est - nd, 1))))
    out = []
    at = 0
    while at < B:
        per_ind = J * (K + 2) * (K + 2) * (6 if inst.has_windows else 4) * 8 + J * (K + 2) * 200
        chunk = max(1, min(B - at, int(2e9 // per_ind)))
        pop = Population(sess.dinst, chunk, J, K, 1 << 10)
        try:
            left = pop.construct(ooff[at * nd: (at + chunk) * nd + 1] - ooff[at * nd],
                                 order[ooff[at * nd]: ooff[(at + chunk) * nd]], nc)
            if any(left):
                pop.repair(int(InsertionOperator.IBI), left)
        except CapacityError:
            if J >= 4094 and K >= 500:
                raise
            J, K = min(4094, 2 * J), min(500, 2 * K)
            continue
        routes, _ = pop.download()
        for rt in routes:
            sol = Solution([Route(d, a, list(c)) for d, a, c in rt])
            sol.drop_empty_routes()
            out.append(sol)
        at += chunk
    return out


def initial_solution(inst, consts, penalties, rng, device: int = 0) -> Solution:
    """Nearest-depot assignment, randomized greedy construction per depot, then
    relaxed insertion of whatever could not be placed feasibly (genetic.py:251-294)."""
    return initial_solutions(inst, consts, penalties, [rng], device)[0]


def initialize_population(inst, mu: int, consts, penalties, rng, device: int = 0) -> list:
    """mu initial solutions drawn from one rng stream (genetic.py:297-301), built in one batch."""
    if mu < 2:
        raise ValueError("population size must be >= 2")
    return initial_solutions(inst, consts, penalties, [rng] * mu, device)


# --------------------------------------------------------------------------- #
# route-exchange crossover (genetic.py:300-446)
# --------------------------------------------------------------------------- #

def diversity_bounds(level: int, inst, main_parent) -> tuple:
    base = inst.n_customers + len(main_parent.routes)
    return level / DIVERSITY_LEVELS * base, (level + 1) / DIVERSITY_LEVELS * base


@dataclass
class CrossoverResult:
    offspring: Solution
    diversity_level: int
    insertion_op: InsertionOperator
    sigma: float
    main_index: int = -1


def route_exchange(population: Sequence, inst, diversity_bandit: DiscountedUCB1, rng,
                   main_index: Optional[int] = None, device: int = 0):
    """The exchange half of DCREX (genetic.py:343-405) for one offspring, on the
    device: returns (offspring with duplicates removed, unrouted customers,
    level, sigma, main_index) and advances rng as the reference does."""
    return route_exchange_batch(population, inst, diversity_bandit, [rng], device,
                                None if main_index is None else [main_index])[0]


def route_exchange_batch(population: Sequence, inst, diversity_bandit: DiscountedUCB1, rngs, device: int = 0,
                         main_indices=None):
    """route_exchange for len(rngs) offspring of one generation at once: offspring j is
    what route_exchange(population, inst, diversity_bandit, rngs[j]) returns, and
    rngs[j] is advanced the same way.  The host draws each main parent and donor
    order (rng.randrange, rng.shuffle); the exchanges themselves -- pair scoring,
    the top-five choices on the continued MT19937 stream, redundancy removal --
    run on the device, one CTA per offspring (mdr_route_exchange)."""
    from . import _lib
    import ctypes as C
    M, B = len(population), len(rngs)
    if M < 2:
        raise ValueError("crossover needs at least two parents")
    if B == 0:
        return []
    level = diversity_bandit.select()  # no update inside a batch: one level for all
    mroute = np.zeros(M + 1, np.int32)
    routes = [r for sol in population for r in sol.routes]
    mroute[1:] = np.cumsum([len(sol.routes) for sol in population])
    coff = np.zeros(len(routes) + 1, np.int32)
    coff[1:] = np.cumsum([len(r.customers) for r in routes])
    cust = np.ascontiguousarray([c for r in routes for c in r.customers] or [0], np.int32)
    dep = np.ascontiguousarray([r.depart for r in routes] or [0], np.int32)
    arr = np.ascontiguousarray([r.arrive for r in routes] or [0], np.int32)
    mains = np.zeros(B, np.int32)
    donors = np.zeros((B, M - 1), np.int32)
    mt = np.zeros((B, 625), np.uint32)
    sig = np.zeros((B, 2), np.float64)
    for j, rng in enumerate(rngs):
        m = rng.randrange(M) if main_indices is None else int(main_indices[j])
        if not 0 <= m < M:
            raise ValueError("main index out of range")
        order = [i for i in range(M) if i != m]
        rng.shuffle(order)
        mains[j], donors[j] = m, order
        mt[j] = rng.getstate()[1]
        sig[j] = diversity_bounds(level, inst, population[m])
    J = max(len(s.routes) for s in population)
    Jcap = 2 * J + 8
    Ccap = 2 * inst.n_customers + 8
    refs = np.zeros((B, Jcap), np.int32)
    nref = np.zeros(B, np.int32)
    keep = np.zeros((B, Ccap), np.int32)
    unr = np.zeros((B, inst.n_customers), np.int32)
    nunr = np.zeros(B, np.int32)
    sigma = np.zeros(B, np.float64)
    sess = session_for(inst, None, None, device)
    P = _lib.ptr
    _lib.check(_lib.lib().mdr_route_exchange(
        sess.dinst.handle, M, P(mroute, _lib.i32p), P(coff, _lib.i32p), P(cust, _lib.i32p), P(dep, _lib.i32p),
        P(arr, _lib.i32p), B, P(mains, _lib.i32p), P(donors, _lib.i32p), P(mt, C.POINTER(C.c_uint32)),
        P(sig, _lib.f64p), Jcap, Ccap, P(refs, _lib.i32p), P(nref, _lib.i32p), P(keep, _lib.i32p),
        P(unr, _lib.i32p), P(nunr, _lib.i32p), P(sigma, _lib.f64p)), "mdr_route_exchange")
    out = []
    cl = cust.tolist()
    for j, rng in enumerate(rngs):
        st = rng.getstate()
        rng.setstate((st[0], tuple(int(x) for x in mt[j]), st[2]))
        cls = _route_cls(population[int(mains[j])])
        off_routes, at = [], 0
        for r in refs[j, :nref[j]].tolist():
            c0, c1 = int(coff[r]), int(coff[r + 1])
            kept = [cl[p] for p, k in zip(range(c0, c1), keep[j, at:at + c1 - c0]) if k]
            at += c1 - c0
            off_routes.append(cls(int(dep[r]), int(arr[r]), kept))
        off = type(population[int(mains[j])])(off_routes)
        off.meta = dict(getattr(population[int(mains[j])], "meta", {}))
        out.append((off, unr[j, :nunr[j]].tolist(), level, float(sigma[j]), int(mains[j])))
    return out


def dcrex(population: Sequence, inst, consts, penalties, diversity_bandit: DiscountedUCB1,
          insertion_bandit: DiscountedUCB1, rng, main_index: Optional[int] = None) -> CrossoverResult:
    """Diversity-controlled route exchange over multiple parents, then repair
    on the GPU (genetic.py:343-421)."""
    off, unrouted, level, sigma, main_index = route_exchange(population, inst, diversity_bandit, rng, main_index)
    op = InsertionOperator(insertion_bandit.select())
    repair_insert(off, unrouted, op, inst, consts, penalties, rng)
    off.drop_empty_routes()
    for r in off.routes:
        r.attr = None  # repaired routes: stale caches dropped (the descent refreshes them)
    return CrossoverResult(off, level, op, sigma, main_index)
