"""Repair insertion on the GPU (mirrors `mdroute.genetic.repair_insert`,
genetic.py:174-244).

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

from enum import IntEnum

from ._lib import CapacityError
from .device import Population
from .model import INF, Route
from .session import session_for


class InsertionOperator(IntEnum):
    FBI = 0  # feasible best insertion (new route as fallback)
    IBI = 1  # relaxed best insertion
    FRI = 2  # feasible regret insertion
    IRI = 3  # relaxed regret insertion
    RI = 4   # uniformly random insertion


def _route_cls(sol):
    return type(sol.routes[0]) if sol.routes else Route


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
            sess._repair_pop = None
            pop = sess._repair_pop = Population(sess.dinst, max(len(sols), 1), J, K, 1 << 10)
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
