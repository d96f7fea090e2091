"""Scalar restatement of the reference's initial construction -- TEST
INFRASTRUCTURE ONLY (the checker of the device construction, mdr_construct +
mdr_repair IBI; also the host source of start states for CPU-only tests and
the CPU reference arm when the reference package is not installed).

Follows genetic.initial_solution (genetic.py:251-294) with _RouteEval
(genetic.py:71-97), _attr_feasible (genetic.py:109-116) and the IBI branch of
repair_insert (genetic.py:174-244) of /root/reference/pkg/src/mdroute; pinned
to the reference's start states by tests/test_host_inputs.py and
tests/test_large_golden.py.
"""
from __future__ import annotations

from oracle.scalar_ref import concat, single_attr
from paper_2605_05208_b200.model import INF, Route, Solution

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
