"""Best-improvement multi-move local search on the GPU (mirrors `mdroute.localsearch`).

`local_search` keeps the reference signature (localsearch.py:97-140) and runs
the whole descent on the device: per round every active individual evaluates
one operator of its pre-drawn permutation stream (the exact `rng.shuffle`
results, drawn from a clone of the caller's rng), the leader and its
route-disjoint followers are selected and applied on the device, the tables
are rebuilt and the penalty coefficients adapted -- with no host round trip.

`local_search_population` is the B200 addition: B independent descents
(e.g. a GA generation's offspring) advance together in the same kernels.
Each individual's trajectory is bit-identical to a separate reference call.
"""
from __future__ import annotations

import array
import ctypes as C
import gc
import time
import weakref
from dataclasses import dataclass
from typing import Optional

import numpy as np

from ._lib import CapacityError
from .batch import SolutionCache, evaluate_candidates, leader_and_followers
from .device import Population
from .evaluation import RouteAttr
from .moves import ALL_OPS, Move, Op, move_plan
from .session import same_consts, session_for

VIOLATION_TOL = 1e-9


@dataclass
class SearchConfig:
    depth: int = 500
    multi_move: bool = False

    def __post_init__(self):
        if self.depth < 1:
            raise ValueError("depth must be >= 1")


def enabled_operators(inst) -> list:
    ops = list(ALL_OPS)
    if inst.has_windows:
        ops.remove(Op.TWO_OPT)
    return ops


def evaluate_batch(sol, cands, penalties, consts, inst, cache=None, multi_move: bool = True):
    if cache is None:
        cache = SolutionCache(sol, inst, consts)
    deltas = evaluate_candidates(cache, cands, penalties)
    return leader_and_followers(cache, cands, deltas, multi_move)


def select_moves(leader, followers) -> list:
    """Greedy route-disjoint selection (localsearch.py:45-55)."""
    chosen = [leader]
    used = leader.routes_touched()
    for mv in followers:
        t = mv.routes_touched()
        if used & t:
            continue
        chosen.append(mv)
        used |= t
    return chosen


_STALE = object()  # attr of a route a replayed step rewrote: refreshed from the device at the end


def apply_moves(sol, moves, inst, _stale=None) -> None:
    """Host twin of the device apply (localsearch.py:58-82); rewritten routes'
    attr caches are reset (the device refreshes them after a descent)."""
    used: set = set()
    for mv in moves:
        t = mv.routes_touched()
        if used & t:
            raise ValueError("conflicting moves: route sets intersect")
        used |= t
    plans = [move_plan(sol, mv, inst) for mv in moves]
    from .genetic import _route_cls
    route_cls = _route_cls(sol)
    new_routes = []
    for ps in plans:
        for p in ps:
            if p.route_index is None:
                nr = route_cls(p.depart, p.arrive, p.customers)
                if hasattr(nr, "attr"):
                    nr.attr = _stale
                new_routes.append(nr)
            else:
                r = sol.routes[p.route_index]
                r.depart, r.arrive, r.customers = p.depart, p.arrive, p.customers
                if hasattr(r, "attr"):
                    r.attr = _stale
    sol.routes.extend(nr for nr in new_routes if nr.customers)
    sol.drop_empty_routes()


def _mt_state(rng):
    if not (hasattr(rng, "getstate") and hasattr(rng, "setstate")):
        raise TypeError("rng must be a random.Random (getstate/setstate) so the operator stream can be pre-drawn")
    st = rng.getstate()
    if not (isinstance(st, tuple) and len(st) == 3 and len(st[1]) == 625):
        raise TypeError("rng state is not a MT19937 random.Random state")
    return st, np.frombuffer(array.array("I", st[1]), dtype=np.uint32)  # 3x faster than np.asarray(tuple)


def draw_permutations(rng, ops, n_passes: int, start: Optional[list] = None) -> np.ndarray:
    """The first n_passes `rng.shuffle(list(ops))` results (rng not advanced):
    CPython's shuffle on the MT19937 state, run natively (mdr_shuffle_stream).
    start: if given, receives (state, MT words) of rng before the draw, for _advance."""
    from . import _lib
    st, mt = _mt_state(rng)
    if start is not None:
        start.append((st, mt.copy()))
    items = np.ascontiguousarray([int(o) for o in ops], dtype=np.uint8)
    out = np.empty((n_passes, len(ops)), np.uint8)
    _lib.check(_lib.lib().mdr_shuffle_stream(_lib.ptr(mt, C.POINTER(C.c_uint32)), len(items),
                                             _lib.ptr(items, _lib.u8p), n_passes, _lib.ptr(out, _lib.u8p)),
               "mdr_shuffle_stream")
    return out


def _advance(rng, ops, passes: int, start=None) -> None:
    """Advance rng exactly as `passes` calls of rng.shuffle(list(ops)) would
    (from start = draw_permutations' saved state when given: rng itself has
    not been used since)."""
    from . import _lib
    st, mt = start if start is not None else _mt_state(rng)
    items = np.ascontiguousarray([int(o) for o in ops], dtype=np.uint8)
    _lib.check(_lib.lib().mdr_shuffle_stream(_lib.ptr(mt, C.POINTER(C.c_uint32)), len(items),
                                             _lib.ptr(items, _lib.u8p), passes, None), "mdr_shuffle_stream")
    rng.setstate((st[0], tuple(array.array("I", mt.tobytes())), st[2]))


class DeviceSearch:
    """Reusable device population for repeated batched descents."""

    def __init__(self, inst, consts, nbr, device: int = 0):
        self.session = session_for(inst, consts, nbr, device)
        self.pop: Optional[Population] = None
        self.last_stats = None

    @property
    def inst(self):
        return self.session.inst

    def _ensure(self, sols, need=None):
        J, K = Population.caps_for(sols, self.inst)
        F = 1 << 15
        if need:  # grow what the failed attempt reported (at least doubling it); never shrink
            p = self.pop
            J = max(J, p.J_cap, 2 * p.J_cap if need["J"] else J, need["J"] + 64)
            K = max(K, p.K_cap, need["K"])
            F = max(F, p.F_cap * 2 if (need["F"] or need["G"]) else p.F_cap, need["F"] + 1024,
                    (need["G"] + 1024) // max(len(sols), 1))
        J, K = min(4094, J), min(500, K)
        p = self.pop
        if p is None or p.B_cap < len(sols) or p.J_cap < J or p.K_cap < K or p.F_cap < F:
            self.pop = None
            p = self.pop = Population(self.session.dinst, max(len(sols), p.B_cap if p else 0), J, K, F)
        return p

    def run(self, sols, lams, perms, cfg: SearchConfig, kappa=0.5, lam_min=0.01, lam_max=1e4,
            deadline_s: float = -1.0, snapshot_best: bool = False, trace: bool = False):
        """Descents of all `sols` (not modified). Returns (routes, lams, stats)."""
        need = None
        for attempt in range(8):
            pop = self._ensure(sols, need)
            pop.upload(sols, lams)
            try:
                stats = pop.local_search(perms, cfg.depth, cfg.multi_move, kappa, lam_min, lam_max, deadline_s,
                                         snapshot_best=snapshot_best, trace=trace)
                break
            except CapacityError as e:
                need = getattr(e, "need", None) or dict(F=1, G=0, J=0, K=0)
                if attempt == 7:
                    raise
        routes, lam_out = pop.download()
        self.last_stats = stats
        return routes, lam_out, stats


def _apply_result(sol, routes, attrs=None, open_routes: bool = False):
    """Write a descent's final routes into `sol` in place (localsearch.py:58-82): route
    objects are reused by index, changed routes get their route_attr refreshed (from
    the device fold when `attrs` [J, 6] is given, else reset), new routes are appended
    and the list is cut to the new route count (the device already dropped empties)."""
    from .genetic import _route_cls
    cls = _route_cls(sol)
    old = sol.routes
    rows = attrs[:len(routes)].tolist() if attrs is not None else None
    def attr_of(i, d, a, c):  # built only for the routes that take it
        return RouteAttr(*rows[i], d, c[-1] if open_routes else a) if rows is not None and c else None

    for i, (d, a, c) in enumerate(routes):
        if i < len(old):
            r = old[i]
            if r.depart != d or r.arrive != a or r.customers != c:
                r.depart, r.arrive, r.customers = d, a, c
                if hasattr(r, "attr"):
                    r.attr = attr_of(i, d, a, c)
            elif getattr(r, "attr", None) is _STALE:
                r.attr = attr_of(i, d, a, c)
        else:
            r = cls(d, a, list(c))
            if hasattr(r, "attr"):
                r.attr = attr_of(i, d, a, c)
            old.append(r)
    del old[len(routes):]


def _move_of(op: int, key: int) -> Move:
    """Inverse of the device's 58-bit packing of Move.key() (csrc/mdr_device.cuh pack_key)."""
    f = lambda sh, m: (key >> sh) & m  # noqa: E731
    return Move(Op(op), f(46, 0xfff) - 1, f(25, 0x1ff) - 1, f(34, 0xfff) - 1, f(16, 0x1ff) - 1, f(14, 3), f(12, 3),
                bool(f(11, 1)), bool(f(10, 1)), f(2, 0xff) - 1, f(0, 3) - 1)


def _replay(sol, steps, inst, on_feasible) -> None:
    """Re-apply a traced descent on the host (apply_moves per accepted step) and
    call on_feasible(D, sol) on every feasible post-step state, in order
    (localsearch.py:126-134); D is the device's totals()[0] of that state."""
    for op, feasible, D, keys in steps:
        apply_moves(sol, [_move_of(op, k) for k in keys], inst, _STALE)
        if feasible:
            on_feasible(D, sol)


_SEARCHERS: dict = {}


def _searcher(inst, consts, nbr, device: int = 0) -> DeviceSearch:
    """The reusable device search of (instance, device).  Other lists or other
    scaling constants (baked into the device instance) replace the entry and
    free the old device population."""
    key = (id(inst), device)
    s = _SEARCHERS.get(key)
    if (s is None or s.inst is not inst or s.session.nbr is not nbr
            or (consts is not None and not same_consts(consts, s.session.consts))):
        _SEARCHERS.pop(key, None)
        s = _SEARCHERS[key] = DeviceSearch(inst, consts, nbr, device)
        try:  # the entry (and its device population) goes with the instance
            weakref.finalize(inst, _SEARCHERS.pop, key, None)
        except TypeError:
            pass
    return s


def _finish(search, sols, penalties, rngs, routes, lam, stats, inst, ops, on_feasible, best_only: bool,
            starts=None):
    """Hand a device descent back to the caller's objects: rng advanced by the
    passes used, penalties updated, routes mutated in place with route_attr
    refreshed from the device, and on_feasible called -- per feasible post-step
    state by replaying the traced steps (localsearch.py:126-134), or, with
    best_only, once with the lowest-D feasible state (first reached on ties)."""
    pop = search.pop
    attrs = pop.route_attrs(0, len(sols))
    best = pop.download_best() if (on_feasible is not None and best_only) else None
    for b, (sol, pen, rng) in enumerate(zip(sols, penalties, rngs)):
        _advance(rng, ops, stats[b]["passes"], None if starts is None else starts[b])
        pen.lam[:] = [float(x) for x in lam[b]]
        if on_feasible is not None and not best_only:
            _replay(sol, pop.trace(b), inst, on_feasible)
            got = [(r.depart, r.arrive, list(r.customers)) for r in sol.routes]
            if got != [(d, a, list(c)) for d, a, c in routes[b]]:
                raise RuntimeError("host replay of the traced descent diverged from the device result")
        _apply_result(sol, routes[b], attrs[b], inst.open_routes)
        if best is not None and stats[b]["n_feasible"] > 0:
            snap = sol.clone()
            _apply_result(snap, best[0][b])
            on_feasible(float(best[1][b]), snap)


def local_search(sol, penalties, cfg: SearchConfig, nbr, consts, inst, rng, deadline: Optional[float] = None,
                 on_feasible=None, feasible_best_only: bool = False):
    """Reference-compatible descent of one solution (in place), run on the GPU
    (localsearch.py:97-140): `sol`'s routes are mutated in place with their
    attr caches refreshed, `penalties.lam` adapted, `rng` advanced by one shuffle
    per pass, and on_feasible(D, sol) called on every feasible post-step state
    (the device records the accepted steps; the host replays them only when a
    callback is given).  feasible_best_only=True calls it once, with the
    lowest-D feasible state -- all a best-tracking callback keeps -- without the
    replay."""
    local_search_population([sol], [penalties], cfg, nbr, consts, inst, [rng], deadline, on_feasible=on_feasible,
                            feasible_best_only=feasible_best_only)
    return sol


def local_search_population(sols, penalties, cfg: SearchConfig, nbr, consts, inst, rngs,
                            deadline: Optional[float] = None, device: int = 0, on_feasible=None,
                            feasible_best_only: bool = False):
    """B independent descents in one device run; each solution, penalty state
    and rng is updated in place exactly as a separate `local_search` call would
    do it (on_feasible(D, sol) per individual, in order).  Returns the
    per-individual stats."""
    if not (len(sols) == len(penalties) == len(rngs)):
        raise ValueError("sols, penalties and rngs must have the same length")
    if not sols:
        return []
    p0 = penalties[0]
    for p in penalties[1:]:  # one device launch carries one (kappa, lam_min, lam_max)
        if (p.kappa, p.lam_min, p.lam_max) != (p0.kappa, p0.lam_min, p0.lam_max):
            raise ValueError("local_search_population: all penalty states must share kappa, lam_min and lam_max")
    # the call creates ~100 small acyclic objects per individual: keep the cyclic collector
    # from pausing inside it (a gen-2 pass over a large heap costs up to ~1 s)
    gc_on = gc.isenabled()
    gc.disable()
    try:
        search = _searcher(inst, consts, nbr, device)
        ops = enabled_operators(inst)
        starts: list = []
        perms = np.stack([draw_permutations(r, ops, cfg.depth + 1, starts) for r in rngs])
        lams = [p.lam for p in penalties]
        dl = -1.0 if deadline is None else max(0.0, deadline - time.monotonic())
        replay = on_feasible is not None and not feasible_best_only
        routes, lam, stats = search.run(sols, lams, perms, cfg, p0.kappa, p0.lam_min, p0.lam_max, dl,
                                        snapshot_best=on_feasible is not None and feasible_best_only, trace=replay)
        _finish(search, sols, penalties, rngs, routes, lam, stats, inst, ops, on_feasible, feasible_best_only,
                starts)
    finally:
        if gc_on:
            gc.enable()
    return stats
