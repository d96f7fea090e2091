"""Host restatement of the route exchange of DCREX -- TEST INFRASTRUCTURE ONLY
(the checker of the device exchange, csrc/mdr_exchange.cu; also the CPU
stand-in the engine's control-plane tests run with).

Follows genetic.py:308-446 of /root/reference/pkg/src/mdroute:
score_route_pair (the per-pair set algebra, here from exact integer incidence
counts), the donor loop with the five best (score, oi, dj) pairs and
rng.choice, and _remove_redundant.  Pinned to the reference through the
engine goldens (tests/golden/engine.json: identical RunStats).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from paper_2605_05208_b200.genetic import diversity_bounds
from paper_2605_05208_b200.model import route_edges, solution_edges


@dataclass
class RoutePairScore:
    new_edges: int
    missing: int
    duplicated: int
    conflicting: int
    score: int
    delta_sigma: int


def score_route_pair(route_out, route_in, main_edges: set, main_customers: set, introduced_customers: set,
                     inst) -> RoutePairScore:
    """Exchange `route_out` (leaves the offspring) for `route_in` (donor)."""
    cin, cout = set(route_in.customers), set(route_out.customers)
    new_edges = len(route_edges(route_in, inst.open_routes) - main_edges)
    missing = len(cout - cin)
    duplicated = len(cin & (main_customers - cout))
    conflicting = len(cin & introduced_customers)
    return RoutePairScore(new_edges, missing, duplicated, conflicting,
                          -(new_edges - missing - duplicated - 10 * conflicting), new_edges + missing + duplicated)


def _removal_saving(route, pos: int, inst) -> float:
    seq = route.sequence(inst.open_routes)
    i = pos + 1
    prev, here = seq[i - 1], seq[i]
    if i + 1 >= len(seq):
        return float(inst.dist[prev, here])
    nxt = seq[i + 1]
    return float(inst.dist[prev, here] + inst.dist[here, nxt] - inst.dist[prev, nxt])


def _remove_redundant(offspring, origin_main: list, inst) -> None:
    """One copy per duplicated customer: donor copies first, then the copy whose
    removal saves the least distance is kept (genetic.py:424-446)."""
    where: dict = {}
    for ri, r in enumerate(offspring.routes):
        for pos, c in enumerate(r.customers):
            where.setdefault(c, []).append((ri, pos))
    drop = []
    for occ in where.values():
        if len(occ) > 1:
            keep = min(occ, key=lambda it: (origin_main[it[0]], _removal_saving(offspring.routes[it[0]], it[1], inst)))
            drop.extend(o for o in occ if o != keep)
    for ri, pos in sorted(drop, key=lambda t: (t[0], -t[1])):
        del offspring.routes[ri].customers[pos]


def _pair_scores(off, origin_main, donor, used, main_edges, main_customers, introduced, inst, donor_cache):
    """Every admissible (offspring main-origin route oi, donor route dj) pair as
    (score, oi, dj, delta_sigma), in the order of score_route_pair's formula:
    new_edges(dj) = |E(dj) - E(main)|, missing = |C(oi)| - |C(oi) & C(dj)|,
    duplicated = |C(dj) & MC| - |C(dj) & C(oi)| (C(oi) is part of MC),
    conflicting = |C(dj) & introduced| -- exact integers from one incidence
    product instead of per-pair set algebra."""
    import numpy as np
    outs = [oi for oi in range(len(off.routes)) if origin_main[oi]]
    ins = [dj for dj, r in enumerate(donor.routes) if dj not in used and r.customers]
    if not outs or not ins:
        return None
    n = inst.n_nodes
    if "dc" not in donor_cache:  # per-donor flat customers / route ids and new-edge counts (main_edges is fixed)
        dc = [c for r in donor.routes for c in r.customers]
        donor_cache["dc"] = np.asarray(dc, np.int64)
        donor_cache["dr"] = np.asarray([j for j, r in enumerate(donor.routes) for _ in r.customers], np.int64)
        donor_cache["e"] = np.array([len(route_edges(r, inst.open_routes) - main_edges) for r in donor.routes],
                                    np.int64)
    dc, dr, nd = donor_cache["dc"], donor_cache["dr"], len(donor.routes)
    row_of = np.full(n, -1, np.int64)
    n_out = np.empty(len(outs), np.int64)
    for a, oi in enumerate(outs):
        cs = off.routes[oi].customers
        row_of[cs] = a
        n_out[a] = len(cs)
    col_of = np.full(nd, -1, np.int64)
    col_of[ins] = np.arange(len(ins))
    rows, cols = row_of[dc], col_of[dr]
    ok = (rows >= 0) & (cols >= 0)
    inter = np.bincount(rows[ok] * len(ins) + cols[ok], minlength=len(outs) * len(ins)).reshape(len(outs), len(ins))
    mc = np.zeros(n, np.int64)
    mc[list(main_customers)] = 1
    intro = np.zeros(n, np.int64)
    if introduced:
        intro[list(introduced)] = 1
    in_mc = np.bincount(dr, weights=mc[dc], minlength=nd).astype(np.int64)[ins][None, :]
    n_c = np.bincount(dr, weights=intro[dc], minlength=nd).astype(np.int64)[ins][None, :]
    e = donor_cache["e"][ins][None, :]
    missing = n_out[:, None] - inter
    dup = in_mc - inter
    score = -(e - missing - dup - 10 * n_c)
    dsig = e + missing + dup
    oi_a = np.broadcast_to(np.asarray(outs)[:, None], inter.shape)
    dj_a = np.broadcast_to(np.asarray(ins)[None, :], inter.shape)
    return score.ravel(), oi_a.ravel(), dj_a.ravel(), dsig.ravel()


def route_exchange(population: Sequence, inst, diversity_bandit, rng,
                   main_index: Optional[int] = None):
    """The exchange half of DCREX (genetic.py:343-405): returns (offspring with
    duplicates removed, unrouted customers, level, sigma, main_index)."""
    import numpy as np
    if len(population) < 2:
        raise ValueError("crossover needs at least two parents")
    if main_index is None:
        main_index = rng.randrange(len(population))
    main = population[main_index]
    level = diversity_bandit.select()
    sigma_min, sigma_max = diversity_bounds(level, inst, main)
    off = main.clone()
    origin_main = [True] * len(off.routes)
    main_edges = solution_edges(main, inst.open_routes)
    main_customers = set()
    for r in off.routes:
        main_customers.update(r.customers)
    introduced: set = set()
    donors = [p for i, p in enumerate(population) if i != main_index]
    rng.shuffle(donors)
    sigma = 0.0
    for donor in donors:
        used: set = set()
        cache: dict = {}
        reached = False
        while True:
            ps = _pair_scores(off, origin_main, donor, used, main_edges, main_customers, introduced, inst, cache)
            if ps is None:
                break
            score, oi_a, dj_a, dsig = ps
            # pairs.sort(key=(score, oi, dj))[:5] via one exact int64 key and a partial sort
            nd = len(donor.routes)
            key = (score - score.min()) * ((len(off.routes) + 1) * nd) + oi_a * nd + dj_a
            if key.size > 5:
                part = np.argpartition(key, 4)[:5]
                top = part[np.argsort(key[part])]
            else:
                top = np.argsort(key)
            k = top[rng.choice(range(len(top)))]         # rng.choice over the first five
            oi, dj, ds = int(oi_a[k]), int(dj_a[k]), int(dsig[k])
            if sigma + ds >= sigma_max:
                break
            main_customers.difference_update(off.routes[oi].customers)
            del off.routes[oi]
            del origin_main[oi]
            r_new = donor.routes[dj].clone()
            off.routes.append(r_new)
            origin_main.append(False)
            introduced.update(r_new.customers)
            used.add(dj)
            sigma += ds
            if sigma >= sigma_min:
                reached = True
                break
        if reached:
            break
    _remove_redundant(off, origin_main, inst)
    covered = set(off.customer_list())
    unrouted = [c for c in inst.customers() if c not in covered]
    return off, unrouted, level, sigma, main_index


