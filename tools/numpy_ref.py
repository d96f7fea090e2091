"""The UNMODIFIED reference package (mdroute, installed into baseline/_ref by
baseline/install_reference.sh) timed on the host cores: bench.py's numpy
reference leg (SURVEY.md 8(d) "CPU baseline").

Each worker process imports mdroute from baseline/_ref, rebuilds the same
instance (same nodes, same distance matrix), the same neighbour lists and the
same start state through the reference's own API, and runs
`mdroute.localsearch.local_search` (depth 500, multi-move, lambda 1, kappa 0.5,
rng Random(i)) under a wall-clock deadline.  Candidates are counted by
wrapping the name `mdroute.localsearch.enumerate_candidates` with a counter that
calls straight through (the reference's code path is unchanged).  Nothing here
touches this repo's library or kernels.
"""
from __future__ import annotations

import os
import random
import sys
import time

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def available() -> bool:
    return os.path.isfile(os.path.join(REF, "mdroute", "localsearch.py"))


def _worker(args):
    (variant, nodes, n_depots, dist, fleet, cap, dur, theta, routes, seed, depth, seconds) = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import mdroute.localsearch as LS
    from mdroute import evaluation as E, model as M, neighborhood as NB
    rnodes = [M.Node(*n) for n in nodes]
    inst = M.Instance(M.Variant(variant), rnodes, n_depots, dist, fleet_per_depot=fleet, capacity=cap,
                      max_duration=dur)
    consts = E.ScalingConstants.from_instance(inst)
    nbr = NB.build(inst, NB.NeighborConfig(theta), consts)
    sol = M.Solution([M.Route(d, a, list(c)) for d, a, c in routes])
    count = [0]
    real = LS.enumerate_candidates

    def counting(*a, **k):
        cs = real(*a, **k)
        count[0] += len(cs)
        return cs

    LS.enumerate_candidates = counting
    try:
        t0 = time.perf_counter()
        LS.local_search(sol, E.PenaltyState(), LS.SearchConfig(depth=depth, multi_move=True), nbr, consts, inst,
                        random.Random(seed), deadline=time.monotonic() + seconds)
        dt = time.perf_counter() - t0
    finally:
        LS.enumerate_candidates = real
    return count[0], dt


def leg(inst, theta, sols, ids, depth=500, seconds=15.0, workers=None):
    """Reference local_search on `workers` processes (one start state each) for
    about `seconds` of wall time each; returns a cpu_baseline-style dict."""
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    workers = workers or (os.cpu_count() or 1)
    k = min(len(sols), workers)
    nodes = [(n.id, n.kind, n.x, n.y, n.demand, n.service, n.tw_early, n.tw_late) for n in inst.nodes]
    jobs = [(inst.variant.value, nodes, inst.n_depots, inst.dist, inst.fleet_per_depot, inst.capacity,
             inst.max_duration, theta, [(r.depart, r.arrive, list(r.customers)) for r in sols[j].routes], ids[j],
             depth, seconds) for j in range(k)]
    t0 = time.perf_counter()
    with ProcessPoolExecutor(k, mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(_worker, jobs))
    wall = time.perf_counter() - t0
    cands = sum(c for c, _ in res)
    busy = max(dt for _, dt in res)
    return {"value": cands / busy, "unit": "move-evals/s", "cores": k, "kind": "reference",
            "sample": f"UNMODIFIED mdroute (numpy, baseline/_ref) local_search of start states {ids[0]}..{ids[k-1]} "
                      f"(depth {depth}, multi-move) on {k} processes, each stopped by its deadline after "
                      f"{seconds:.0f} s; {cands} candidates; rate = candidates / slowest worker's search time "
                      f"({busy:.1f} s; {wall:.1f} s wall incl. process start and instance build)",
            "per_core": cands / sum(dt for _, dt in res)}
