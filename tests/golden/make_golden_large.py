"""Golden fixtures at the benchmark's own shapes, from the REAL reference package.

BASELINE.json configs[3] (C4: MDVRPTW 1000x10, theta 50) and configs[4]
(C5: MDVRP 4000x20, theta 40), SURVEY.md Appendix A generator (seed 2026):

* start states: reference genetic.initial_solution(..., random.Random(100+i))
  for individuals 0..3 (full routes) -- pins workload.initial_solution;
* operator level on individual 0's start state: per operator the candidate
  count, the SHA-256 of the full candidate/delta arrays (as make_golden.py),
  the leader key, follower count and the select_moves result;
* complete descents (C4, individuals 0 and 1): reference local_search with
  SearchConfig(depth=500, multi_move=True), lambda = 1, kappa = 0.5 and
  rng random.Random(i), recording the final routes, lambda, passes, accepted
  steps and the per-operator candidate counts (counted by wrapping the
  module-level name enumerate_candidates that local_search calls).

Run once in the build container (the reference lives at /root/reference, which
the GPU box does not have); C4 descents take ~150 s each:

    python tests/golden/make_golden_large.py

Outputs (committed): tests/golden/large.npz, tests/golden/large.json.
"""
from __future__ import annotations

import json
import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402  (puts the reference on sys.path)
from mdroute import batch, evaluation, genetic, localsearch, model, moves, neighborhood  # noqa: E402

SHAPES = {
    "C4": (model.Variant.MDVRPTW, 1000, 10, 30, 200, 450, 50),
    "C5": (model.Variant.MDVRP, 4000, 20, model.INF, 200, model.INF, 40),
}


def appendix_a(variant, nc, nd, nv, q, dur, seed=2026):
    r = random.Random(seed)
    windows = variant is model.Variant.MDVRPTW
    depots = [(r.uniform(0, 100), r.uniform(0, 100)) for _ in range(nd)]
    cust = []
    for _ in range(nc):
        x = r.uniform(0, 100); y = r.uniform(0, 100); qq = r.randint(1, 25)
        if windows:
            s = r.uniform(1, 20); e = r.uniform(0, 700)
            cust.append((x, y, qq, s, e, e + r.uniform(30, 200)))
        else:
            cust.append((x, y, qq, r.choice([0.0, 10.0])))
    return model.Instance.from_coords(variant, depots, cust, fleet_per_depot=nv, capacity=q, max_duration=dur,
                                      depot_windows=[(0.0, 1000.0)] * nd if windows else None)


def routes(sol):
    return [[r.depart, r.arrive, list(r.customers)] for r in sol.routes]


def main():
    store, man = {}, {}
    for name, (v, nc, nd, nv, q, dur, th) in SHAPES.items():
        t0 = time.time()
        inst = appendix_a(v, nc, nd, nv, q, dur)
        consts = evaluation.ScalingConstants.from_instance(inst)
        nbr = neighborhood.build(inst, neighborhood.NeighborConfig(th), consts)
        _, _, meta = MG.inst_record(inst, consts, nbr)
        meta["lists_sha"] = MG.hashlib.sha256(np.ascontiguousarray(nbr.lists, np.int32).tobytes()).hexdigest()
        starts = [genetic.initial_solution(inst, consts, evaluation.PenaltyState(), random.Random(100 + i))
                  for i in range(4)]
        meta["starts"] = [routes(s) for s in starts]
        # operator level on individual 0's start (SHA of the full arrays, as make_golden.py)
        sol, pen = starts[0], evaluation.PenaltyState()
        cache = batch.SolutionCache(sol, inst, consts)
        sidx = moves.SolutionIndex(sol, inst)
        ops = {}
        for op in moves.ALL_OPS:
            cs = moves.enumerate_candidates(sol, op, nbr, inst, sidx)
            d = batch.evaluate_candidates(cache, cs, pen)
            cm, dm = MG.cand_matrix(cs), MG.delta_matrix(d)
            leader, followers = batch.leader_and_followers(cache, cs, d, True)
            chosen = localsearch.select_moves(leader, followers) if leader is not None else []
            ops[int(op)] = dict(n=len(cs), sha=MG.canon_sha(cm, dm, d.fleet_neutral),
                                leader=list(leader.key()) if leader is not None else None,
                                leader_dF=leader.dF.hex() if leader is not None else None,
                                n_followers=len(followers), chosen=[list(m.key()) for m in chosen])
        meta["ops"] = ops
        meta["totals"] = [float(x).hex() for x in cache.totals()]
        meta["seconds_setup"] = round(time.time() - t0, 1)
        # complete descents (C4 only: a C5 descent is ~25 min of numpy)
        meta["descents"] = {}
        for i in ((0, 1) if name == "C4" else ()):
            counts = [0] * 6
            orig = localsearch.enumerate_candidates

            def counting(s, op, nb, ins, sx=None, _o=orig):
                cs = _o(s, op, nb, ins, sx)
                counts[int(op)] += len(cs)
                return cs

            work, pen = starts[i].clone(), evaluation.PenaltyState()
            crng = MG.CountingRng(random.Random(i))
            steps = []
            orig_apply = localsearch.apply_moves

            def apply_wrap(s, mvs, ins, _o=orig_apply):
                steps.append(len(mvs))
                return _o(s, mvs, ins)

            localsearch.enumerate_candidates, localsearch.apply_moves = counting, apply_wrap
            t1 = time.time()
            try:
                localsearch.local_search(work, pen, localsearch.SearchConfig(depth=500, multi_move=True), nbr,
                                         consts, inst, crng)
            finally:
                localsearch.enumerate_candidates, localsearch.apply_moves = orig, orig_apply
            meta["descents"][str(i)] = dict(final=routes(work), lam=[x.hex() for x in pen.lam],
                                            passes=crng.shuffles, accepted=len(steps), moves=sum(steps),
                                            cands=counts, ref_seconds=round(time.time() - t1, 1))
            print(name, i, meta["descents"][str(i)]["ref_seconds"], "s", sum(counts), "cands", flush=True)
        man[name] = meta
        print(name, "done", round(time.time() - t0, 1), "s", flush=True)
    with open(os.path.join(HERE, "large.json"), "w") as f:
        json.dump(man, f, sort_keys=True)
    print("wrote large.json")


if __name__ == "__main__":
    main()
