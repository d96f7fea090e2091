"""Golden values of the reference's scalar oracles
from the REAL reference: evaluation.move_delta / evaluate and
model.check_feasible / simulate_route / minimal_duration.

Run in the build container (the reference is mounted read-only at /root/reference):

    python tests/golden/make_scalar_golden.py

Writes tests/golden/scalar.json: per case the instance recipe (reference test
fixture generator, seed), a random solution, lambda, evaluate() of it, the
feasibility report, per-route simulation and minimal duration, and move_delta
for a sample of every operator's enumerated candidates (exact, as float hex).
"""
from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import conftest as rconf  # noqa: E402
from mdroute import evaluation, model, moves, neighborhood  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
H = lambda x: float(x).hex()  # noqa: E731


def main():
    rng = random.Random(99)
    specs = [("mdvrp", 30, 3, dict(fleet=2)), ("mdvrptw", 25, 2, dict(max_duration=600.0, fleet=3)),
             ("mdvrptw", 35, 3, {}), ("mdovrp", 28, 4, {}), ("mdvrp", 20, 2, dict(max_duration=200.0, capacity=20))]
    out = []
    for variant, nc, nd, kw in specs:
        for rep in range(2):
            iseed, sseed = rng.randrange(1 << 30), rng.randrange(1 << 30)
            inst = rconf.make_instance(random.Random(iseed), variant, n_customers=nc, n_depots=nd, **kw)
            sol = rconf.random_solution(random.Random(sseed), inst)
            if rep == 1 and sol.routes:  # structural edge: an emptied route and a missing customer
                sol.routes[0].customers = []
            consts = evaluation.ScalingConstants.from_instance(inst)
            lam = [rng.choice([0.1, 1.0, 20.0]) for _ in range(4)]
            pen = evaluation.PenaltyState(lam=list(lam))
            nbr = neighborhood.build(inst, neighborhood.NeighborConfig(6), consts)
            bd = evaluation.evaluate(sol, pen, consts, inst)
            fr = model.check_feasible(sol, inst)
            sims = []
            for r in sol.routes:
                if not r.customers:
                    continue
                s = model.simulate_route(r, inst)
                sims.append([H(s.distance), H(s.load), H(s.duration), H(s.time_warp), s.late_count,
                             H(model.minimal_duration(r, inst))])
            deltas = []
            for op in moves.ALL_OPS:
                cs = moves.enumerate_candidates(sol, op, nbr, inst)
                n = len(cs)
                for i in sorted(rng.sample(range(n), min(n, 25))):
                    mv = moves.Move(op, int(cs.r1[i]), int(cs.p1[i]), int(cs.r2[i]), int(cs.p2[i]),
                                    int(cs.len1[i]), int(cs.len2[i]), bool(cs.rev1[i]), bool(cs.rev2[i]),
                                    int(cs.depot[i]), int(cs.mode[i]))
                    d = evaluation.move_delta(sol, mv, pen, consts, inst)
                    deltas.append([list(mv.key()), [H(d.D), H(d.V1), H(d.V2), H(d.V3), H(d.V4), H(d.F)]])
            out.append(dict(variant=variant, nc=nc, nd=nd, kw=kw, iseed=iseed, sseed=sseed, emptied=rep == 1,
                            lam=lam, evaluate=[H(bd.D), H(bd.V1), H(bd.V2), H(bd.V3), H(bd.V4), H(bd.F)],
                            report=dict(structural_error=fr.structural_error, missing=fr.missing,
                                        duplicated=fr.duplicated, capacity_excess=H(fr.capacity_excess),
                                        duration_excess=H(fr.duration_excess), time_warp=H(fr.time_warp),
                                        late_count=fr.late_count, closure_violations=fr.closure_violations,
                                        fleet_excess=fr.fleet_excess, all_ok=fr.all_ok),
                            sims=sims, move_deltas=deltas))
    with open(os.path.join(HERE, "scalar.json"), "w") as f:
        json.dump(out, f)
    print(len(out), "cases,", sum(len(c["move_deltas"]) for c in out), "move deltas")


if __name__ == "__main__":
    main()
