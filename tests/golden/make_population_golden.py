"""Golden survivor selections from the REAL reference population manager
(population.py:70-122): edge-set distance matrices and the survivors, in order,
of Population.survivor_selection.

Run in the build container (the reference is mounted read-only at /root/reference):

    python tests/golden/make_population_golden.py

Writes tests/golden/population.json: per case the instance recipe (reference
test fixture generator and seed), the members' routes, breakdown fields,
lambda, mu and xi; the reference's distance matrix (float hex) and the births
of the survivors in member order.  Members include exact clones (distance-0
ties) and equal-cost pairs, so both rank tie-breaks by birth are exercised.
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
from mdroute import evaluation, population  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
H = lambda x: float(x).hex()  # noqa: E731


def main():
    rng = random.Random(4242)
    specs = [("mdvrp", 30, 3, 20, 0.7, 31), ("mdvrptw", 25, 2, 10, 0.7, 25), ("mdovrp", 28, 4, 8, 0.3, 20),
             ("mdvrp", 12, 2, 5, 0.7, 12), ("mdvrptw", 40, 3, 20, 1.5, 45), ("mdvrp", 8, 2, 1, 0.7, 3),
             ("mdvrp", 60, 4, 40, 0.7, 90)]
    out = []
    for variant, nc, nd, mu, xi, n in specs:
        iseed = rng.randrange(1 << 30)
        inst = rconf.make_instance(random.Random(iseed), variant, n_customers=nc, n_depots=nd)
        consts = evaluation.ScalingConstants.from_instance(inst)
        pen = evaluation.PenaltyState(lam=[rng.choice([0.5, 1.0, 2.0]) for _ in range(4)])
        pop = population.Population(mu, xi)
        sols = []
        for i in range(n):
            if sols and rng.random() < 0.2:
                s = rng.choice(sols).clone()  # exact clone: distance 0 and equal cost
            else:
                s = rconf.random_solution(random.Random(rng.randrange(1 << 30)), inst)
            sols.append(s)
            bd = evaluation.evaluate(s, pen, consts, inst)
            pop.add(s, bd, bd.V1 + bd.V2 + bd.V3 + bd.V4 <= 1e-9, inst)
        members = [dict(routes=[[r.depart, r.arrive, list(r.customers)] for r in m.sol.routes],
                        bd=[H(m.breakdown.D), H(m.breakdown.V1), H(m.breakdown.V2), H(m.breakdown.V3),
                            H(m.breakdown.V4)], feasible=m.feasible, birth=m.birth) for m in pop.members]
        dist = [[H(x) for x in row] for row in pop.distance_matrix()]
        pop.survivor_selection(pen)
        out.append(dict(spec=[variant, nc, nd, iseed], mu=mu, xi=xi, lam=pen.lam, members=members, dist=dist,
                        survivors=[m.birth for m in pop.members]))
    json.dump(out, open(os.path.join(HERE, "population.json"), "w"))
    print("wrote", len(out), "cases")


if __name__ == "__main__":
    main()
