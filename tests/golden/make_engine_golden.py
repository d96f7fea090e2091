"""Golden generation-loop runs from the REAL reference (mdroute.engine.run).

Run in the build container (the reference is mounted read-only at /root/reference):

    python tests/golden/make_engine_golden.py

Writes tests/golden/engine.json: small seeded instances (the reference test
fixture generator) and SolverConfigs, and the reference's RunStats for each --
best and best-infeasible cost (exact, as float hex), their routes, the number of
generations, the per-generation best-cost curve and stagnation trace.
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
from mdroute import engine  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # tag, instance (variant, n_customers, n_depots, kwargs, seed), SolverConfig kwargs
    ("vrp_mm", ("mdvrp", 22, 2, dict(fleet=3), 11), dict(generations=30, mu=4, theta=8, depth=40, multi_move=True, seed=1)),
    ("vrp_sm", ("mdvrp", 18, 3, {}, 12), dict(generations=24, mu=5, theta=6, depth=25, multi_move=False, seed=2)),
    ("tw_mm", ("mdvrptw", 20, 2, dict(fleet=3, max_duration=700.0), 13), dict(generations=25, mu=4, theta=8, depth=40, multi_move=True, seed=3)),
    ("open_mm", ("mdovrp", 24, 3, {}, 14), dict(generations=25, mu=4, theta=10, depth=40, multi_move=True, seed=4)),
    ("stagnate", ("mdvrp", 12, 2, {}, 15), dict(generations=60, patience=6, mu=3, theta=5, depth=30, multi_move=True, seed=5)),
    ("tw_sm", ("mdvrptw", 26, 3, dict(fleet=2), 16), dict(generations=20, mu=6, theta=12, depth=30, multi_move=False, seed=6)),
    ("open_sm", ("mdovrp", 30, 2, dict(fleet=3), 17), dict(generations=20, mu=5, theta=8, depth=35, multi_move=False, seed=7)),
    ("vrp_dur", ("mdvrp", 28, 4, dict(max_duration=250.0, fleet=2), 18), dict(generations=22, mu=4, theta=9, depth=45, multi_move=True, xi=0.4, seed=8)),
    ("tw_big", ("mdvrptw", 45, 4, dict(max_duration=900.0), 19), dict(generations=12, mu=8, theta=15, depth=60, multi_move=True, kappa=0.3, seed=9)),
    ("vrp_one", ("mdvrp", 16, 1, {}, 20), dict(generations=15, mu=3, theta=4, depth=20, multi_move=True, seed=10)),
    ("tight_cap", ("mdvrp", 24, 2, dict(capacity=25), 21), dict(generations=18, mu=4, theta=6, depth=40, multi_move=True, seed=11)),
]


def routes(sol):
    return None if sol is None else [[r.depart, r.arrive, list(r.customers)] for r in sol.routes]


def main():
    out = {}
    for tag, (variant, nc, nd, kw, iseed), cfg_kw in CASES:
        inst = rconf.make_instance(random.Random(iseed), variant, n_customers=nc, n_depots=nd, **kw)
        st = engine.run(inst, engine.SolverConfig(**cfg_kw))
        out[tag] = dict(instance=[variant, nc, nd, kw, iseed], config=cfg_kw,
                        best_cost=float(st.best_cost).hex(), feasible_found=st.feasible_found,
                        best_infeasible_cost=float(st.best_infeasible_cost).hex(),
                        best=routes(st.best), best_infeasible=routes(st.best_infeasible),
                        generations=st.generations, cost_curve=[float(x).hex() for x in st.cost_curve],
                        stagnation_trace=list(st.stagnation_trace))
        print(tag, st.generations, st.best_cost, st.feasible_found, round(st.wall_time, 2))
    with open(os.path.join(HERE, "engine.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
