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
