"""Golden repair-insertion results from the REAL reference (mdroute.genetic.repair_insert).

Run in the build container (the reference is mounted read-only at /root/reference):

    python tests/golden/make_repair_golden.py

Writes tests/golden/repair.npz + repair.json.  Each case: an instance (node table),
a partial solution (a full solution with a random subset of customers removed;
routes may be left empty), the unrouted customers in the order handed to
repair_insert, the insertion operator (FBI/IBI/FRI/IRI/RI), lambda, the seed of
the rng passed in (used by RI only), and the reference's output routes.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import conftest as rconf  # noqa: E402
from mdroute import evaluation, genetic, model  # noqa: E402
from mdroute.model import INF, Route, Solution  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OPS = ["FBI", "IBI", "FRI", "IRI", "RI"]


def flat(sol):
    off = np.zeros(len(sol.routes) + 1, np.int32)
    if sol.routes:
        off[1:] = np.cumsum([len(r.customers) for r in sol.routes])
    cust = np.array([c for r in sol.routes for c in r.customers], np.int32)
    dep = np.array([r.depart for r in sol.routes], np.int32)
    arr = np.array([r.arrive for r in sol.routes], np.int32)
    return off, cust, dep, arr


def main():
    rng = random.Random(777)
    store, manifest = {}, {}
    shapes = [
        ("vrp", "mdvrp", 30, 3, dict(fleet=3)),
        ("vrp_inf", "mdvrp", 40, 2, {}),
        ("tw", "mdvrptw", 35, 3, dict(max_duration=900.0, fleet=4)),
        ("tw_tight", "mdvrptw", 25, 2, dict(capacity=20, max_duration=500.0)),
        ("open", "mdovrp", 40, 4, {}),
        ("vrp_dur", "mdvrp", 50, 4, dict(max_duration=300.0, fleet=2)),
    ]
    n = 0
    for sname, variant, nc, nd, kw in shapes:
        for rep in range(4):
            inst = rconf.make_instance(random.Random(rng.randrange(1 << 30)), variant, n_customers=nc,
                                       n_depots=nd, **kw)
            consts = evaluation.ScalingConstants.from_instance(inst)
            base = rconf.random_solution(random.Random(rng.randrange(1 << 30)), inst)
            for op in OPS:
                sol = base.clone()
                frac = rng.choice([0.1, 0.3, 0.6, 1.0])
                cust = [c for r in sol.routes for c in r.customers]
                removed = set(rng.sample(cust, max(1, int(len(cust) * frac))))
                for r in sol.routes:
                    r.customers = [c for c in r.customers if c not in removed]
                if rng.random() < 0.5:
                    sol.drop_empty_routes()
                if frac == 1.0 and rng.random() < 0.5:
                    sol.routes = []
                unrouted = sorted(removed)
                rng.shuffle(unrouted)
                lam = [rng.choice([0.01, 0.5, 1.0, 3.0, 100.0]) for _ in range(4)]
                seed = rng.randrange(1 << 30)
                before = flat(sol)
                out = genetic.repair_insert(sol, list(unrouted), genetic.InsertionOperator[op], inst, consts,
                                            evaluation.PenaltyState(lam=list(lam)), random.Random(seed))
                tag = f"c{n:03d}"
                n += 1
                nodes = np.array([[v.x, v.y, v.demand, v.service, v.tw_early, v.tw_late] for v in inst.nodes])
                store[f"{tag}_nodes"] = nodes
                for k, a in zip(("off", "cust", "dep", "arr"), before):
                    store[f"{tag}_in_{k}"] = a
                for k, a in zip(("off", "cust", "dep", "arr"), flat(out)):
                    store[f"{tag}_out_{k}"] = a
                store[f"{tag}_unrouted"] = np.array(unrouted, np.int32)
                manifest[tag] = dict(shape=sname, variant=variant, n_depots=nd,
                                     fleet=float(inst.fleet_per_depot), capacity=float(inst.capacity),
                                     max_duration=float(inst.max_duration), op=op, lam=lam, seed=seed,
                                     gamma=consts.gamma.hex(), theta=consts.theta.hex(),
                                     dist_sha=hashlib.sha256(np.ascontiguousarray(inst.dist).tobytes()).hexdigest())
    np.savez_compressed(os.path.join(HERE, "repair.npz"), **store)
    with open(os.path.join(HERE, "repair.json"), "w") as f:
        json.dump(manifest, f, indent=0)
    print(n, "cases")


if __name__ == "__main__":
    main()
