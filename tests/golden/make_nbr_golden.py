"""Golden neighbour lists from the REAL reference (mdroute.neighborhood.build).

Run in the build container (the reference is mounted read-only at /root/reference):

    python tests/golden/make_nbr_golden.py

Writes tests/golden/nbr_edge.npz: instances chosen for the corners of
neighborhood.py:60-101 -- exact eta ties (duplicated coordinates), mixed finite
and infinite time windows (the nan_to_num path), heavy pruning, theta larger than
the candidate count, theta = 1, and a 4,100-node instance whose rows exceed one
4,096-slot sorting chunk on the device.  Stored per case: node table (x, y, q, s,
e, l), variant, n_depots, theta, gamma (hex), dist sha256, and the reference's
lists and mask row sums.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from mdroute import evaluation, model, neighborhood  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def make(rng, variant, nc, nd, *, dup=0, inf_frac=0.0, tight=False):
    depots = [(rng.uniform(0, 100), rng.uniform(0, 100)) for _ in range(nd)]
    cust = []
    for i in range(nc):
        if dup and i >= nc - dup:  # exact duplicate of an earlier customer's position
            x, y = cust[rng.randrange(nc - dup)][:2]
        else:
            x, y = rng.uniform(0, 100), rng.uniform(0, 100)
        q = rng.randint(1, 25)
        if variant == "mdvrptw" and rng.random() >= inf_frac:
            s = rng.uniform(1, 20)
            e = rng.uniform(0, 700)
            w = rng.uniform(5, 30) if tight else rng.uniform(30, 200)
            cust.append((x, y, q, s, e, e + w))
        else:
            cust.append((x, y, q, rng.choice([0.0, 10.0])))
    dw = [(0.0, 1000.0)] * nd if variant == "mdvrptw" else None
    return model.Instance.from_coords(variant, depots, cust, fleet_per_depot=4, capacity=200,
                                      max_duration=float("inf"), depot_windows=dw)


def main():
    rng = random.Random(5150)
    specs = [
        ("ties", "mdvrp", 40, 3, dict(dup=12), 8),
        ("ties_tw", "mdvrptw", 40, 3, dict(dup=10), 6),
        ("mixed_inf", "mdvrptw", 60, 4, dict(inf_frac=0.3), 10),
        ("all_inf_tw", "mdvrptw", 30, 2, dict(inf_frac=1.0), 7),
        ("tight", "mdvrptw", 80, 5, dict(tight=True), 12),
        ("theta_gt", "mdvrp", 20, 2, {}, 60),
        ("theta1", "mdovrp", 50, 4, {}, 1),
        ("open", "mdovrp", 120, 6, {}, 30),
        ("chunked", "mdvrp", 4090, 10, dict(dup=40), 40),
        ("chunked_tw", "mdvrptw", 4100, 8, dict(inf_frac=0.1), 40),
    ]
    store, manifest = {}, {}
    for tag, variant, nc, nd, kw, theta in specs:
        inst = make(rng, variant, nc, nd, **kw)
        consts = evaluation.ScalingConstants.from_instance(inst)
        nbr = neighborhood.build(inst, neighborhood.NeighborConfig(theta), consts)
        nodes = np.array([[n.x, n.y, n.demand, n.service, n.tw_early, n.tw_late] for n in inst.nodes])
        store[f"{tag}_nodes"] = nodes
        store[f"{tag}_lists"] = np.ascontiguousarray(nbr.lists, np.int32)
        store[f"{tag}_masksum"] = nbr.mask.sum(axis=1).astype(np.int32)
        manifest[tag] = dict(variant=variant, n_depots=nd, theta=theta, gamma=consts.gamma.hex(),
                             theta_c=consts.theta.hex(),
                             dist_sha=hashlib.sha256(np.ascontiguousarray(inst.dist).tobytes()).hexdigest())
        print(tag, inst.n_nodes, theta, int((nbr.lists >= 0).sum()))
    np.savez_compressed(os.path.join(HERE, "nbr_edge.npz"), **store)
    with open(os.path.join(HERE, "nbr_edge.json"), "w") as f:
        json.dump(manifest, f, indent=1)


if __name__ == "__main__":
    main()
