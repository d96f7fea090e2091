"""Generate the golden parity fixtures from the REAL reference package.

Run in the build container (the reference is mounted read-only at
/root/reference; it is not available on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed): tests/golden/{ops_small,ops_medium,ls_traj}.npz and
manifest.json.  Every number in them is produced by the reference's own code:
mdroute.moves.enumerate_candidates, mdroute.batch.evaluate_candidates,
mdroute.batch.leader_and_followers, mdroute.localsearch.select_moves and
mdroute.localsearch.local_search (the latter instrumented only by wrapping the
module-level names it calls, to record the per-step trace).
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import conftest as rconf  # noqa: E402  reference test fixtures
from mdroute import batch, bench, evaluation, genetic, localsearch, model, moves, neighborhood  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
FIELDS = ("r1", "p1", "r2", "p2", "len1", "len2", "rev1", "rev2", "depot", "mode")
DFIELDS = ("dD", "dV1", "dV2", "dV3", "dV4", "dF")
VAR_CODE = {"mdvrp": 0, "mdvrptw": 1, "mdovrp": 2}


def inst_record(inst, consts, nbr):
    nodes = np.array([[n.x, n.y, n.demand, n.service, n.tw_early, n.tw_late] for n in inst.nodes])
    meta = dict(variant=inst.variant.value, n_depots=inst.n_depots,
                fleet=float(inst.fleet_per_depot), capacity=float(inst.capacity),
                max_duration=float(inst.max_duration), gamma=consts.gamma.hex(),
                theta=consts.theta.hex(),
                dist_sha=hashlib.sha256(np.ascontiguousarray(inst.dist).tobytes()).hexdigest(),
                time_is_dist=inst.time is inst.dist)
    return nodes, np.ascontiguousarray(nbr.lists, np.int32), meta


def sol_arrays(sol):
    off = np.zeros(len(sol.routes) + 1, np.int32)
    off[1:] = np.cumsum([len(r.customers) for r in sol.routes]) if sol.routes else []
    cust = np.array([c for r in sol.routes for c in r.customers], np.int32)
    dep = np.array([r.depart for r in sol.routes], np.int32)
    arr = np.array([r.arrive for r in sol.routes], np.int32)
    return off, cust, dep, arr


def cand_matrix(cs):
    return np.stack([getattr(cs, f).astype(np.int64) for f in FIELDS]) if len(cs) else np.zeros((10, 0), np.int64)


def delta_matrix(d):
    return np.stack([getattr(d, f) for f in DFIELDS])


def canon_sha(cm, dm, fn):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(cm, np.int64).tobytes())
    h.update((np.ascontiguousarray(dm, np.float64) + 0.0).tobytes())  # -0 -> +0
    h.update(np.ascontiguousarray(fn, np.uint8).tobytes())
    return h.hexdigest()


def put_case(store, manifest, tag, inst, consts, nbr, sol, lam, extra=None):
    nodes, lists, meta = inst_record(inst, consts, nbr)
    off, cust, dep, arr = sol_arrays(sol)
    store[f"{tag}_nodes"] = nodes
    store[f"{tag}_lists"] = lists
    store[f"{tag}_off"], store[f"{tag}_cust"] = off, cust
    store[f"{tag}_dep"], store[f"{tag}_arr"] = dep, arr
    store[f"{tag}_lam"] = np.array(lam, np.float64)
    meta.update(extra or {})
    manifest[tag] = meta
    return meta


def op_goldens(store, meta, tag, inst, consts, nbr, sol, pen, full: bool, rng):
    cache = batch.SolutionCache(sol, inst, consts)
    sidx = moves.SolutionIndex(sol, inst)
    ops = {}
    for op in moves.ALL_OPS:
        cs = moves.enumerate_candidates(sol, op, nbr, inst, sidx)
        d = batch.evaluate_candidates(cache, cs, pen)
        cm, dm = cand_matrix(cs), delta_matrix(d)
        leader, followers = batch.leader_and_followers(cache, cs, d, True)
        chosen = localsearch.select_moves(leader, followers) if leader is not None else []
        rec = dict(n=len(cs), sha=canon_sha(cm, dm, d.fleet_neutral),
                   leader=list(leader.key()) if leader is not None else None,
                   leader_dF=leader.dF.hex() if leader is not None else None,
                   n_followers=len(followers),
                   followers=[list(f.key()) for f in followers[:256]],
                   chosen=[list(m.key()) for m in chosen])
        if full:
            store[f"{tag}_op{int(op)}_c"] = cm
            store[f"{tag}_op{int(op)}_d"] = dm
            store[f"{tag}_op{int(op)}_fn"] = d.fleet_neutral.astype(np.uint8)
        elif len(cs):
            idx = np.array(sorted(rng.sample(range(len(cs)), min(512, len(cs)))), np.int64)
            store[f"{tag}_op{int(op)}_si"] = idx
            store[f"{tag}_op{int(op)}_sc"] = cm[:, idx]
            store[f"{tag}_op{int(op)}_sd"] = dm[:, idx]
            store[f"{tag}_op{int(op)}_sfn"] = d.fleet_neutral[idx].astype(np.uint8)
        ops[int(op)] = rec
    meta["ops"] = ops
    meta["totals"] = [float(x).hex() for x in cache.totals()]


def perms_for(rng, ops, n):
    clone = random.Random()
    clone.setstate(rng.getstate())
    out = []
    for _ in range(n):
        o = list(ops)
        clone.shuffle(o)
        out.append([int(x) for x in o])
    return np.array(out, np.int32)


class CountingRng:
    """Delegates to a random.Random and counts shuffle calls (one per pass)."""

    def __init__(self, rng):
        self.rng = rng
        self.shuffles = 0

    def shuffle(self, x):
        self.shuffles += 1
        self.rng.shuffle(x)


def ls_golden(store, manifest, tag, inst, consts, nbr, sol, depth, multi_move, ls_seed):
    pen = evaluation.PenaltyState()
    put_case(store, manifest, tag, inst, consts, nbr, sol, pen.lam,
             dict(depth=depth, multi_move=multi_move, ls_seed=ls_seed))
    ops = localsearch.enabled_operators(inst)
    rng = random.Random(ls_seed)
    store[f"{tag}_perms"] = perms_for(rng, ops, depth + 1)
    trace = dict(op=[], nmoves=[], keys=[], lam=[], D=[])
    orig_apply, orig_adapt = localsearch.apply_moves, localsearch.adapt_penalties

    def apply_wrap(s, mvs, i):
        trace["op"].append(int(mvs[0].op))
        trace["nmoves"].append(len(mvs))
        trace["keys"].append([list(m.key()) for m in mvs])
        return orig_apply(s, mvs, i)

    def adapt_wrap(p, violated):
        r = orig_adapt(p, violated)
        trace["lam"].append(list(p.lam))
        return r

    localsearch.apply_moves, localsearch.adapt_penalties = apply_wrap, adapt_wrap
    feas = []
    crng = CountingRng(rng)
    t0 = time.time()
    try:
        work = sol.clone()
        localsearch.local_search(work, pen, localsearch.SearchConfig(depth=depth, multi_move=multi_move),
                                 nbr, consts, inst, crng,
                                 on_feasible=lambda D, s: feas.append(D))
    finally:
        localsearch.apply_moves, localsearch.adapt_penalties = orig_apply, orig_adapt
    off, cust, dep, arr = sol_arrays(work)
    store[f"{tag}_fin_off"], store[f"{tag}_fin_cust"] = off, cust
    store[f"{tag}_fin_dep"], store[f"{tag}_fin_arr"] = dep, arr
    store[f"{tag}_tr_op"] = np.array(trace["op"], np.int32)
    store[f"{tag}_tr_nmoves"] = np.array(trace["nmoves"], np.int32)
    store[f"{tag}_tr_lam"] = np.array(trace["lam"], np.float64).reshape(-1, 4)
    keys = [k for ks in trace["keys"] for k in ks]
    store[f"{tag}_tr_keys"] = np.array(keys, np.int64).reshape(-1, 11)
    store[f"{tag}_feasD"] = np.array(feas, np.float64)
    manifest[tag].update(passes=crng.shuffles, accepted=len(trace["op"]),
                         final_lam=[x.hex() for x in pen.lam], ref_seconds=round(time.time() - t0, 3))


def main():
    small, medium, traj = {}, {}, {}
    man = dict(small={}, medium={}, traj={})
    variants = [model.Variant.MDVRP, model.Variant.MDVRPTW, model.Variant.MDOVRP]

    # ---- small operator cases: full arrays (conftest-style random states) ----
    rng = random.Random(20260101)
    samp = random.Random(7)
    for i in range(60):
        v = variants[i % 3]
        inst = rconf.make_instance(rng, v, n_customers=rng.randint(3, 12), n_depots=rng.randint(1, 3),
                                   fleet=rng.choice([None, 1, 2]),
                                   max_duration=None if v is model.Variant.MDOVRP else rng.choice([None, 300.0]))
        consts = evaluation.ScalingConstants.from_instance(inst)
        theta = rng.choice([2, 4, 8, inst.n_nodes])
        nbr = neighborhood.build(inst, neighborhood.NeighborConfig(theta), consts)
        sol = rconf.random_solution(rng, inst, scramble_depots=rng.random() < 0.8)
        if i % 10 == 9:
            sol.routes.insert(rng.randrange(len(sol.routes) + 1),
                              model.Route(rng.randrange(inst.n_depots), rng.randrange(inst.n_depots), []))
        if i % 10 == 4 and sum(len(r.customers) for r in sol.routes) > 3:
            r = max(sol.routes, key=lambda r: len(r.customers))
            r.customers.pop()  # partial coverage: one unrouted customer
        pen = evaluation.PenaltyState(lam=[rng.uniform(0.2, 4) for _ in range(4)])
        tag = f"s{i}"
        meta = put_case(small, man["small"], tag, inst, consts, nbr, sol, pen.lam)
        op_goldens(small, meta, tag, inst, consts, nbr, sol, pen, True, samp)

    # ---- medium operator cases: sha-pinned full arrays + samples ----
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
        inst = model.Instance.from_coords(variant, depots, cust, fleet_per_depot=nv, capacity=q,
                                          max_duration=dur,
                                          depot_windows=[(0.0, 1000.0)] * nd if windows else None)
        return inst, r

    INF = model.INF
    shapes = {
        "C1": (model.Variant.MDVRP, 50, 4, 4, 80, INF, 50),
        "C2": (model.Variant.MDVRPTW, 288, 6, 12, 200, 450, 50),
        "C3": (model.Variant.MDOVRP, 360, 9, INF, 200, INF, 50),
    }
    built = {}
    for name, (v, nc, nd, nv, q, dur, th) in shapes.items():
        inst, r = appendix_a(v, nc, nd, nv, q, dur)
        consts = evaluation.ScalingConstants.from_instance(inst)
        nbr = neighborhood.build(inst, neighborhood.NeighborConfig(th), consts)
        built[name] = (inst, consts, nbr)
        sol = genetic.initial_solution(inst, consts, evaluation.PenaltyState(), r)
        pen = evaluation.PenaltyState()
        meta = put_case(medium, man["medium"], f"{name}_init", inst, consts, nbr, sol, pen.lam,
                        dict(shape=name))
        op_goldens(medium, meta, f"{name}_init", inst, consts, nbr, sol, pen, False, samp)
        sol2 = rconf.random_solution(random.Random(11), inst)
        pen2 = evaluation.PenaltyState(lam=[0.7, 3.0, 1.5, 2.5])
        meta = put_case(medium, man["medium"], f"{name}_rand", inst, consts, nbr, sol2, pen2.lam,
                        dict(shape=name))
        op_goldens(medium, meta, f"{name}_rand", inst, consts, nbr, sol2, pen2, False, samp)
    p01 = os.path.join(REF, "src/mdroute/data/instances/c97/p01")
    for v in (model.Variant.MDVRP, model.Variant.MDOVRP):
        inst = bench.parse_instance(p01, v)
        consts = evaluation.ScalingConstants.from_instance(inst)
        nbr = neighborhood.build(inst, neighborhood.NeighborConfig(50), consts)
        built[f"p01_{v.value}"] = (inst, consts, nbr)
        sol = genetic.initial_solution(inst, consts, evaluation.PenaltyState(), random.Random(1))
        pen = evaluation.PenaltyState()
        tag = f"p01_{v.value}"
        meta = put_case(medium, man["medium"], tag, inst, consts, nbr, sol, pen.lam, dict(shape="p01"))
        op_goldens(medium, meta, tag, inst, consts, nbr, sol, pen, True, samp)

    # ---- local-search trajectories ----
    rng = random.Random(424242)
    for i in range(36):
        v = variants[i % 3]
        inst = rconf.make_instance(rng, v, n_customers=rng.randint(5, 30), n_depots=rng.randint(1, 4),
                                   fleet=rng.choice([None, 1, 2, 3]),
                                   max_duration=None if v is model.Variant.MDOVRP else rng.choice([None, 300.0]))
        consts = evaluation.ScalingConstants.from_instance(inst)
        nbr = neighborhood.build(inst, neighborhood.NeighborConfig(rng.choice([4, 8, 50])), consts)
        sol = rconf.random_solution(rng, inst)
        ls_golden(traj, man["traj"], f"t{i}", inst, consts, nbr, sol,
                  rng.choice([3, 20, 500]), i % 2 == 0, 1000 + i)
    for s in range(3):
        inst, consts, nbr = built["C1"]
        sol = genetic.initial_solution(inst, consts, evaluation.PenaltyState(), random.Random(100 + s))
        ls_golden(traj, man["traj"], f"C1_d{s}", inst, consts, nbr, sol, 500, True, s)
    for v in ("mdvrp", "mdovrp"):
        inst, consts, nbr = built[f"p01_{v}"]
        sol = genetic.initial_solution(inst, consts, evaluation.PenaltyState(), random.Random(100))
        ls_golden(traj, man["traj"], f"p01_{v}_d0", inst, consts, nbr, sol, 500, True, 0)
    inst, consts, nbr = built["C3"]
    sol = genetic.initial_solution(inst, consts, evaluation.PenaltyState(), random.Random(100))
    ls_golden(traj, man["traj"], "C3_d0", inst, consts, nbr, sol, 500, True, 0)
    inst, consts, nbr = built["C2"]
    sol = genetic.initial_solution(inst, consts, evaluation.PenaltyState(), random.Random(100))
    ls_golden(traj, man["traj"], "C2_d0", inst, consts, nbr, sol, 60, True, 0)

    np.savez_compressed(os.path.join(HERE, "ops_small.npz"), **small)
    np.savez_compressed(os.path.join(HERE, "ops_medium.npz"), **medium)
    np.savez_compressed(os.path.join(HERE, "ls_traj.npz"), **traj)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(man, f, indent=1, sort_keys=True)
    print("cases:", {k: len(v) for k, v in man.items()})


if __name__ == "__main__":
    main()
