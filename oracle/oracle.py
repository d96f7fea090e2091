"""ctypes binding of the C oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference leg of bench.py.  The product package
(paper_2605_05208_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class InstanceDesc(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_depots", C.c_int32),
                ("dist", _f64p), ("time", _f64p), ("demand", _f64p), ("service", _f64p),
                ("tw_early", _f64p), ("tw_late", _f64p),
                ("capacity", C.c_double), ("max_duration", C.c_double),
                ("fleet_per_depot", C.c_double),
                ("open_routes", C.c_int32), ("has_windows", C.c_int32),
                ("gamma", C.c_double), ("theta", C.c_double),
                ("lists", _i32p), ("width", C.c_int32)]


class FlatSol(C.Structure):
    _fields_ = [("m", C.c_int32), ("off", _i32p), ("cust", _i32p), ("depart", _i32p),
                ("arrive", _i32p)]


class Cands(C.Structure):
    _fields_ = [("n", C.c_int64)] + [(f, _i64p) for f in
                                    ("r1", "p1", "r2", "p2", "len1", "len2", "depot", "mode")] + \
               [("rev1", _u8p), ("rev2", _u8p)]


class Deltas(C.Structure):
    _fields_ = [(f, _f64p) for f in ("dD", "dV1", "dV2", "dV3", "dV4", "dF")] + \
               [("fleet_neutral", _u8p)]


class LsCfg(C.Structure):
    _fields_ = [("depth", C.c_int32), ("multi_move", C.c_int32), ("kappa", C.c_double),
                ("lam_min", C.c_double), ("lam_max", C.c_double), ("max_passes", C.c_int32),
                ("n_ops", C.c_int32), ("perms", _i32p)]


class LsStats(C.Structure):
    _fields_ = [("passes", C.c_int32), ("accepted", C.c_int32), ("op_evals", C.c_int32),
                ("status", C.c_int32), ("cands", C.c_int64 * 6), ("moves_applied", C.c_int64),
                ("n_feasible", C.c_int32), ("best_feasible_D", C.c_double)]


class LsTrace(C.Structure):
    _fields_ = [("cap", C.c_int32), ("op", _i32p), ("n_moves", _i32p), ("lam", _f64p),
                ("D", _f64p), ("feasible", _u8p), ("snap_cap_routes", C.c_int32), ("snap_cap_cust", C.c_int32),
                ("snap_m", _i32p), ("snap_off", _i32p), ("snap_cust", _i32p), ("snap_dep", _i32p),
                ("snap_arr", _i32p)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            subprocess.check_call(["make", "-s", "-C", _HERE])
        L = C.CDLL(path)
        L.orc_count.restype = C.c_int64
        L.orc_enumerate.restype = C.c_int64
        L.orc_evaluate.restype = C.c_int
        L.orc_leader_followers.restype = C.c_int64
        L.orc_local_search.restype = C.c_int
        L.orc_local_search_many.restype = C.c_int
        L.orc_local_search_many_out.restype = C.c_int
        L.orc_eval_all_many.restype = C.c_int64
        L.orc_repair.restype = C.c_int
        L.orc_repair_many.restype = C.c_int
        _LIB = L
    return _LIB


def _p(a, t):
    return a.ctypes.data_as(t)


INF = float("inf")


class OracleInstance:
    """Keeps the numpy arrays alive behind the borrowed C descriptor."""

    def __init__(self, inst, consts, nbr):
        self.inst = inst
        self.dist = np.ascontiguousarray(inst.dist, dtype=np.float64)
        self.time = self.dist if inst.time is inst.dist else np.ascontiguousarray(inst.time, np.float64)
        self.demand = np.ascontiguousarray(inst.demand, np.float64)
        self.service = np.ascontiguousarray(inst.service, np.float64)
        self.e = np.ascontiguousarray(inst.tw_early, np.float64)
        self.l = np.ascontiguousarray(inst.tw_late, np.float64)
        self.lists = np.ascontiguousarray(nbr.lists, np.int32)
        d = InstanceDesc()
        d.n_nodes = inst.n_nodes
        d.n_depots = inst.n_depots
        d.dist, d.time = _p(self.dist, _f64p), _p(self.time, _f64p)
        d.demand, d.service = _p(self.demand, _f64p), _p(self.service, _f64p)
        d.tw_early, d.tw_late = _p(self.e, _f64p), _p(self.l, _f64p)
        d.capacity = float(inst.capacity)
        d.max_duration = float(inst.max_duration)
        d.fleet_per_depot = float(inst.fleet_per_depot)
        d.open_routes = int(bool(inst.open_routes))
        d.has_windows = int(bool(inst.has_windows))
        d.gamma, d.theta = float(consts.gamma), float(consts.theta)
        d.lists = _p(self.lists, _i32p)
        d.width = self.lists.shape[1]
        self.desc = d


class _Flat:
    def __init__(self, sol):
        routes = sol.routes
        m = len(routes)
        self.off = np.zeros(m + 1, np.int32)
        if m:
            np.cumsum([len(r.customers) for r in routes], out=self.off[1:])
        self.cust = np.array([c for r in routes for c in r.customers] or [0], np.int32)
        self.dep = np.array([r.depart for r in routes] or [0], np.int32)
        self.arr = np.array([r.arrive for r in routes] or [0], np.int32)
        f = FlatSol()
        f.m = m
        f.off, f.cust = _p(self.off, _i32p), _p(self.cust, _i32p)
        f.depart, f.arrive = _p(self.dep, _i32p), _p(self.arr, _i32p)
        self.s = f


FIELDS = ("r1", "p1", "r2", "p2", "len1", "len2", "rev1", "rev2", "depot", "mode")


def _cands_struct(arrs):
    c = Cands()
    c.n = len(arrs["r1"])
    for f in ("r1", "p1", "r2", "p2", "len1", "len2", "depot", "mode"):
        setattr(c, f, _p(arrs[f], _i64p))
    c.rev1, c.rev2 = _p(arrs["rev1"], _u8p), _p(arrs["rev2"], _u8p)
    return c


def enumerate_op(oi: OracleInstance, sol, op: int) -> dict:
    L = lib()
    fl = _Flat(sol)
    n = L.orc_count(C.byref(oi.desc), C.byref(fl.s), C.c_int32(op))
    arrs = {f: np.zeros(max(n, 1), np.int64) for f in FIELDS if not f.startswith("rev")}
    arrs["rev1"] = np.zeros(max(n, 1), np.uint8)
    arrs["rev2"] = np.zeros(max(n, 1), np.uint8)
    cs = _cands_struct(arrs)
    got = L.orc_enumerate(C.byref(oi.desc), C.byref(fl.s), C.c_int32(op), C.byref(cs), C.c_int64(n))
    assert got == n
    out = {f: a[:n] for f, a in arrs.items()}
    out["rev1"] = out["rev1"].astype(bool)
    out["rev2"] = out["rev2"].astype(bool)
    return out


def evaluate(oi: OracleInstance, sol, op: int, cands: dict, lam) -> dict:
    L = lib()
    fl = _Flat(sol)
    n = len(cands["r1"])
    arrs = {f: np.ascontiguousarray(cands[f], np.int64) for f in FIELDS if not f.startswith("rev")}
    arrs["rev1"] = np.ascontiguousarray(cands["rev1"], np.uint8)
    arrs["rev2"] = np.ascontiguousarray(cands["rev2"], np.uint8)
    for k in arrs:
        if len(arrs[k]) == 0:
            arrs[k] = np.zeros(1, arrs[k].dtype)
    cs = _cands_struct(arrs)
    cs.n = n
    out = {f: np.zeros(max(n, 1)) for f in ("dD", "dV1", "dV2", "dV3", "dV4", "dF")}
    out["fleet_neutral"] = np.zeros(max(n, 1), np.uint8)
    d = Deltas()
    for f in ("dD", "dV1", "dV2", "dV3", "dV4", "dF"):
        setattr(d, f, _p(out[f], _f64p))
    d.fleet_neutral = _p(out["fleet_neutral"], _u8p)
    lam_a = np.ascontiguousarray(lam, np.float64)
    rc = L.orc_evaluate(C.byref(oi.desc), C.byref(fl.s), C.c_int32(op), C.byref(cs),
                        _p(lam_a, _f64p), C.byref(d))
    if rc:
        raise ValueError(f"unknown operator {op}")
    res = {f: a[:n] for f, a in out.items()}
    res["fleet_neutral"] = res["fleet_neutral"].astype(bool)
    return res


def leader_followers(cands: dict, deltas: dict, multi_move: bool):
    L = lib()
    n = len(cands["r1"])
    if n == 0:
        return -1, np.zeros(0, np.int64)
    arrs = {f: np.ascontiguousarray(cands[f], np.int64) for f in FIELDS if not f.startswith("rev")}
    arrs["rev1"] = np.ascontiguousarray(cands["rev1"], np.uint8)
    arrs["rev2"] = np.ascontiguousarray(cands["rev2"], np.uint8)
    cs = _cands_struct(arrs)
    dd = {f: np.ascontiguousarray(deltas[f], np.float64) for f in ("dD", "dV1", "dV2", "dV3", "dV4", "dF")}
    fn = np.ascontiguousarray(deltas["fleet_neutral"], np.uint8)
    d = Deltas()
    for f, a in dd.items():
        setattr(d, f, _p(a, _f64p))
    d.fleet_neutral = _p(fn, _u8p)
    fol = np.zeros(n, np.int64)
    nf = C.c_int64(0)
    best = L.orc_leader_followers(C.byref(cs), C.byref(d), C.c_int32(int(multi_move)),
                                  _p(fol, _i64p), C.byref(nf))
    return int(best), fol[:nf.value]


def totals(oi: OracleInstance, sol):
    fl = _Flat(sol)
    out = np.zeros(5)
    lib().orc_totals(C.byref(oi.desc), C.byref(fl.s), _p(out, _f64p))
    return tuple(float(x) for x in out)


def _cfg(depth, multi_move, kappa, lam_min, lam_max, perms):
    perms = np.ascontiguousarray(perms, np.int32)
    c = LsCfg()
    c.depth, c.multi_move = int(depth), int(bool(multi_move))
    c.kappa, c.lam_min, c.lam_max = float(kappa), float(lam_min), float(lam_max)
    c.max_passes, c.n_ops = perms.shape[0], perms.shape[1]
    c.perms = _p(perms, _i32p)
    return c, perms


def local_search(oi: OracleInstance, sol, lam, depth, multi_move, kappa, lam_min, lam_max,
                 perms, trace_cap=0, snapshot=False):
    """Returns (routes as (depart, arrive, customers) list, lam, stats dict, trace dict)."""
    L = lib()
    fl = _Flat(sol)
    cfg, perms_keep = _cfg(depth, multi_move, kappa, lam_min, lam_max, perms)
    lam_a = np.ascontiguousarray(lam, np.float64).copy()
    ncust = int(fl.off[-1]) + 1
    cap_r = len(sol.routes) * 4 + 64 + ncust
    out_m = C.c_int32(0)
    off = np.zeros(cap_r + 1, np.int32)
    cust = np.zeros(ncust, np.int32)
    dep = np.zeros(cap_r, np.int32)
    arr = np.zeros(cap_r, np.int32)
    st = LsStats()
    tr = None
    tarr = None
    if trace_cap or snapshot:
        tc = max(trace_cap, 1)
        tarr = dict(op=np.zeros(tc, np.int32), n_moves=np.zeros(tc, np.int32),
                    lam=np.zeros(tc * 4), D=np.zeros(tc),
                    feasible=np.zeros(tc, np.uint8))
        tr = LsTrace()
        tr.cap = trace_cap
        tr.op, tr.n_moves = _p(tarr["op"], _i32p), _p(tarr["n_moves"], _i32p)
        tr.lam, tr.D = _p(tarr["lam"], _f64p), _p(tarr["D"], _f64p)
        tr.feasible = _p(tarr["feasible"], _u8p)
        if snapshot:
            sm = np.zeros(1, np.int32)
            so, sc = np.zeros(cap_r + 1, np.int32), np.zeros(ncust, np.int32)
            sd, sa = np.zeros(cap_r, np.int32), np.zeros(cap_r, np.int32)
            tarr.update(snap_m=sm, snap_off=so, snap_cust=sc, snap_dep=sd, snap_arr=sa)
            tr.snap_cap_routes, tr.snap_cap_cust = cap_r, ncust
            tr.snap_m, tr.snap_off, tr.snap_cust = _p(sm, _i32p), _p(so, _i32p), _p(sc, _i32p)
            tr.snap_dep, tr.snap_arr = _p(sd, _i32p), _p(sa, _i32p)
    rc = L.orc_local_search(C.byref(oi.desc), C.byref(fl.s), _p(lam_a, _f64p), C.byref(cfg),
                            C.c_int32(cap_r), C.c_int32(ncust), C.byref(out_m), _p(off, _i32p),
                            _p(cust, _i32p), _p(dep, _i32p), _p(arr, _i32p), C.byref(st),
                            C.byref(tr) if tr is not None else None)
    if rc == 2:
        raise ValueError("conflicting moves: route sets intersect")
    if rc not in (0,):
        raise RuntimeError(f"oracle local_search status {rc}")
    m = out_m.value
    routes = [(int(dep[r]), int(arr[r]), [int(c) for c in cust[off[r]:off[r + 1]]]) for r in range(m)]
    stats = dict(passes=st.passes, accepted=st.accepted, op_evals=st.op_evals,
                 cands=list(st.cands), moves_applied=st.moves_applied,
                 n_feasible=st.n_feasible, best_feasible_D=st.best_feasible_D)
    trace = None
    if tarr is not None:
        k = min(st.accepted, trace_cap)
        trace = dict(op=tarr["op"][:k], n_moves=tarr["n_moves"][:k],
                     lam=tarr["lam"][:4 * k].reshape(k, 4), D=tarr["D"][:k],
                     feasible=tarr["feasible"][:k].astype(bool))
        if snapshot:
            m = int(tarr["snap_m"][0])
            so, sc = tarr["snap_off"], tarr["snap_cust"]
            trace["best_feasible"] = None if m < 0 else [
                (int(tarr["snap_dep"][r]), int(tarr["snap_arr"][r]), [int(c) for c in sc[so[r]:so[r + 1]]])
                for r in range(m)]
    return routes, [float(x) for x in lam_a], stats, trace


def local_search_many(oi: OracleInstance, sols, lams, depth, multi_move, kappa, lam_min, lam_max,
                      perms_list, nthreads):
    """Independent descents on nthreads threads; returns list of stats dicts."""
    L = lib()
    B = len(sols)
    flats = [_Flat(s) for s in sols]
    FS = (FlatSol * B)(*[f.s for f in flats])
    cfgs_keep = [_cfg(depth, multi_move, kappa, lam_min, lam_max, p) for p in perms_list]
    CF = (LsCfg * B)(*[c for c, _ in cfgs_keep])
    lam_a = np.ascontiguousarray(np.asarray(lams, np.float64).reshape(B, 4)).copy()
    ST = (LsStats * B)()
    L.orc_local_search_many(C.byref(oi.desc), C.c_int32(B), FS, _p(lam_a, _f64p), CF,
                            C.c_int32(nthreads), ST)
    return [dict(passes=s.passes, accepted=s.accepted, op_evals=s.op_evals, cands=list(s.cands),
                 status=s.status) for s in ST]


class SolOut(C.Structure):
    _fields_ = [("cap_routes", C.c_int32), ("cap_cust", C.c_int32), ("m", C.c_int32), ("status", C.c_int32),
                ("off", _i32p), ("cust", _i32p), ("depart", _i32p), ("arrive", _i32p)]


def local_search_many_routes(oi: OracleInstance, sols, lams, depth, multi_move, kappa, lam_min, lam_max,
                             perms_list, nthreads):
    """local_search_many that also returns each individual's final routes and
    penalties: [(routes, lam, stats)] in input order."""
    L = lib()
    B = len(sols)
    flats = [_Flat(s) for s in sols]
    FS = (FlatSol * B)(*[f.s for f in flats])
    cfgs_keep = [_cfg(depth, multi_move, kappa, lam_min, lam_max, p) for p in perms_list]
    CF = (LsCfg * B)(*[c for c, _ in cfgs_keep])
    lam_a = np.ascontiguousarray(np.asarray(lams, np.float64).reshape(B, 4)).copy()
    ST = (LsStats * B)()
    OUT = (SolOut * B)()
    keep = []
    for b, s in enumerate(sols):
        nc = sum(len(r.customers) for r in s.routes) + 1
        cap_r = len(s.routes) * 4 + 64 + nc
        bufs = (np.zeros(cap_r + 1, np.int32), np.zeros(nc, np.int32), np.zeros(cap_r, np.int32),
                np.zeros(cap_r, np.int32))
        keep.append(bufs)
        o = OUT[b]
        o.cap_routes, o.cap_cust = cap_r, nc
        o.off, o.cust, o.depart, o.arrive = (_p(a, _i32p) for a in bufs)
    rc = L.orc_local_search_many_out(C.byref(oi.desc), C.c_int32(B), FS, _p(lam_a, _f64p), CF,
                                     C.c_int32(nthreads), ST, OUT)
    if rc:
        raise RuntimeError(f"oracle local_search_many_out status {rc}")
    res = []
    for b in range(B):
        off, cust, dep, arr = keep[b]
        m = OUT[b].m
        routes = [(int(dep[r]), int(arr[r]), [int(c) for c in cust[off[r]:off[r + 1]]]) for r in range(m)]
        s = ST[b]
        res.append((routes, [float(x) for x in lam_a[b]],
                    dict(passes=s.passes, accepted=s.accepted, op_evals=s.op_evals, cands=list(s.cands),
                         status=s.status)))
    return res


def eval_all_many(oi: OracleInstance, sols, lams, nthreads):
    L = lib()
    B = len(sols)
    flats = [_Flat(s) for s in sols]
    FS = (FlatSol * B)(*[f.s for f in flats])
    lam_a = np.ascontiguousarray(np.asarray(lams, np.float64).reshape(B, 4))
    chk = C.c_double(0)
    n = L.orc_eval_all_many(C.byref(oi.desc), C.c_int32(B), FS, _p(lam_a, _f64p),
                            C.c_int32(nthreads), C.byref(chk))
    return int(n), chk.value


REPAIR_OPS = {"FBI": 0, "IBI": 1, "FRI": 2, "IRI": 3}


def repair(oi: OracleInstance, sol, unrouted, op: int, lam):
    """genetic.repair_insert (op 0..3) -> (routes as (depart, arrive, customers), slot_evals)."""
    L = lib()
    fl = _Flat(sol)
    pend = np.ascontiguousarray(list(unrouted) or [0], np.int32)
    npend = len(unrouted)
    lam_a = np.ascontiguousarray(lam, np.float64)
    nc = int(fl.off[-1]) + npend + 1
    cap_r = len(sol.routes) + npend + 1
    out_m = C.c_int32(0)
    off = np.zeros(cap_r + 1, np.int32)
    cust = np.zeros(nc, np.int32)
    dep = np.zeros(cap_r, np.int32)
    arr = np.zeros(cap_r, np.int32)
    ev = C.c_int64(0)
    rc = L.orc_repair(C.byref(oi.desc), C.byref(fl.s), _p(pend, _i32p), C.c_int32(npend), C.c_int32(op),
                      _p(lam_a, _f64p), C.c_int32(cap_r), C.c_int32(nc), C.byref(out_m), _p(off, _i32p),
                      _p(cust, _i32p), _p(dep, _i32p), _p(arr, _i32p), C.byref(ev))
    if rc == 1:
        raise ValueError("unknown insertion operator")
    if rc:
        raise RuntimeError(f"oracle repair status {rc}")
    m = out_m.value
    return [(int(dep[r]), int(arr[r]), [int(c) for c in cust[off[r]:off[r + 1]]]) for r in range(m)], ev.value


def repair_many(oi: OracleInstance, sols, unrouteds, op: int, lams, nthreads):
    """Independent repairs on nthreads threads; returns total slot evaluations."""
    L = lib()
    B = len(sols)
    flats = [_Flat(s) for s in sols]
    FS = (FlatSol * B)(*[f.s for f in flats])
    off = np.zeros(B + 1, np.int32)
    np.cumsum([len(u) for u in unrouteds], out=off[1:])
    pend = np.ascontiguousarray([c for u in unrouteds for c in u] or [0], np.int32)
    lam_a = np.ascontiguousarray(np.asarray(lams, np.float64).reshape(B, 4))
    ev = np.zeros(B, np.int64)
    st = np.zeros(B, np.int32)
    L.orc_repair_many(C.byref(oi.desc), C.c_int32(B), FS, _p(off, _i32p), _p(pend, _i32p), C.c_int32(op),
                      _p(lam_a, _f64p), C.c_int32(nthreads), _p(ev, _i64p), _p(st, _i32p))
    if st.any():
        raise RuntimeError(f"oracle repair_many status {st.max()}")
    return int(ev.sum())
