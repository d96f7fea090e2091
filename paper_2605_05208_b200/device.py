"""Device-resident instance and population handles (libmdr_sm100 C-ABI).

`DeviceInstance` uploads an instance once per GPU: distance/time matrix,
node attributes, fleet/capacity/duration scalars, Gamma/Theta and the
granular neighbour lists (mdr_instance_create).  `Population` owns B
individuals' route storage and subsequence tables on that GPU
(mdr_pop_create / upload / download) and runs the batched local search.
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from ._lib import (Cands, CapacityError, Deltas, InstanceDesc, LsCfg, LsStats, Timing, check, f64p, i32p,
                   i64p, ptr, u8p)


def _cur_stream(device: int):
    """Handle of torch's current stream on `device` (0 = legacy default)."""
    try:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    except Exception:  # torch optional for plain C-ABI users
        pass
    return C.c_void_p(0)


class DeviceInstance:
    def __init__(self, inst, consts, nbr=None, device: int = 0):
        L = _lib.lib()
        self.device = device
        self.n_nodes = int(inst.n_nodes)
        self.n_depots = int(inst.n_depots)
        self.has_windows = bool(inst.has_windows)
        self.open_routes = bool(inst.open_routes)
        self._dist = np.ascontiguousarray(inst.dist, dtype=np.float64)
        same = inst.time is inst.dist
        self._time = self._dist if same else np.ascontiguousarray(inst.time, dtype=np.float64)
        self._demand = np.ascontiguousarray(inst.demand, np.float64)
        self._service = np.ascontiguousarray(inst.service, np.float64)
        self._e = np.ascontiguousarray(inst.tw_early, np.float64)
        self._l = np.ascontiguousarray(inst.tw_late, np.float64)
        if nbr is not None:
            self._lists = np.ascontiguousarray(nbr.lists, np.int32)
        else:
            self._lists = np.full((self.n_nodes, 1), -1, np.int32)
        self.width = int(self._lists.shape[1])
        d = InstanceDesc()
        d.n_nodes, d.n_depots = self.n_nodes, self.n_depots
        d.dist, d.time = ptr(self._dist, f64p), ptr(self._time, f64p)
        d.demand, d.service = ptr(self._demand, f64p), ptr(self._service, f64p)
        d.tw_early, d.tw_late = ptr(self._e, f64p), ptr(self._l, f64p)
        d.capacity = float(inst.capacity)
        d.max_duration = float(inst.max_duration)
        d.fleet_per_depot = float(inst.fleet_per_depot)
        d.open_routes, d.has_windows = int(self.open_routes), int(self.has_windows)
        d.gamma, d.theta = float(consts.gamma), float(consts.theta)
        d.lists, d.width = ptr(self._lists, i32p), self.width
        h = C.c_void_p()
        check(L.mdr_instance_create(C.byref(d), device, C.byref(h)), "mdr_instance_create")
        self.handle = h
        self._fin = weakref.finalize(self, L.mdr_instance_destroy, h)


def flatten_population(sols):
    """B solutions -> (rbase, coff, cust, dep, arr) int32 arrays."""
    rb = [0]
    coff = [0]
    cust, dep, arr = [], [], []
    ext, cap, dap, aap = cust.extend, coff.append, dep.append, arr.append
    for s in sols:
        for r in s.routes:
            ext(r.customers)
            cap(len(cust))
            dap(r.depart)
            aap(r.arrive)
        rb.append(len(dep))
    f = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.int32).reshape(-1)) if len(x) else np.zeros(1, np.int32)
    return (np.asarray(rb, np.int32), np.asarray(coff, np.int32), f(cust), f(dep), f(arr))


class Population:
    """B individuals resident on one GPU."""

    def __init__(self, dinst: DeviceInstance, B_cap: int, J_cap: int, K_cap: int, F_cap: int = 1 << 15):
        L = _lib.lib()
        self.dinst = dinst
        self.B_cap, self.J_cap, self.K_cap, self.F_cap = B_cap, J_cap, K_cap, F_cap
        h = C.c_void_p()
        check(L.mdr_pop_create(dinst.handle, B_cap, J_cap, K_cap, F_cap, C.byref(h)), "mdr_pop_create")
        self.handle = h
        self._fin = weakref.finalize(self, L.mdr_pop_destroy, h)
        self.B = 0
        self.n_cust = 0

    @staticmethod
    def caps_for(sols, inst):
        m = max((len(s.routes) for s in sols), default=1)
        k = max((len(r.customers) for s in sols for r in s.routes), default=1)
        J = min(4094, max(2 * m, m + 64))
        K = min(500, max(2 * k, k + 16, 32))
        return J, K

    def upload(self, sols, lams, stream=None):
        rbase, coff, cust, dep, arr = flatten_population(sols)
        lam = np.ascontiguousarray(np.asarray(lams, np.float64).reshape(-1, 4))
        B = len(sols)
        s = stream if stream is not None else _cur_stream(self.dinst.device)
        check(_lib.lib().mdr_pop_upload(self.handle, B, ptr(rbase, i32p), ptr(coff, i32p), ptr(cust, i32p),
                                        ptr(dep, i32p), ptr(arr, i32p), ptr(lam, f64p), s), "mdr_pop_upload")
        self.B = B
        self.n_cust = int(coff[-1])
        self.h2d_bytes = sum(a.nbytes for a in (rbase, coff, cust, dep, arr, lam))

    def _download(self, best: bool, stream=None):
        B = self.B
        cap_r = B * self.J_cap
        cap_c = max(self.n_cust, 1) + 16
        rbase = np.zeros(B + 1, np.int32)
        coff = np.zeros(cap_r + 1, np.int32)
        cust = np.zeros(cap_c, np.int32)
        dep = np.zeros(max(cap_r, 1), np.int32)
        arr = np.zeros(max(cap_r, 1), np.int32)
        nr, nc = C.c_int32(cap_r), C.c_int32(cap_c)
        s = stream if stream is not None else _cur_stream(self.dinst.device)
        L = _lib.lib()
        if best:
            extra = np.zeros(max(B, 1), np.float64)
            rc = L.mdr_pop_download_best(self.handle, ptr(rbase, i32p), ptr(coff, i32p), ptr(cust, i32p),
                                         ptr(dep, i32p), ptr(arr, i32p), ptr(extra, f64p), C.byref(nr),
                                         C.byref(nc), s)
        else:
            extra = np.zeros(max(B, 1) * 4, np.float64)
            rc = L.mdr_pop_download(self.handle, ptr(rbase, i32p), ptr(coff, i32p), ptr(cust, i32p),
                                    ptr(dep, i32p), ptr(arr, i32p), ptr(extra, f64p), C.byref(nr), C.byref(nc), s)
        check(rc, "mdr_pop_download")
        self.d2h_bytes = int(rbase.nbytes + 4 * (nr.value + 1) + 4 * nc.value + 8 * nr.value + extra.nbytes)
        R = int(rbase[B]) if B else 0
        cl, ol = cust[:int(coff[R])].tolist(), coff[:R + 1].tolist()
        dl, al, bl = dep[:R].tolist(), arr[:R].tolist(), rbase.tolist()
        out = [[(dl[r], al[r], cl[ol[r]:ol[r + 1]]) for r in range(bl[b], bl[b + 1])] for b in range(B)]
        return out, extra

    def download(self, stream=None):
        """[(depart, arrive, customers)] per individual, lam [B,4]."""
        routes, lam = self._download(False, stream)
        return routes, lam.reshape(-1, 4)[:self.B]

    def download_range(self, b0: int, nb: int, stream=None):
        """Routes of individuals b0 .. b0+nb-1 only (mdr_pop_download_range)."""
        cap_r = max(nb * self.J_cap, 1)
        cap_c = max(self.n_cust, 1) + 16
        rbase = np.zeros(nb + 1, np.int32)
        coff = np.zeros(cap_r + 1, np.int32)
        cust = np.zeros(cap_c, np.int32)
        dep = np.zeros(cap_r, np.int32)
        arr = np.zeros(cap_r, np.int32)
        nr, nc = C.c_int32(cap_r), C.c_int32(cap_c)
        s = stream if stream is not None else _cur_stream(self.dinst.device)
        check(_lib.lib().mdr_pop_download_range(self.handle, b0, nb, ptr(rbase, i32p), ptr(coff, i32p),
                                                ptr(cust, i32p), ptr(dep, i32p), ptr(arr, i32p), C.byref(nr),
                                                C.byref(nc), s), "mdr_pop_download_range")
        cl, ol, dl, al = cust.tolist(), coff.tolist(), dep.tolist(), arr.tolist()
        return [[(dl[r], al[r], cl[ol[r]:ol[r + 1]]) for r in range(rbase[b], rbase[b + 1])] for b in range(nb)]

    def breakdowns(self, lams=None, stream=None) -> np.ndarray:
        """[B, 6] {D, V1, V2, V3, V4, F} of the uploaded individuals, computed on the
        device with evaluation.evaluate's scalar semantics (mdr_pop_breakdown)."""
        out = np.zeros((max(self.B, 1), 6), np.float64)
        lam = None if lams is None else np.ascontiguousarray(np.asarray(lams, np.float64).reshape(-1, 4))
        s = stream if stream is not None else _cur_stream(self.dinst.device)
        check(_lib.lib().mdr_pop_breakdown(self.handle, None if lam is None else ptr(lam, f64p), ptr(out, f64p), s),
              "mdr_pop_breakdown")
        return out[:self.B]

    def download_best(self, stream=None):
        routes, bestD = self._download(True, stream)
        return routes, bestD[:self.B]

    def local_search(self, perms: np.ndarray, depth: int, multi_move: bool, kappa: float, lam_min: float,
                     lam_max: float, deadline_s: float = -1.0, rounds_per_sync: int = 0, stream=None,
                     snapshot_best: bool = False, trace: bool = False):
        """perms: uint8 [B, max_passes, n_ops]. Returns a list of per-individual stats dicts."""
        B = self.B
        perms = np.ascontiguousarray(perms, dtype=np.uint8)
        assert perms.shape[0] == B
        cfg = LsCfg()
        cfg.depth, cfg.multi_move = int(depth), int(bool(multi_move))
        cfg.kappa, cfg.lam_min, cfg.lam_max = float(kappa), float(lam_min), float(lam_max)
        cfg.max_passes, cfg.n_ops = perms.shape[1], perms.shape[2]
        cfg.perms = ptr(perms, u8p)
        cfg.deadline_s = float(deadline_s)
        cfg.rounds_per_sync = int(rounds_per_sync)
        cfg.use_graph = 0
        cfg.snapshot_best = int(bool(snapshot_best))
        cfg.trace = int(bool(trace))
        st = (LsStats * max(B, 1))()
        s = stream if stream is not None else _cur_stream(self.dinst.device)
        rc = _lib.lib().mdr_local_search(self.handle, C.byref(cfg), st, s)
        stats = [dict(passes=x.passes, accepted=x.accepted, op_evals=x.op_evals, status=x.status,
                      cands=list(x.cands), moves_applied=x.moves_applied, n_feasible=x.n_feasible,
                      n_improving=x.n_improving, best_feasible_D=x.best_feasible_D) for x in st[:B]]
        if rc == _lib.MDR_ERR_CAPACITY:
            need = dict(F=max(x.need_followers for x in st[:B]), G=max(x.need_queue for x in st[:B]),
                        J=max(x.need_routes for x in st[:B]), K=max(x.need_positions for x in st[:B]))
            try:
                check(rc, "mdr_local_search")
            except CapacityError as e:
                e.need = need
                raise
        check(rc, "mdr_local_search")
        return stats

    def repair(self, op: int, unrouteds, stream=None):
        """mdr_repair on the uploaded individuals; the population is left holding the
        repaired solutions.  Returns per-individual stats dicts."""
        B = self.B
        off = np.zeros(B + 1, np.int32)
        np.cumsum([len(u) for u in unrouteds], out=off[1:])
        pend = np.ascontiguousarray([int(c) for u in unrouteds for c in u] or [0], np.int32)
        st = (_lib.RepairStats * max(B, 1))()
        s = stream if stream is not None else _cur_stream(self.dinst.device)
        rc = _lib.lib().mdr_repair(self.handle, int(op), ptr(off, i32p), ptr(pend, i32p), st, s)
        stats = [dict(status=x.status, inserted=x.inserted, slot_evals=x.slot_evals,
                      ref_slot_evals=x.ref_slot_evals) for x in st[:B]]
        if rc == _lib.MDR_ERR_CAPACITY:
            need = dict(J=max(x.need_j for x in st[:B]), K=max(x.need_k for x in st[:B]))
            try:
                check(rc, "mdr_repair")
            except CapacityError as e:
                e.need = need
                raise
        check(rc, "mdr_repair")
        self.n_cust += int(off[-1])  # download buffers hold the inserted customers too
        self.h2d_bytes_repair = int(off.nbytes + pend.nbytes)
        return stats

    def construct(self, ooff, order, n_customers: int, stream=None):
        """mdr_construct: initial solutions of B = len(ooff)//ND individuals into this
        population; returns each individual's leftover customers."""
        B = (len(ooff) - 1) // self.dinst.n_depots
        ooff = np.ascontiguousarray(ooff, np.int32)
        order = np.ascontiguousarray(order if len(order) else [0], np.int32)
        n_left = np.zeros(max(B, 1), np.int32)
        left = np.zeros(max(B, 1) * n_customers, np.int32)
        s = stream if stream is not None else _cur_stream(self.dinst.device)
        check(_lib.lib().mdr_construct(self.handle, B, ptr(ooff, i32p), ptr(order, i32p), ptr(n_left, i32p),
                                       ptr(left, i32p), s), "mdr_construct")
        self.B = B
        self.n_cust = int(ooff[-1])
        return [left[b * n_customers: b * n_customers + n_left[b]].tolist() for b in range(B)]

    def trace(self, b: int) -> list:
        """Accepted steps of individual b's last traced descent: [(op, feasible, D, [keys])]."""
        n = C.c_int64(0)
        L = _lib.lib()
        rc = L.mdr_pop_trace(self.handle, b, None, 0, C.byref(n))
        if rc not in (_lib.MDR_OK, _lib.MDR_ERR_CAPACITY) or n.value < 0:
            check(rc, "mdr_pop_trace")
        buf = np.zeros(max(n.value, 1), np.uint64)
        check(L.mdr_pop_trace(self.handle, b, ptr(buf, C.POINTER(C.c_uint64)), buf.size, C.byref(n)), "mdr_pop_trace")
        out, at, w = [], 0, buf.tolist()
        while at < n.value:
            head = w[at]
            k = head & 0xffffffff
            D = float(np.array([w[at + 1]], np.uint64).view(np.float64)[0])
            out.append((int(head >> 56), bool((head >> 55) & 1), D, w[at + 2: at + 2 + k]))
            at += 2 + k
        return out

    def route_attrs(self, b0: int, nb: int, stream=None) -> np.ndarray:
        """[nb, J_cap, 6] route_attr {dist, load, T, E, L, TW} of every route (mdr_pop_route_attrs)."""
        out = np.zeros((max(nb, 1), self.J_cap, 6), np.float64)
        s = stream if stream is not None else _cur_stream(self.dinst.device)
        check(_lib.lib().mdr_pop_route_attrs(self.handle, b0, nb, ptr(out, f64p), s), "mdr_pop_route_attrs")
        return out[:nb]

    def info(self) -> dict:
        """Evaluator shape of this population (mdr_pop_info)."""
        out = np.zeros(4, np.int32)
        check(_lib.lib().mdr_pop_info(self.handle, ptr(out, i32p)), "mdr_pop_info")
        return dict(staged=int(out[0]), items_per_task=int(out[1]), warps_per_cta=int(out[2]), B_cap=int(out[3]))

    def set_profiling(self, on: bool):
        check(_lib.lib().mdr_set_profiling(self.handle, int(on)))

    def timing(self) -> dict:
        t = Timing()
        check(_lib.lib().mdr_get_timing(self.handle, C.byref(t)))
        out = {f: getattr(t, f) for f, _ in Timing._fields_ if f != "kern_ms"}
        # profiling pass, evaluation phase serialised: per-evaluator CUDA-event times
        for i, n in enumerate(("relocate", "relocate_intra", "swap", "swap_intra", "two_opt_star", "depot_generic")):
            out["kern_" + n + "_ms"] = t.kern_ms[i]
        return out

    # ---- operator-level -----------------------------------------------------
    def count(self, b: int, op: int) -> int:
        n = _lib.lib().mdr_count(self.handle, b, op)
        if n < 0:
            check(_lib.MDR_ERR_ARG, "mdr_count")
        return int(n)

    def enumerate(self, b: int, op: int) -> dict:
        n = self.count(b, op)
        arrs = {f: np.zeros(max(n, 1), np.int64) for f in ("r1", "p1", "r2", "p2", "len1", "len2", "depot", "mode")}
        arrs["rev1"] = np.zeros(max(n, 1), np.uint8)
        arrs["rev2"] = np.zeros(max(n, 1), np.uint8)
        cs = cands_struct(arrs, n)
        check(_lib.lib().mdr_enumerate(self.handle, b, op, C.byref(cs)), "mdr_enumerate")
        out = {f: a[:cs.n] for f, a in arrs.items()}
        out["rev1"] = out["rev1"].astype(bool)
        out["rev2"] = out["rev2"].astype(bool)
        return out

    def evaluate(self, b: int, op: int, cands: dict, lam) -> dict:
        arrs = as_cand_arrays(cands)
        n = len(arrs["r1"])
        cs = cands_struct(arrs, n)
        out = {f: np.zeros(max(n, 1)) for f in ("dD", "dV1", "dV2", "dV3", "dV4", "dF")}
        out["fleet_neutral"] = np.zeros(max(n, 1), np.uint8)
        d = deltas_struct(out)
        lam_a = np.ascontiguousarray(lam, np.float64)
        check(_lib.lib().mdr_evaluate(self.handle, b, op, C.byref(cs), ptr(lam_a, f64p), C.byref(d)),
              "mdr_evaluate")
        res = {f: a[:n] for f, a in out.items()}
        res["fleet_neutral"] = res["fleet_neutral"].astype(bool)
        return res

    def leader_followers(self, cands: dict, deltas: dict, multi_move: bool):
        arrs = as_cand_arrays(cands)
        n = len(arrs["r1"])
        cs = cands_struct(arrs, n)
        dd = {f: np.ascontiguousarray(deltas[f], np.float64) for f in ("dD", "dV1", "dV2", "dV3", "dV4", "dF")}
        dd["fleet_neutral"] = np.ascontiguousarray(deltas["fleet_neutral"], np.uint8)
        d = deltas_struct(dd)
        lead = C.c_int64(-1)
        fol = np.zeros(max(n, 1), np.int64)
        nf = C.c_int64(0)
        check(_lib.lib().mdr_leader_followers(self.handle, C.byref(cs), C.byref(d), int(bool(multi_move)),
                                              C.byref(lead), ptr(fol, i64p), C.byref(nf)), "mdr_leader_followers")
        return int(lead.value), fol[:nf.value]

    def totals(self, b: int):
        out = np.zeros(5)
        check(_lib.lib().mdr_totals(self.handle, b, ptr(out, f64p)), "mdr_totals")
        return tuple(float(x) for x in out)


CAND_FIELDS = ("r1", "p1", "r2", "p2", "len1", "len2", "rev1", "rev2", "depot", "mode")


def as_cand_arrays(cands) -> dict:
    get = (lambda f: cands[f]) if isinstance(cands, dict) else (lambda f: getattr(cands, f))
    out = {}
    for f in CAND_FIELDS:
        a = np.asarray(get(f))
        out[f] = np.ascontiguousarray(a, dtype=np.uint8 if f.startswith("rev") else np.int64)
        if out[f].size == 0:
            out[f] = np.zeros(1, out[f].dtype)[:0]
    return out


def cands_struct(arrs: dict, n: int) -> Cands:
    keep = {}
    for f, a in arrs.items():
        if a.size == 0:
            a = np.zeros(1, a.dtype)
        keep[f] = a
    cs = Cands()
    cs.n = n
    for f in ("r1", "p1", "r2", "p2", "len1", "len2", "depot", "mode"):
        setattr(cs, f, ptr(keep[f], i64p))
    cs.rev1, cs.rev2 = ptr(keep["rev1"], u8p), ptr(keep["rev2"], u8p)
    cs._keep = keep
    return cs


def deltas_struct(out: dict) -> Deltas:
    d = Deltas()
    for f in ("dD", "dV1", "dV2", "dV3", "dV4", "dF"):
        setattr(d, f, ptr(out[f], f64p))
    d.fleet_neutral = ptr(out["fleet_neutral"], u8p)
    return d
