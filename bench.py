"""Benchmark: population-batched multi-move local search on B200 (sm_100a).

Workload (BASELINE.json configs[3]): synthetic MDVRPTW,
1000 customers x 10 depots, theta = 50, population 256.  Individual i
starts from genetic.initial_solution(..., random.Random(100 + i)) and descends with
local_search(depth=500, multi_move=True, lambda=1, kappa=0.5, rng=Random(i)).

One step = one complete population descent (every individual to its local
optimum or depth 500).  Metric: move-evaluations per second (candidates
scored, duplicates included, exactly as enumerate_candidates counts them),
whole job; descents/s is reported beside it.

The population (256 at C4) is sharded over the GPUs (strong scaling, as
BASELINE.json configs[3] states); the per-step elite all_gather is inside the
timed region.  `--weak` keeps --pop individuals per GPU instead.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import random
import statistics
import subprocess
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2605_05208_b200 import workload as W  # noqa: E402
from paper_2605_05208_b200.evaluation import PenaltyState, ScalingConstants  # noqa: E402
from paper_2605_05208_b200.neighborhood import NeighborConfig, build  # noqa: E402

# algorithmic bytes per candidate (fp64 table pieces,
# node pieces, distance links, old-route terms, descriptor), inter-route
# figures for relocate/swap.  Windows (C2, C4) / no windows (C1, C3, C5).
ALG_BYTES_WIN = {0: 436, 1: 500, 2: 372, 3: 0, 4: 304, 5: 204}
ALG_BYTES_NOWIN = {0: 316, 1: 356, 2: 276, 3: 204, 4: 208, 5: 148}
# algorithmic fp64 ops (add/sub/mul/div/max/min of the
# reference DAG) per candidate, inter-route figures for relocate/swap.
ALG_FP64_WIN = {0: 111, 1: 133, 2: 89, 3: 0, 4: 106, 5: 69}
ALG_FP64_NOWIN = {0: 50, 1: 55, 2: 45, 3: 30, 4: 45, 5: 30}


def _init_one(args):
    """Host start state for the CPU reference arm: the reference's own
    genetic.initial_solution from baseline/_ref when installed, else the oracle's
    restatement of it (both pinned equal to the device construction by the tests)."""
    name, i = args
    spec = W.CONFIGS[name]
    inst, _ = W.appendix_a_instance(spec)
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isfile(os.path.join(ref, "mdroute", "genetic.py")):
        sys.path.insert(0, ref)
        from mdroute import evaluation as RE, genetic as RG, model as RM
        rinst = RM.Instance(RM.Variant(inst.variant.value),
                            [RM.Node(n.id, n.kind, n.x, n.y, n.demand, n.service, n.tw_early, n.tw_late)
                             for n in inst.nodes], inst.n_depots, inst.dist, fleet_per_depot=inst.fleet_per_depot,
                            capacity=inst.capacity, max_duration=inst.max_duration)
        s = RG.initial_solution(rinst, RE.ScalingConstants.from_instance(rinst), RE.PenaltyState(),
                                random.Random(100 + i))
    else:
        from oracle import initial_ref
        s = initial_ref.initial_solution(inst, ScalingConstants.from_instance(inst), PenaltyState(),
                                         random.Random(100 + i))
    return [(r.depart, r.arrive, list(r.customers)) for r in s.routes]


def make_workload(name, ids, host=False, device=0):
    """Instance, constants, lists and the start states of individuals `ids`
    (initial_solution(..., Random(100+i))): built on the device in one batch
    (genetic.initial_solutions), or on the host cores for the CPU reference arm."""
    spec = W.CONFIGS[name]
    inst, _ = W.appendix_a_instance(spec)
    consts = ScalingConstants.from_instance(inst)
    nbr = build(inst, NeighborConfig(spec.theta), consts)
    from paper_2605_05208_b200.model import Route, Solution
    if not host:
        from paper_2605_05208_b200.genetic import initial_solutions
        return spec, inst, consts, nbr, initial_solutions(inst, consts, PenaltyState(),
                                                          [random.Random(100 + i) for i in ids], device)
    import multiprocessing as mp
    workers = max(1, min(len(ids), (os.cpu_count() or 2) - 1, 64))
    with ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn")) as ex:
        raw = list(ex.map(_init_one, [(name, i) for i in ids], chunksize=1))
    sols = [Solution([Route(d, a, c) for d, a, c in rs]) for rs in raw]
    return spec, inst, consts, nbr, sols


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, gpu: int):
        self.path = f"/tmp/mdr_clocks_{os.getpid()}.csv"
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sms:
            return None
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


def flush_l2(torch, dev):
    buf = torch.empty(64 << 22, dtype=torch.float32, device=dev)  # 1 GiB > 126 MB L2
    buf.fill_(1.0)
    del buf


def measure_l2_gbs(device, mib=32, iters=200):
    """L2 read bandwidth (native probe: L1-bypassing loads over a 32 MiB
    L2-resident buffer) -- the on-chip denominator next to the HBM one."""
    from paper_2605_05208_b200 import _lib
    out = ctypes.c_double(0.0)
    _lib.check(_lib.lib().mdr_probe_l2_gbs(device, mib << 20, iters, ctypes.byref(out)), "mdr_probe_l2_gbs")
    return out.value


def measure_fp64_gops(device, iters=4096):
    """fp64 dadd/dmul issue rate (native probe, FMA contraction off)."""
    from paper_2605_05208_b200 import _lib
    out = ctypes.c_double(0.0)
    _lib.check(_lib.lib().mdr_probe_fp64_gops(device, iters, ctypes.byref(out)), "mdr_probe_fp64_gops")
    return out.value


def repair_workload(sols, ids, frac=0.2):
    """GA-offspring-like repair inputs: individual i = its start with a seeded
    `frac` of its customers removed (emptied routes kept)."""
    out, pend = [], []
    for s, i in zip(sols, ids):
        rng = random.Random(7000 + i)
        c = s.clone()
        cust = [x for r in c.routes for x in r.customers]
        removed = set(rng.sample(cust, int(len(cust) * frac)))
        for r in c.routes:
            r.customers = [x for x in r.customers if x not in removed]
        out.append(c)
        pend.append(sorted(removed))
    return out, pend


def bench_repair(name, inst, consts, sols, ids, device, steps, cpu=True, op=3):
    """batched repair insertion (IRI by default) of the
    population; slot evaluations counted as the reference's full re-scan does."""
    import torch
    from paper_2605_05208_b200.device import Population
    from paper_2605_05208_b200.genetic import InsertionOperator, repair_population
    from paper_2605_05208_b200.session import session_for
    rs, pend = repair_workload(sols, ids)
    lams = [[1.0] * 4] * len(rs)
    sess = session_for(inst, consts, None, device)
    J, K = Population.caps_for(rs, inst)
    pop = Population(sess.dinst, len(rs), min(4094, J + max(len(u) for u in pend)), min(500, K + 32), 1 << 10)
    dev_ms, ref_ev, dev_ev = [], 0, 0
    for k in range(steps + 1):
        pop.upload(rs, lams)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = pop.repair(op, pend)
        torch.cuda.synchronize()
        if k:  # first call: warm-up (scratch allocation)
            dev_ms.append(1000 * (time.perf_counter() - t0))
            ref_ev += sum(x["ref_slot_evals"] for x in st)
            dev_ev += sum(x["slot_evals"] for x in st)
    ms = sum(dev_ms) / len(dev_ms)
    e2e = []
    for k in range(2):  # first call allocates the session's population (warm-up)
        work = [s.clone() for s in rs]
        t0 = time.perf_counter()
        repair_population(work, pend, InsertionOperator(op), inst, consts,
                          [PenaltyState() for _ in rs], device=device)
        e2e.append(1000 * (time.perf_counter() - t0))
    e2e_ms = e2e[-1]
    line = {"op": InsertionOperator(op).name, "individuals": len(rs),
            "pending_per_individual": sum(len(u) for u in pend) / len(pend),
            "device_call_ms": ms, "e2e_ms": e2e_ms, "repairs_per_s": len(rs) / (ms / 1000.0),
            "ref_slot_evals_per_s": ref_ev / steps / (ms / 1000.0),
            "device_slot_evals_per_repair": dev_ev / steps / len(rs),
            "ref_slot_evals_per_repair": ref_ev / steps / len(rs)}
    if cpu:
        from oracle import oracle as O
        threads = os.cpu_count() or 1
        k = min(len(rs), threads)
        oi = O.OracleInstance(inst, consts, build(inst, NeighborConfig(1), consts))
        t0 = time.perf_counter()
        ev = O.repair_many(oi, rs[:k], pend[:k], op, [[1.0] * 4] * k, threads)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"repairs_per_s": k / dt, "ref_slot_evals_per_s": ev / dt, "cores": min(k, threads),
                                "kind": "port", "sample": f"{k} repairs on {threads} threads, {dt:.1f} s"}
    return line


def eval_only_line(name, inst, consts, nbr, sols, cands, eval_s, cpu=True):
    line = {"value": cands / eval_s, "unit": "move-evals/s",
            "how": "profiled step: candidates / evaluation-phase time (evaluators serialised, CUDA events)"}
    if cpu:
        from oracle import oracle as O
        threads = os.cpu_count() or 1
        k = len(sols)
        oi = O.OracleInstance(inst, consts, nbr)
        t0 = time.perf_counter()
        n, _ = O.eval_all_many(oi, sols[:k], [[1.0] * 4] * k, threads)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n / dt, "unit": "move-evals/s", "cores": min(k, threads), "kind": "port",
                                "sample": f"all operators of {k} start states on {threads} threads, {dt:.1f} s"}
    return line


def cpu_info():
    model, phys = None, set()
    try:
        cur = {}
        for line in open("/proc/cpuinfo"):
            if ":" not in line:
                if cur:
                    phys.add((cur.get("physical id"), cur.get("core id")))
                cur = {}
                continue
            k, v = (x.strip() for x in line.split(":", 1))
            cur[k] = v
            if k == "model name" and model is None:
                model = v
        if cur:
            phys.add((cur.get("physical id"), cur.get("core id")))
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "physical_cores": len(phys) or None}


def python_permutations(rng, ops, n_passes):
    """The first n_passes `rng.shuffle(order)` results of localsearch.py:110-113,
    drawn with CPython's own random.shuffle on a copy of rng (pure Python; the
    reference arm never maps this repo's library)."""
    r = random.Random()
    r.setstate(rng.getstate())
    out = np.empty((n_passes, len(ops)), np.uint8)
    for p in range(n_passes):
        order = list(ops)
        r.shuffle(order)
        out[p] = [int(o) for o in order]
    return out


def workload_config(name, spec, total, depth):
    """The `config` block -- identical for both arms and every N (strong scaling)."""
    return {"workload": f"{name}: synthetic {spec.variant.value} {spec.n_customers} customers x {spec.n_depots} "
                        f"depots, theta {spec.theta}, population {total} (Appendix-A start states "
                        f"initial_solution(Random(100+i)), LS rng Random(i)) sharded over the GPUs; one step = all "
                        f"{total} descents to their local optimum (depth {depth}, multi-move, lambda 1, kappa 0.5)",
            "population": total, "depth": depth, "multi_move": True,
            "l2": "flushed (1 GiB write) between timed steps"}


def cpu_baseline(name, inst, consts, nbr, sols, ids, depth):
    """Oracle (C port of the reference) descents on all host threads, bounded sample;
    also returns the final routes so the timed device results can be checked."""
    from oracle import oracle as O
    from paper_2605_05208_b200.localsearch import enabled_operators
    oi = O.OracleInstance(inst, consts, nbr)
    ops = enabled_operators(inst)
    threads = os.cpu_count() or 1
    k = min(len(sols), threads)
    perms = [python_permutations(random.Random(i), ops, depth + 1) for i in ids[:k]]
    t0 = time.perf_counter()
    res = O.local_search_many_routes(oi, sols[:k], [[1.0] * 4] * k, depth, True, 0.5, 0.01, 1e4, perms, threads)
    dt = time.perf_counter() - t0
    cands = sum(sum(st["cands"]) for _, _, st in res)
    line = {"value": cands / dt, "unit": "move-evals/s", "cores": min(k, threads), "kind": "port",
            "sample": f"{k} complete {name} descents (individuals {ids[0]}..{ids[k-1]}, depth {depth}, multi-move) "
                      f"of the C oracle (scalar C restatement of the reference) on {min(k, threads)} host threads, "
                      f"{dt:.1f} s, {cands} candidates",
            "descents_per_s": k / dt}
    line.update(cpu_info())
    return line, res


def numpy_reference_leg(inst, spec, sols, ids, depth, seconds=15.0):
    """The unmodified numpy reference (baseline/_ref) timed on the host cores."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import numpy_ref
    if not numpy_ref.available():
        return {"unavailable": "baseline/_ref/mdroute not installed (baseline/install_reference.sh)"}
    try:
        line = numpy_ref.leg(inst, spec.theta, sols, ids, depth, seconds)
    except Exception as e:  # reported, never fatal for the GPU arm
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    line.update(cpu_info())
    return line


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU local search on the box's host cores.

    The reference is Python/numpy; its arm here is the C oracle port of it
    (oracle/, pinned bit-exactly to the reference) on all host threads: 16
    complete descents of the config's start states per step (a bounded sample
    of the population).  The unmodified numpy reference from baseline/_ref is
    timed beside it (`cpu_baseline_numpy`).  Rank 0 only; pure host code (the
    operator-order permutations come from CPython's random.shuffle)."""
    if rank != 0:
        return
    name = args.config
    spec = W.CONFIGS[name]
    total = args.pop or spec.population
    threads = os.cpu_count() or 1
    ids = list(range(min(threads, total)))
    spec, inst, consts, nbr, sols = make_workload(name, ids, host=True)
    from oracle import oracle as O
    from paper_2605_05208_b200.localsearch import enabled_operators
    oi = O.OracleInstance(inst, consts, nbr)
    ops = enabled_operators(inst)
    perms = [python_permutations(random.Random(i), ops, args.depth + 1) for i in ids]

    def step(depth=args.depth):
        t0 = time.perf_counter()
        st = O.local_search_many(oi, sols, [[1.0] * 4] * len(sols), depth, True, 0.5, 0.01, 1e4, perms,
                                 threads)
        return time.perf_counter() - t0, sum(sum(s["cands"]) for s in st)

    for _ in range(args.warmup):
        step(depth=10)  # untimed warm-up (page-in, thread start-up); kept short on the CPU
    tt, cc = 0.0, 0
    for _ in range(args.steps):
        dt, c = step()
        tt += dt
        cc += c
    v = cc / tt
    cpu = {"value": v, "unit": "move-evals/s", "cores": min(len(sols), threads), "kind": "port",
           "sample": f"per step {len(sols)} complete descents (individuals 0..{len(sols)-1} of the population "
                     f"of {total}, depth {args.depth}, multi-move) of the C oracle port on {threads} host threads"}
    cpu.update(cpu_info())
    line = {"impl": "reference", "metric": "move_evals_per_s", "value": v, "unit": "move-evals/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * tt / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(name, spec, total, args.depth),
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": "move-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "descents_per_s": len(sols) * args.steps / tt}
    if not args.no_numpy_ref:
        line["cpu_baseline_numpy"] = numpy_reference_leg(inst, spec, sols, ids, args.depth)
    print(json.dumps(line), flush=True)


def load_ncu(name, evaluator="relocate"):
    """ncu roofs of a config's evaluator from the committed captures
    (profiles/ncu_roofline.json, written by tools/ncu_roofline.py).  An
    evaluator launched as several kernels (relocate's granular and boundary
    families) gets the duration-weighted mean of their roofs."""
    try:
        allj = json.load(open(os.path.join(ROOT, "profiles", "ncu_roofline.json"))).get(name) or {}
    except Exception:
        return None
    parts = [v for k, v in allj.items() if k == evaluator or k.startswith(evaluator + "_")]
    if not parts:
        return None
    if len(parts) == 1:
        return parts[0]
    w = [p["metrics"].get("duration_ns") or 1.0 for p in parts]
    roofs = {k: sum(p["roofs"].get(k, 0.0) * x for p, x in zip(parts, w)) / sum(w) for k in parts[0]["roofs"]}
    binding = max(roofs, key=roofs.get)
    traffic = sum(p.get("dram_bytes_per_launch") or 0.0 for p in parts)
    return {"binding": binding, "achieved": roofs[binding], "peak": 1.0, "frac": roofs[binding],
            "unit": "fraction of the ncu peak of that unit (duration-weighted over the evaluator's kernels)",
            "roofs": roofs, "dram_bytes_per_launch": traffic, "kernel": " + ".join(p["kernel"] for p in parts),
            "metrics": {"parts": [p["metrics"] for p in parts]}, "source": parts[0]["source"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--pop", type=int, default=None,
                    help="total population, sharded over the GPUs (default: the config's)")
    ap.add_argument("--weak", action="store_true", help="--pop individuals per GPU instead (weak scaling)")
    ap.add_argument("--depth", type=int, default=500)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-numpy-ref", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-repair", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    backend = os.environ.get("MDR_BENCH_BACKEND", "nccl")  # "gloo": functional dry run of the N>1 flow
    if backend != "nccl":
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    import paper_2605_05208_b200 as P
    from paper_2605_05208_b200.device import DeviceInstance, Population
    from paper_2605_05208_b200.localsearch import draw_permutations, enabled_operators
    from paper_2605_05208_b200 import distributed as DS

    name = args.config
    spec = W.CONFIGS[name]
    total = (args.pop or spec.population) * (world if args.weak else 1)
    ids = list(DS.shard_range(total, world, rank))  # strong scaling: the population is split over the ranks
    per = len(ids)
    spec, inst, consts, nbr, sols = make_workload(name, ids, device=local)
    ops = enabled_operators(inst)
    perms = np.stack([draw_permutations(random.Random(i), ops, args.depth + 1) for i in ids])
    lams = [[1.0] * 4] * per
    dinst = DeviceInstance(inst, consts, nbr, local)
    J, K = Population.caps_for(sols, inst)
    pop = Population(dinst, per, J, K, 1 << 15)
    stream = torch.cuda.current_stream(dev)
    sh = ctypes.c_void_p(stream.cuda_stream)
    cfg = P.SearchConfig(depth=args.depth, multi_move=True)
    elen = DS.encode_len(inst.n_customers, inst.n_customers)

    def elite_exchange(st, download):
        """NCCL all_gather of every rank's elite (its lowest-D feasible individual, else
        its first) as a fixed-size int32 encoding -- the only collective of the job."""
        if world == 1:
            return None
        Ds = [s["best_feasible_D"] for s in st]
        best = int(np.argmin(Ds))
        routes = download(best)
        # fixed length on every rank: routes with customers never exceed the customer count
        enc = DS.encode_elite(routes, Ds[best], inst.n_customers, inst.n_customers)
        return DS.best_of(DS.exchange_elites(enc, device=dev))

    def device_step(profile=False):
        """One step, start states resident: the population descent and the elite
        exchange, CUDA-event timed on the launching stream."""
        pop.upload(sols, lams, sh)
        pop.set_profiling(profile)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st = pop.local_search(perms, cfg.depth, True, 0.5, 0.01, 1e4, stream=sh)
        if not profile:
            elite_exchange(st, lambda b: pop.download_range(b, 1, sh)[0])
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1), st

    for _ in range(args.warmup):
        device_step()
    # timed region: K complete population descents (+ elite exchange), device-timed
    flush_l2(torch, dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    tot_ms, cands, descents, rounds0 = 0.0, 0, 0, pop.timing()["rounds"]
    stats_last = None
    for k in range(args.steps):
        ms, st = device_step()
        tot_ms += ms
        cands += sum(sum(s["cands"]) for s in st)
        descents += len(st)
        stats_last = st
        if k + 1 < args.steps:
            flush_l2(torch, dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    rounds = pop.timing()["rounds"] - rounds0
    # the timed individuals' final states (checked against the oracle below)
    final_routes = [pop.download_range(b, 1, sh)[0] for b in range(min(per, os.cpu_count() or 1))]
    # per round: plan, the staged evaluators (relocate as two family kernels on windowed
    # instances with the large shape), the depot (+ 2-opt without windows) enumerators,
    # 3 generic-path drains (one per queue region), select; per step: unpack + rebuild
    n_enum = 2 if inst.has_windows else 3
    n_staged = 4 if (inst.has_windows and pop.info()["items_per_task"] == 32) else 3
    launches = rounds * (1 + n_staged + n_enum + 3 + 1) + 2 * args.steps

    # profiled pass (untimed; evaluation phase serialised): per-evaluator times,
    # eval-kernel share, per-op candidates
    tm0 = pop.timing()
    ms_p, st_p = device_step(profile=True)
    tm1 = pop.timing()
    tm = {k: tm1[k] - tm0[k] for k in tm1}
    pop.set_profiling(False)
    op_c = np.sum([s["cands"] for s in st_p], axis=0)
    ab = ALG_BYTES_WIN if inst.has_windows else ALG_BYTES_NOWIN
    af = ALG_FP64_WIN if inst.has_windows else ALG_FP64_NOWIN
    alg_bytes = float(sum(op_c[o] * ab[o] for o in range(6)))
    alg_fp64 = float(sum(op_c[o] * af[o] for o in range(6)))
    n_rounds_p = max(tm["kern_rounds"], 1)
    eval_ms = sum(tm["kern_" + k + "_ms"] for k in ("relocate", "relocate_intra", "swap", "swap_intra",
                                                     "two_opt_star", "depot_generic"))
    # dominant evaluator: the operator whose kernels (staged evaluator + its intra-route drain)
    # take the most time in the profiled pass; SURVEY.md 8(d) per-candidate figures x its candidates
    ev_ms = {0: tm["kern_relocate_ms"] + tm["kern_relocate_intra_ms"],
             1: tm["kern_swap_ms"] + tm["kern_swap_intra_ms"], 2: tm["kern_two_opt_star_ms"]}
    dom = max(ev_ms, key=ev_ms.get)
    dom_name = ("relocate", "swap", "two_opt_star")[dom]
    rel_avg_ms = ev_ms[dom] / n_rounds_p
    rel_fp64 = op_c[dom] * af[dom] / n_rounds_p  # per launch
    rel_bytes = op_c[dom] * ab[dom] / n_rounds_p
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    l2_gbs = measure_l2_gbs(local)
    fp64_peak = measure_fp64_gops(local)
    ncu = load_ncu(name, dom_name)
    fp64_gops = rel_fp64 / (rel_avg_ms * 1e-3) / 1e9 if rel_avg_ms > 0 else 0.0
    rel_gbs = rel_bytes / (rel_avg_ms * 1e-3) / 1e9 if rel_avg_ms > 0 else 0.0
    live = {"kernel": f"{dom_name} evaluator: staged kernel(s) + its intra-route drain (k_eval_g)" if dom < 2
            else "two_opt_star evaluator (staged kernel)",
            "avg_launch_ms": rel_avg_ms, "launches": int(n_rounds_p),
            "share_of_eval_phase": ev_ms[dom] / eval_ms if eval_ms > 0 else None,
            "fp64": {"achieved_gops": fp64_gops, "peak_gops": fp64_peak, "frac": fp64_gops / fp64_peak,
                     "per_candidate": af[dom],
                     "how": "SURVEY.md 8(d) fp64 ops per candidate x candidates per launch / CUDA-event launch "
                            "time (profiled pass, evaluators serialised); peak = mdr_probe_fp64_gops "
                            "(independent dadd/dmul chains, no FMA)"},
            "l2": {"achieved_gbs": rel_gbs, "peak_gbs": l2_gbs, "frac": rel_gbs / l2_gbs,
                   "per_candidate_bytes": ab[dom],
                   "how": "SURVEY.md 8(d) algorithmic bytes per candidate; peak = mdr_probe_l2_gbs "
                          "(ld.global.cg over a 32 MiB L2-resident buffer)"},
            "hbm_peak_gbs": hbm, "hbm_peak_source": "MEASURED_PEAKS.json" if peaks else "fallback"}
    if ncu:
        roof = {"bound": ncu["binding"], "achieved": ncu["achieved"], "peak": ncu["peak"], "unit": ncu["unit"],
                "frac": ncu["frac"], "traffic": ncu.get("dram_bytes_per_launch"), "roofs": ncu.get("roofs"),
                "kernel": ncu["kernel"], "ncu": ncu["metrics"], "source": ncu["source"], "live": live}
    else:  # no capture of this config committed: the live fp64 roof
        roof = {"bound": "fp64", "achieved": fp64_gops, "peak": fp64_peak, "unit": "Gop/s",
                "frac": fp64_gops / fp64_peak, "traffic": None, "kernel": live["kernel"], "ncu": None,
                "source": None, "live": live}

    # the granular neighbour-list build on the device (one
    # call incl. H2D of the matrix) vs the host restatement, on this instance
    from paper_2605_05208_b200.neighborhood import build_device as nbr_device
    t0 = time.perf_counter()
    nb_dev = nbr_device(inst, NeighborConfig(spec.theta), consts, device=local)
    nb_call_ms = 1000 * (time.perf_counter() - t0)
    t0 = time.perf_counter()
    nb_host = build(inst, NeighborConfig(spec.theta), consts)
    nb_host_ms = 1000 * (time.perf_counter() - t0)
    nbr_line = {"kernel_ms": nb_dev.kernel_ms, "call_ms": nb_call_ms, "host_numpy_ms": nb_host_ms,
                "identical": bool(np.array_equal(nb_dev.lists, nb_host.lists)),
                "nodes": inst.n_nodes, "theta": spec.theta}

    # e2e: through the public API with host Solution objects, H2D + D2H (and the
    # elite exchange at N > 1) inside, CUDA-event timed like `value`
    e2e = None
    if not args.no_e2e:
        e_ms, e_cands, h2d, d2h, e_steps = 0.0, 0, 0, 0, []
        for _ in range(2):  # warm-up (allocation, first-call costs)
            P.local_search_population([s.clone() for s in sols], [P.PenaltyState() for _ in sols], cfg, nbr, consts,
                                      inst, [random.Random(i) for i in ids], device=local)
        for k in range(max(1, args.steps)):
            work = [s.clone() for s in sols]
            pens = [P.PenaltyState() for _ in sols]
            rngs = [random.Random(i) for i in ids]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            st = P.local_search_population(work, pens, cfg, nbr, consts, inst, rngs, device=local)
            elite_exchange(st, lambda b: [(r.depart, r.arrive, list(r.customers)) for r in work[b].routes])
            e1.record(stream)
            e1.synchronize()
            e_ms += e0.elapsed_time(e1)
            e_steps.append(e0.elapsed_time(e1))
            e_cands += sum(sum(s["cands"]) for s in st)
            srch = P.localsearch._searcher(inst, consts, nbr, local)
            h2d = srch.pop.h2d_bytes + perms.nbytes
            d2h = srch.pop.d2h_bytes
        e2e = {"value": e_cands, "unit": "move-evals/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms / max(1, args.steps), "_ms": e_ms,
               "steps_ms": e_steps}

    repair_line = None
    if not args.no_repair and world == 1:
        repair_line = bench_repair(name, inst, consts, sols, ids, local, max(1, args.steps),
                                   cpu=not args.no_cpu_baseline)

    # max over ranks (time), sum over ranks (work)
    t = torch.tensor([tot_ms, float(cands), float(descents), e2e["_ms"] if e2e else 0.0,
                      float(e2e["value"]) if e2e else 0.0], dtype=torch.float64, device=dev)
    tmax = t.clone()
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    tot_ms = float(tmax[0])
    cands_all, desc_all = float(t[1]), float(t[2])
    if e2e is not None:
        e2e["value"] = float(t[4]) / (float(tmax[3]) / 1000.0)
        e2e["ms_per_step"] = float(tmax[3]) / max(1, args.steps)
        del e2e["_ms"]
    if rank == 0:
        cpu, cpu_np, parity = None, None, None
        if world == 1 and not args.no_cpu_baseline:
            cpu, res = cpu_baseline(name, inst, consts, nbr, sols, ids, args.depth)
            # the timed device descents of the sampled individuals vs the oracle: bit-exact routes
            ok = sum(1 for (routes, _, _), got in zip(res, final_routes) if routes == got)
            parity = {"checked": len(res), "bit_exact": ok,
                      "what": "final routes of the timed descents of individuals "
                              f"{ids[0]}..{ids[len(res)-1]} == the C oracle's (pinned to the reference)"}
            if not args.no_numpy_ref:
                cpu_np = numpy_reference_leg(inst, spec, sols, ids, args.depth)
        value = cands_all / (tot_ms / 1000.0)
        line = {
            "metric": "move_evals_per_s", "value": value, "unit": "move-evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(name, spec, total, args.depth),
            "population_per_gpu": per,
            "descents_per_s": desc_all / (tot_ms / 1000.0),
            "candidates_per_step": cands_all / args.steps,
            "parity_checked": parity,
            "roofline": roof,
            "cpu_baseline": cpu,
            "cpu_baseline_numpy": cpu_np,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "neighbor_build": nbr_line,
            "repair": repair_line,
            "clocks": clocks,
            "profile": {"rounds_per_step": rounds / args.steps, "plan_ms": tm["plan_ms"],
                        "eval_ms_serialised": eval_ms, "select_ms": tm["select_ms"], "total_ms": tm["total_ms"],
                        "evaluators_ms": {k[5:-3]: tm[k] for k in tm if k.startswith("kern_") and k.endswith("_ms")},
                        # per-operator candidate counts of the profiled step (the
                        # GPU tests assert them equal to the reference's / the oracle's)
                        "cands_per_op": {n: int(op_c[o]) for o, n in enumerate(
                            ("relocate", "swap", "two_opt_star", "two_opt", "depot_insert", "depot_replace"))}},
            # SURVEY.md 8(d) flavour 1: candidates scored per second of evaluation
            # phase only (enumerate + evaluate + leader/follower reduction), beside
            # the oracle's evaluate-all-operators on the start states on all host threads
            "eval_only": eval_only_line(name, inst, consts, nbr, sols, float(np.sum(op_c)), eval_ms * 1e-3,
                                        cpu=world == 1 and not args.no_cpu_baseline),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
