"""Generation loop against the reference's own engine.run
(tests/golden/engine.json from make_engine_golden.py).

CPU: the loop's host control plane (route exchange, bandits, population
management, evaluation, best tracking) with the oracle standing in for the two
device kernels it calls (local search, repair) -- the RunStats must equal the
reference's exactly.  GPU: the same runs through the device path."""
import json
import os
import random

import pytest

from oracle import oracle as O
from paper_2605_05208_b200 import engine as E
from paper_2605_05208_b200 import genetic as GN
from paper_2605_05208_b200 import workload as W
from paper_2605_05208_b200.localsearch import _advance, _apply_result, draw_permutations, enabled_operators
from paper_2605_05208_b200.neighborhood import NeighborConfig, build

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "engine.json")))


def _instance(spec):
    variant, nc, nd, kw, seed = spec
    return W.make_instance(random.Random(seed), variant, n_customers=nc, n_depots=nd, **kw)


def _routes(sol):
    return None if sol is None else [[r.depart, r.arrive, list(r.customers)] for r in sol.routes]


def _check(st, want):
    assert st.generations == want["generations"]
    assert [float(x).hex() for x in st.cost_curve] == want["cost_curve"]
    assert list(st.stagnation_trace) == want["stagnation_trace"]
    assert float(st.best_cost).hex() == want["best_cost"] and st.feasible_found == want["feasible_found"]
    assert float(st.best_infeasible_cost).hex() == want["best_infeasible_cost"]
    assert _routes(st.best) == want["best"]
    assert _routes(st.best_infeasible) == want["best_infeasible"]


def _oracle_kernels(setattr_):
    """Route the loop's two device calls through the oracle (CPU)."""
    cache = {}

    def oi_for(inst, consts, nbr):
        k = (id(inst), id(nbr))
        if k not in cache:
            cache[k] = O.OracleInstance(inst, consts, nbr)
        return cache[k]

    def local_search(sol, penalties, cfg, nbr, consts, inst, rng, deadline=None, on_feasible=None,
                     feasible_best_only=False):
        ops = enabled_operators(inst)
        perms = draw_permutations(rng, ops, cfg.depth + 1)
        routes, lam, st, tr = O.local_search(oi_for(inst, consts, nbr), sol, penalties.lam, cfg.depth,
                                             cfg.multi_move, penalties.kappa, penalties.lam_min, penalties.lam_max,
                                             perms, snapshot=on_feasible is not None)
        _advance(rng, ops, st["passes"])
        _apply_result(sol, routes)
        penalties.lam[:] = lam
        if on_feasible is not None and tr["best_feasible"] is not None:
            snap = sol.clone()
            _apply_result(snap, tr["best_feasible"])
            on_feasible(st["best_feasible_D"], snap)
        return sol

    def local_search_population(sols, penalties, cfg, nbr, consts, inst, rngs, deadline=None, device=0,
                                on_feasible=None, feasible_best_only=False):
        for s, p, r in zip(sols, penalties, rngs):
            local_search(s, p, cfg, nbr, consts, inst, r, deadline, on_feasible)

    def repair_population(sols, unrouteds, op, inst, consts, penalties, device=0):
        if not isinstance(penalties, (list, tuple)):
            penalties = [penalties] * len(sols)
        oi = oi_for(inst, consts, build(inst, NeighborConfig(1), consts)) if id(inst) not in cache else cache[id(inst)]
        cache[id(inst)] = oi
        for s, u, p in zip(sols, unrouteds, penalties):
            GN._write_back(s, O.repair(oi, s, u, int(op), p.lam)[0])
        return [dict(inserted=len(u)) for u in unrouteds]

    setattr_(E, "local_search", local_search)
    setattr_(E, "local_search_population", local_search_population)
    setattr_(E, "repair_population", repair_population)
    setattr_(GN, "repair_population", repair_population)
    setattr_(E, "build_device", build)
    from oracle import population_ref as PR, scalar_ref as SR
    from paper_2605_05208_b200.population import Population
    import numpy as np

    def host_select(self, mu, costs):  # the restatement standing in for mdr_population_select
        edges = [m.edges for m in self.members]
        self._dist, self._known = np.asarray(PR.distance_rows(edges), np.float64).reshape(len(edges), -1), len(edges)
        if costs is None or len(edges) <= mu:
            return []
        return PR.removal_order(edges, costs, [m.birth for m in self.members], mu, self.xi)

    setattr_(Population, "_device_select", host_select)
    setattr_(E, "evaluate", SR.evaluate)
    from oracle import initial_ref

    def init_pop(inst, mu, consts, penalties, rng, device=0):  # the restatement for the device construction
        return [initial_ref.initial_solution(inst, consts, penalties, rng) for _ in range(mu)]

    setattr_(E, "initialize_population", init_pop)

    from oracle import exchange_ref as XR

    def exchange_batch(population, inst, bandit, rngs, device=0):  # the host exchange, one rng per offspring
        return [XR.route_exchange(population, inst, bandit, r) for r in rngs]

    setattr_(E, "route_exchange_batch", exchange_batch)
    setattr_(GN, "route_exchange", lambda population, inst, bandit, rng, main_index=None, device=0:
             XR.route_exchange(population, inst, bandit, rng, main_index))

    class _HostPop:  # breakdowns of the last oracle batch, by the host evaluate
        sols = []

        def breakdowns(self, lams):
            from paper_2605_05208_b200.evaluation import PenaltyState
            from oracle.scalar_ref import evaluate
            out = []
            for s, l in zip(self.sols, lams):
                b = evaluate(s, PenaltyState(lam=l), self.consts, self.inst)
                out.append([b.D, b.V1, b.V2, b.V3, b.V4, b.F])
            return out

    host_pop = _HostPop()

    class _Searcher:
        pop = host_pop

    def lsp_capture(sols, penalties, cfg, nbr, consts, inst, rngs, deadline=None, device=0, on_feasible=None,
                    feasible_best_only=False):
        host_pop.sols, host_pop.consts, host_pop.inst = sols, consts, inst
        return local_search_population(sols, penalties, cfg, nbr, consts, inst, rngs, deadline, device, on_feasible)

    setattr_(E, "local_search_population", lsp_capture)
    setattr_(E, "_searcher", lambda *a, **k: _Searcher())


@pytest.fixture
def oracle_kernels(monkeypatch):
    _oracle_kernels(monkeypatch.setattr)


@pytest.mark.parametrize("tag", sorted(GOLD))
def test_engine_control_plane_equals_reference(tag, oracle_kernels):
    want = GOLD[tag]
    st = E.run(_instance(want["instance"]), E.SolverConfig(**want["config"]))
    _check(st, want)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted(GOLD))
def test_engine_on_device_equals_reference(tag):
    want = GOLD[tag]
    st = E.run(_instance(want["instance"]), E.SolverConfig(**want["config"]))
    _check(st, want)


@pytest.mark.gpu
@pytest.mark.parametrize("variant,fleet,dur", [("mdvrp", 2, None), ("mdvrptw", 3, 600.0), ("mdovrp", None, None),
                                               ("mdvrp", None, 200.0)])
def test_device_breakdown_equals_evaluate(variant, fleet, dur):
    """mdr_pop_breakdown == evaluation.evaluate bit for bit (infeasible random states,
    empty routes, fleet excess, closures)."""
    from paper_2605_05208_b200.device import DeviceInstance, Population
    from paper_2605_05208_b200.evaluation import PenaltyState, ScalingConstants
    from oracle.scalar_ref import evaluate
    inst = W.make_instance(random.Random(31), variant, n_customers=45, n_depots=3, fleet=fleet, max_duration=dur)
    consts = ScalingConstants.from_instance(inst)
    sols = [W.random_solution(random.Random(700 + i), inst) for i in range(9)]
    sols[3].routes[0].customers = []  # an empty route is skipped
    lams = [[random.Random(i).choice([0.1, 1.0, 30.0]) for _ in range(4)] for i in range(9)]
    J, K = Population.caps_for(sols, inst)
    pop = Population(DeviceInstance(inst, consts, None), 9, J, K)
    pop.upload(sols, lams)
    got = pop.breakdowns(lams)
    for s, l, g in zip(sols, lams, got):
        b = evaluate(s, PenaltyState(lam=l), consts, inst)
        assert [float(x).hex() for x in g] == [float(x).hex() for x in (b.D, b.V1, b.V2, b.V3, b.V4, b.F)]


@pytest.mark.gpu
def test_batched_engine_runs_and_keeps_coverage():
    """The lock-step form: B offspring per generation through the batched device
    calls; every offspring keeps full coverage, the best is feasible and its
    cost is the from-scratch evaluation of the returned solution."""
    want = GOLD["tw_mm"]
    inst = _instance(want["instance"])
    cfg = E.SolverConfig(**dict(want["config"], generations=4))
    st = E.run_batched(inst, cfg, batch=16)
    assert st.offspring == 16 * st.generations and st.feasible_found
    assert sorted(st.best.customer_list()) == list(inst.customers())
    from paper_2605_05208_b200.evaluation import PenaltyState, ScalingConstants, evaluate
    bd = evaluate(st.best, PenaltyState(), ScalingConstants.from_instance(inst), inst)
    assert max(bd.V1, bd.V2, bd.V3, bd.V4) <= 1e-9
    assert abs(bd.D - st.best_cost) <= 1e-9 * max(1.0, bd.D)


def _island_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _oracle_kernels(setattr)
    want = GOLD["tw_mm"]
    inst = _instance(want["instance"])
    cfg = E.SolverConfig(**dict(want["config"], generations=3, depth=20))
    st = E.run_islands(inst, cfg, batch=3, exchange_every=2)
    q.put((rank, st.generations, st.offspring, st.migrants, st.best_cost, st.global_best))
    dist.destroy_process_group()


def test_islands_gloo_world2_exchange_elites():
    """Island model host logic on CPU (gloo, 2 ranks, oracle kernels): both
    islands stop together, receive one migrant per exchange, and agree on the
    global best."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_island_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, g0, o0, m0, b0, gb0), (_, g1, o1, m1, b1, gb1) = res
    assert g0 == g1 == 4 and o0 == o1 == 12
    assert m0 == m1 == 2  # exchanges after generations 2 and 4
    assert gb0 == gb1 == min(b0, b1)


@pytest.mark.gpu
@pytest.mark.parametrize("variant,nc,nd,open_", [("mdvrp", 120, 4, False), ("mdvrptw", 90, 3, False),
                                                 ("mdovrp", 100, 5, True)])
def test_device_route_exchange_equals_host(variant, nc, nd, open_):
    """route_exchange_batch (mdr_route_exchange, one CTA per offspring) == the host
    route_exchange (genetic.py:343-446 restated) for every offspring, with each
    rng advanced identically; populations with duplicate members and all levels."""
    from oracle import exchange_ref as XR
    inst = W.make_instance(random.Random(nc), variant, n_customers=nc, n_depots=nd)
    pop = [W.random_solution(random.Random(900 + i), inst) for i in range(9)]
    pop.append(pop[3].clone())  # a duplicate member
    for level in (0, 3, 9, 19):
        bandit = GN.DiscountedUCB1(GN.DIVERSITY_LEVELS)
        for a in range(GN.DIVERSITY_LEVELS):  # make `level` the bandit's choice
            bandit.counts[a] = 1.0
            bandit.rewards[a] = 100.0 if a == level else 0.0
        seeds = [random.Random(level * 1000 + j).getrandbits(64) for j in range(24)]
        got = GN.route_exchange_batch(pop, inst, bandit, [random.Random(s) for s in seeds])
        for s, (off, unr, lv, sig, mi) in zip(seeds, got):
            r = random.Random(s)
            w_off, w_unr, w_lv, w_sig, w_mi = XR.route_exchange(pop, inst, bandit, r)
            assert (mi, lv, sig, unr) == (w_mi, w_lv, w_sig, w_unr)
            assert _routes(off) == _routes(w_off)
        rs = [random.Random(s) for s in seeds]
        GN.route_exchange_batch(pop, inst, bandit, rs)
        for s, r in zip(seeds, rs):
            w = random.Random(s)
            XR.route_exchange(pop, inst, bandit, w)
            assert r.getstate() == w.getstate()
