"""Generation loop on the B200 path (mirrors `mdroute.engine`, engine.py:25-158;
SURVEY.md sec. 8(f) row 3).

`run(inst, cfg)` is the reference's sequential loop -- one offspring per
generation: route exchange, repair (device), local search (device), population
update, bandit rewards, best tracking -- with the same rng stream, so a given
seed reproduces the reference's RunStats exactly (pinned by
tests/golden/engine.json).

`run_batched(inst, cfg, batch)` is the B200 form: every generation builds
`batch` offspring (one route exchange each, from the generation's population
and bandit state, all exchanges in one device call with one rng per offspring
drawn from the run's: `route_exchange_batch`), repairs them in one device call
per insertion operator and descends them together with
`local_search_population`; survivor selection runs on the device too; the population, the
bandits and the best-so-far are then updated offspring by offspring in order.
Each offspring's local search draws from its own `random.Random` seeded from
the run's rng, and starts from the run's current penalty weights; the run's
weights afterwards are those of the last offspring (the sequential loop's
order).  batch = 1 is not the sequential loop (the seeding differs); use
`run` for reference-identical runs.
"""
from __future__ import annotations

import random
import time
from dataclasses import dataclass, field
from typing import Optional

from .evaluation import EvalBreakdown, PenaltyState, ScalingConstants, evaluate
from .genetic import (DIVERSITY_LEVELS, DiscountedUCB1, InsertionOperator, dcrex, improvement_reward,
                      initialize_population, repair_insert, repair_population, route_exchange,
                      route_exchange_batch)
from .localsearch import SearchConfig, _searcher, local_search, local_search_population
from .model import INF, Route, Solution
from .neighborhood import NeighborConfig, build_device
from .population import Population

VIOLATION_TOL = 1e-9


@dataclass
class SolverConfig:
    generations: int = 5000
    patience: int = 500
    time_limit: float = INF
    mu: int = 20
    theta: int = 50
    depth: int = 500
    kappa: float = 0.5
    xi: float = 0.7
    multi_move: bool = False
    seed: int = 1

    def __post_init__(self):
        if min(self.generations, self.patience, self.mu, self.theta, self.depth) < 1:
            raise ValueError("config values must be positive")
        if not (0 < self.kappa < 1) or not (0 < self.xi <= 1):
            raise ValueError("kappa and xi must lie in (0, 1)")
        if self.time_limit < 0:
            raise ValueError("time limit must be >= 0")


@dataclass
class RunStats:
    best_cost: float = INF
    best: Optional[Solution] = None
    feasible_found: bool = False
    best_infeasible_cost: float = INF
    best_infeasible: Optional[Solution] = None
    generations: int = 0
    wall_time: float = 0.0
    cost_curve: list = field(default_factory=list)
    stagnation_trace: list = field(default_factory=list)
    offspring: int = 0
    phase_s: dict = field(default_factory=dict)  # wall time per loop phase (run_batched)
    migrants: int = 0          # elites received from other islands (run_islands)
    global_best: float = INF   # lowest feasible cost over all islands (run_islands)


def gap(f: float, bks: float) -> float:
    if bks <= 0:
        raise ValueError("reference cost must be positive")
    return 100.0 * (f - bks) / bks


def _is_feasible(bd, sol, inst) -> bool:
    if max(bd.V1, bd.V2, bd.V3, bd.V4) > VIOLATION_TOL:
        return False
    return sorted(sol.customer_list()) == list(inst.customers())


def _penalized(bd, penalties) -> float:
    lam = penalties.lam
    return bd.D + lam[0] * bd.V1 + lam[1] * bd.V2 + lam[2] * bd.V3 + lam[3] * bd.V4


def _track_best(stats: RunStats, sol, bd, feas: bool) -> None:
    if feas:
        stats.feasible_found = True
        if bd.D < stats.best_cost:
            stats.best_cost = bd.D
            stats.best = sol.clone()
    elif bd.D < stats.best_infeasible_cost:
        stats.best_infeasible_cost = bd.D
        stats.best_infeasible = sol.clone()


class _Run:
    """State shared by the sequential and the batched loop."""

    def __init__(self, inst, cfg: SolverConfig, nbr=None):
        self.inst, self.cfg = inst, cfg
        self.rng = random.Random(cfg.seed)
        self.start = time.monotonic()
        self.deadline = self.start + cfg.time_limit if cfg.time_limit != INF else None
        self.consts = ScalingConstants.from_instance(inst)
        self.penalties = PenaltyState(cfg.kappa)
        self.nbr = nbr if nbr is not None else build_device(inst, NeighborConfig(cfg.theta), self.consts)
        self.search = SearchConfig(depth=cfg.depth, multi_move=cfg.multi_move)
        self.div_bandit = DiscountedUCB1(DIVERSITY_LEVELS)
        self.ins_bandit = DiscountedUCB1(len(InsertionOperator))
        self.stats = RunStats()
        self.pop = Population(cfg.mu, cfg.xi)
        self.full = list(inst.customers())
        for sol in initialize_population(inst, cfg.mu, self.consts, self.penalties, self.rng):
            bd = evaluate(sol, self.penalties, self.consts, inst)
            feas = _is_feasible(bd, sol, inst)
            self.pop.add(sol, bd, feas, inst)
            _track_best(self.stats, sol, bd, feas)
        self.gen = 0
        self.stagnation = 0

    def running(self) -> bool:
        c = self.cfg
        return (self.gen <= c.generations and self.stagnation <= c.patience
                and time.monotonic() - self.start <= c.time_limit)

    def snapshot_feasible(self, dist, sol) -> None:
        if dist < self.stats.best_cost and sorted(sol.customer_list()) == self.full:
            self.stats.feasible_found = True
            self.stats.best_cost = dist
            self.stats.best = sol.clone()

    def absorb(self, offspring, main, level: int, op: int, bd=None) -> None:
        """Score one offspring against its main parent (a population Member),
        reward the bandits, update population and best.  `bd`: its breakdown if
        already computed (on the device, same semantics as evaluate)."""
        inst, pen = self.inst, self.penalties
        if bd is None:
            bd = evaluate(offspring, pen, self.consts, inst)
        feas = _is_feasible(bd, offspring, inst)
        if sorted(offspring.customer_list()) != self.full:
            raise AssertionError("offspring lost customer coverage")
        if feas and main.feasible:
            reward = improvement_reward(main.breakdown.D, bd.D)
        else:
            reward = improvement_reward(main.penalized(pen), bd.D if feas else _penalized(bd, pen))
        self.div_bandit.update(level, reward)
        self.ins_bandit.update(int(op), reward)
        self.pop.add(offspring, bd, feas, inst)
        if self.pop.needs_selection:
            self.pop.survivor_selection(pen)
        _track_best(self.stats, offspring, bd, feas)
        self.stats.offspring += 1

    def close_generation(self, prev_best: float) -> None:
        self.stagnation = 0 if self.stats.best_cost < prev_best else self.stagnation + 1
        self.gen += 1
        self.stats.cost_curve.append(self.stats.best_cost)
        self.stats.stagnation_trace.append(self.stagnation)

    def finish(self) -> RunStats:
        self.stats.generations = self.gen
        self.stats.wall_time = time.monotonic() - self.start
        return self.stats


def run(inst, cfg: SolverConfig, nbr=None) -> RunStats:
    """The reference's generation loop (engine.py:73-138) on the device path."""
    R = _Run(inst, cfg, nbr)
    while R.running():
        prev = R.stats.best_cost
        x = dcrex([m.sol for m in R.pop.members], inst, R.consts, R.penalties, R.div_bandit, R.ins_bandit, R.rng)
        local_search(x.offspring, R.penalties, R.search, R.nbr, R.consts, inst, R.rng, deadline=R.deadline,
                     on_feasible=R.snapshot_feasible, feasible_best_only=True)  # keeps only the best
        x.offspring.meta["generation"] = R.gen
        R.absorb(x.offspring, R.pop.members[x.main_index], x.diversity_level, x.insertion_op)
        R.close_generation(prev)
    return R.finish()


def _batched_generation(R: "_Run", batch: int, device: int) -> None:
    """One lock-step generation of `batch` offspring (see the module docstring)."""
    inst, ph = R.inst, R.stats.phase_s
    prev = R.stats.best_cost
    t0 = time.perf_counter()
    parents = list(R.pop.members)
    members = [m.sol for m in parents]
    kids, info = [], []
    # one rng per offspring (drawn from the run's), so the B exchanges run together on the device
    xr = [random.Random(R.rng.getrandbits(64)) for _ in range(batch)]
    for off, unrouted, level, _, main_index in route_exchange_batch(members, inst, R.div_bandit, xr, device):
        op = InsertionOperator(R.ins_bandit.select())
        kids.append((off, unrouted))
        info.append((parents[main_index], level, op))
    t1 = time.perf_counter()
    for op in InsertionOperator:  # one device call per operator; RI draws from the run's rng
        idx = [j for j in range(batch) if info[j][2] == op and kids[j][1]]
        if not idx:
            continue
        if op == InsertionOperator.RI:
            for j in idx:
                repair_insert(kids[j][0], kids[j][1], op, inst, R.consts, R.penalties, R.rng)
        else:
            repair_population([kids[j][0] for j in idx], [kids[j][1] for j in idx], op, inst, R.consts,
                              R.penalties, device=device)
    offspring = []
    for off, _ in kids:
        off.drop_empty_routes()
        for r in off.routes:
            r.attr = None  # repaired: the cache is refreshed by the descent
        offspring.append(off)
    t2 = time.perf_counter()
    pens = [R.penalties.clone() for _ in offspring]
    rngs = [random.Random(R.rng.getrandbits(64)) for _ in offspring]
    local_search_population(offspring, pens, R.search, R.nbr, R.consts, inst, rngs, deadline=R.deadline,
                            device=device, on_feasible=R.snapshot_feasible, feasible_best_only=True)
    R.penalties.lam[:] = pens[-1].lam
    t3 = time.perf_counter()
    # evaluation.evaluate of every offspring on the device, where the descent left them
    bds = _searcher(inst, R.consts, R.nbr, device).pop.breakdowns([R.penalties.lam] * len(offspring))
    for off, (main, level, op), x in zip(offspring, info, bds):
        off.meta["generation"] = R.gen
        R.absorb(off, main, level, op, EvalBreakdown(*(float(v) for v in x)))
    R.close_generation(prev)
    t4 = time.perf_counter()
    for k, v in (("exchange", t1 - t0), ("repair", t2 - t1), ("local_search", t3 - t2), ("update", t4 - t3)):
        ph[k] = ph.get(k, 0.0) + v


def run_batched(inst, cfg: SolverConfig, batch: int = 64, nbr=None, device: int = 0) -> RunStats:
    """Lock-step generations of `batch` offspring (see the module docstring)."""
    if batch < 1:
        raise ValueError("batch must be >= 1")
    R = _Run(inst, cfg, nbr)
    while R.running():
        _batched_generation(R, batch, device)
    return R.finish()


def _elite(R: "_Run"):
    m = R.pop.best(R.penalties, feasible_only=True) or R.pop.best(R.penalties, feasible_only=False)
    return m.sol, (m.breakdown.D if m.feasible else INF)


def run_islands(inst, cfg: SolverConfig, batch: int = 64, exchange_every: int = 1, nbr=None, device: int = 0,
                group=None, comm_device=None) -> RunStats:
    """Island model over the ranks of an initialised torch.distributed group:
    rank r runs `run_batched` generations with seed cfg.seed + r; every
    `exchange_every` generations the ranks all_gather their elite (best feasible
    member, else best penalised) as a fixed-size int32 vector -- the only
    collective -- and each island adds the other islands' elites to its
    population.  All ranks stop together (a MIN all_reduce of the loop
    condition).  Returns this rank's RunStats; `global_best` holds the lowest
    feasible cost over all islands after the last exchange."""
    import torch
    import torch.distributed as dist
    from . import distributed as DS
    from dataclasses import replace
    if int(exchange_every) < 1:  # checked before the first collective: no rank may fail mid-loop
        raise ValueError("exchange_every must be >= 1")
    if int(batch) < 1:
        raise ValueError("batch must be >= 1")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    R = _Run(inst, replace(cfg, seed=cfg.seed + rank), nbr)
    cap = inst.n_customers  # routes with customers never exceed the customer count
    while True:
        flag = torch.tensor([1 if R.running() else 0], dtype=torch.int32, device=comm_device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag.item()) == 0:
            break
        _batched_generation(R, batch, device)
        if world > 1 and R.gen % exchange_every == 0:
            sol, D = _elite(R)
            routes = [(r.depart, r.arrive, list(r.customers)) for r in sol.routes if r.customers]
            vecs = DS.exchange_elites(DS.encode_elite(routes, D, inst.n_customers, cap), group=group,
                                      device=comm_device)
            for j, v in enumerate(vecs):
                if j == rank:
                    continue
                rts, _ = DS.decode_elite(v)
                mig = Solution([Route(d, a, c) for d, a, c in rts])
                mig.meta["migrant_from"] = j
                bd = evaluate(mig, R.penalties, R.consts, inst)
                feas = _is_feasible(bd, mig, inst)
                R.pop.add(mig, bd, feas, inst)
                if R.pop.needs_selection:
                    R.pop.survivor_selection(R.penalties)
                _track_best(R.stats, mig, bd, feas)
                R.stats.migrants += 1
    st = R.finish()
    best = torch.tensor([st.best_cost], dtype=torch.float64, device=comm_device)
    dist.all_reduce(best, op=dist.ReduceOp.MIN, group=group)
    st.global_best = float(best.item())
    return st
