"""The drop-in boundary itself: the UNMODIFIED reference
package, installed in baseline/_ref by baseline/install_reference.sh, has its
local-search path rebound to this package exactly as INTEGRATION.md sec. 2
says (localsearch.py:15 and engine.py:17 bind the names), and its own
engine.run must return the same RunStats -- cost curve, stagnation trace, best
and best-infeasible solutions -- as the unpatched reference on the same seed.

The reference engine calls local_search(..., on_feasible=snapshot_feasible)
(engine.py:109-110), so this also exercises the per-state on_feasible replay
and the in-place route mutation on the reference's own Solution/Route types.
"""
import os
import random
import sys

import pytest

from paper_2605_05208_b200 import workload as W

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isfile(os.path.join(REF, "mdroute", "engine.py")),
                                 reason="reference not installed (baseline/install_reference.sh)")]


def _mdroute():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import mdroute.engine
    import mdroute.localsearch
    import mdroute.model
    return mdroute


def _ref_instance(M, variant, nc, nd, seed, **kw):
    inst = W.make_instance(random.Random(seed), variant, n_customers=nc, n_depots=nd, **kw)
    nodes = [M.model.Node(n.id, n.kind, n.x, n.y, n.demand, n.service, n.tw_early, n.tw_late) for n in inst.nodes]
    return M.model.Instance(M.model.Variant(inst.variant.value), nodes, inst.n_depots, inst.dist,
                            fleet_per_depot=inst.fleet_per_depot, capacity=inst.capacity,
                            max_duration=inst.max_duration)


def _summary(st):
    r = lambda s: None if s is None else [(x.depart, x.arrive, list(x.customers)) for x in s.routes]  # noqa: E731
    return dict(generations=st.generations, cost_curve=[float(x).hex() for x in st.cost_curve],
                stagnation=list(st.stagnation_trace), best_cost=float(st.best_cost).hex(),
                feasible=st.feasible_found, best=r(st.best), best_inf=float(st.best_infeasible_cost).hex(),
                best_inf_routes=r(st.best_infeasible))


CASES = [("mdvrp", 30, 3, 11, dict(fleet=4), True), ("mdvrptw", 28, 2, 12, dict(max_duration=600.0), True),
         ("mdovrp", 26, 3, 13, {}, False), ("mdvrptw", 24, 3, 14, dict(fleet=3), False)]


@pytest.mark.parametrize("variant,nc,nd,seed,kw,mm", CASES)
def test_reference_engine_with_rebound_local_search(variant, nc, nd, seed, kw, mm, monkeypatch):
    M = _mdroute()
    import paper_2605_05208_b200 as b200
    cfg = M.engine.SolverConfig(generations=12, depth=80, mu=6, multi_move=mm, seed=seed)
    want = _summary(M.engine.run(_ref_instance(M, variant, nc, nd, seed, **kw), cfg))
    # rebind where the names are imported
    monkeypatch.setattr(M.localsearch, "local_search", b200.local_search)
    monkeypatch.setattr(M.engine, "local_search", b200.local_search)
    monkeypatch.setattr(M.localsearch, "SolutionCache", b200.SolutionCache)
    monkeypatch.setattr(M.localsearch, "evaluate_candidates", b200.evaluate_candidates)
    monkeypatch.setattr(M.localsearch, "leader_and_followers", b200.leader_and_followers)
    got = _summary(M.engine.run(_ref_instance(M, variant, nc, nd, seed, **kw), cfg))
    assert got == want


def test_rebound_operator_level_contract(monkeypatch):
    """The reference's own evaluate_batch (localsearch.py:34-42) running on the
    rebound SolutionCache / evaluate_candidates / leader_and_followers returns
    the same leader and followers as the unpatched reference."""
    M = _mdroute()
    import mdroute.moves as RM
    import mdroute.evaluation as RE
    import mdroute.neighborhood as RN
    import paper_2605_05208_b200 as b200
    inst = _ref_instance(M, "mdvrptw", 40, 3, 21, fleet=4)
    consts = RE.ScalingConstants.from_instance(inst)
    nbr = RN.build(inst, RN.NeighborConfig(12), consts)
    sol = M.model.Solution([M.model.Route(r.depart, r.arrive, list(r.customers))
                            for r in W.random_solution(random.Random(5), inst).routes])
    pen = RE.PenaltyState(lam=[2.0, 1.0, 0.5, 3.0])

    def run_all():
        out = []
        for op in M.localsearch.enabled_operators(inst):
            cs = RM.enumerate_candidates(sol, op, nbr, inst)
            lead, fol = M.localsearch.evaluate_batch(sol, cs, pen, consts, inst, multi_move=True)
            out.append((None if lead is None else (lead.key(), lead.dF.hex()), [(f.key(), f.dF.hex()) for f in fol]))
        return out

    want = run_all()
    monkeypatch.setattr(M.localsearch, "SolutionCache", b200.SolutionCache)
    monkeypatch.setattr(M.localsearch, "evaluate_candidates", b200.evaluate_candidates)
    monkeypatch.setattr(M.localsearch, "leader_and_followers", b200.leader_and_followers)
    assert run_all() == want
