"""Device caches (session.py, localsearch._SEARCHERS) must not keep an instance
alive: their entries, and the device memory behind them, go with it (a fuzz of
1000 fresh instances ran the B200 out of memory before)."""
import gc
import random

import pytest

from paper_2605_05208_b200 import localsearch as LS
from paper_2605_05208_b200 import session as S
from paper_2605_05208_b200 import workload as W
from paper_2605_05208_b200.evaluation import PenaltyState, ScalingConstants
from paper_2605_05208_b200.genetic import InsertionOperator, repair_population
from paper_2605_05208_b200.neighborhood import NeighborConfig, build


def test_ref_is_weak_where_possible():
    class X:
        pass

    x = X()
    r = S._ref(x)
    assert r() is x
    del x
    gc.collect()
    assert r() is None
    assert S._ref(3)() == 3  # ints take no weak references: held strongly


@pytest.mark.gpu
def test_caches_release_instances():
    n0, m0 = len(S._SESSIONS), len(LS._SEARCHERS)
    for seed in range(3):
        r = random.Random(seed)
        inst = W.make_instance(r, "mdvrp", n_customers=30, n_depots=2)
        consts = ScalingConstants.from_instance(inst)
        nbr = build(inst, NeighborConfig(10), consts)
        sol = W.random_solution(random.Random(seed), inst)
        repair_population([sol.clone()], [[]], InsertionOperator.FBI, inst, consts, [PenaltyState()])
        LS._searcher(inst, consts, nbr)
        assert len(S._SESSIONS) > n0 and len(LS._SEARCHERS) > m0
        del inst, consts, nbr, sol
        gc.collect()
        assert len(S._SESSIONS) == n0 and len(LS._SEARCHERS) == m0


class _FakeDev:
    """Stand-in for the device instance (no GPU): records what it was built with."""

    def __init__(self, inst, consts, nbr=None, device=0):
        self.consts, self.nbr = consts, nbr


def test_searcher_rebuilt_when_scaling_constants_change(monkeypatch):
    monkeypatch.setattr(S, "DeviceInstance", _FakeDev)
    inst = W.make_instance(random.Random(4), "mdvrp", n_customers=12, n_depots=2)
    nbr = build(inst, NeighborConfig(5), ScalingConstants.from_instance(inst))
    a = LS._searcher(inst, ScalingConstants(1.0, 19.0), nbr)
    assert LS._searcher(inst, ScalingConstants(1.0, 19.0), nbr) is a
    b = LS._searcher(inst, ScalingConstants(2.0, 19.0), nbr)
    assert b is not a and b.session.dinst.consts.gamma == 2.0
    c = LS._searcher(inst, ScalingConstants(2.0, 7.0), nbr)
    assert c is not b and c.session.dinst.consts.theta == 7.0


def test_fresh_lists_per_run_do_not_accumulate_sessions(monkeypatch):
    """engine runs build new NeighborLists each time: one entry per instance stays."""
    monkeypatch.setattr(S, "DeviceInstance", _FakeDev)
    inst = W.make_instance(random.Random(5), "mdvrp", n_customers=12, n_depots=2)
    consts = ScalingConstants.from_instance(inst)
    n0, m0 = len(S._SESSIONS), len(LS._SEARCHERS)
    for _ in range(5):
        nbr = build(inst, NeighborConfig(5), consts)
        LS._searcher(inst, consts, nbr)
        S.session_for(inst, consts, None)
    assert len(S._SESSIONS) == n0 + 2  # with and without lists
    assert len(LS._SEARCHERS) == m0 + 1
