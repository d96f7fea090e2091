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
