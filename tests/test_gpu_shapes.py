"""GPU parity at the shapes the benchmark times.

The evaluator shape of a population (items per CTA task, warps per CTA) is
chosen from its size (mdr_pop_create); these tests pin the kernels the
benchmark actually launches:

* the 64-case descent fuzz re-run with the large shape forced (MDR_CT=32);
* BASELINE.json configs[3] itself -- C4, MDVRPTW 1000x10, the Appendix-A
  population of 256 (start i = initial_solution(Random(100+i)), LS rng
  Random(i)) -- complete depth-500 descents of all 256 on the device, 16 of
  them checked against the oracle, plus all 256 at depth 30;
* configs[4] -- C5, MDVRP 4000x20 (theta 40, dist > L2), population 64 at
  depth 20.

Bit-exact (`==`): final routes in order, penalties, pass counts, per-operator
candidate counts.  The oracle itself is pinned to the reference
(tests/test_oracle_golden.py); reference: batch.py:365-553,
localsearch.py:97-140.
"""
import os
import random
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import golden_io as G
import paper_2605_05208_b200 as P
from paper_2605_05208_b200 import workload as W
from paper_2605_05208_b200.localsearch import _searcher, draw_permutations
from oracle import oracle as O

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


def _start(args):
    """Oracle start state (the scalar restatement of genetic.initial_solution)."""
    from oracle import initial_ref
    name, i = args
    spec = W.CONFIGS[name]
    inst, _ = W.appendix_a_instance(spec)
    consts = P.ScalingConstants.from_instance(inst)
    s = initial_ref.initial_solution(inst, consts, P.PenaltyState(), random.Random(100 + i))
    return [(r.depart, r.arrive, list(r.customers)) for r in s.routes]


_CACHE = {}


def appendix_a(name, n):
    """Instance, constants, lists and the first n Appendix-A start states of a
    config, built on the device (genetic.initial_solutions: mdr_construct + IBI
    repair); the first few are checked against the oracle's restatement."""
    if (name, n) not in _CACHE:
        spec = W.CONFIGS[name]
        inst, _ = W.appendix_a_instance(spec)
        consts = P.ScalingConstants.from_instance(inst)
        nbr = P.build_neighbors(inst, P.NeighborConfig(spec.theta), consts)
        sols = P.initial_solutions(inst, consts, P.PenaltyState(), [random.Random(100 + i) for i in range(n)])
        k = min(n, max(2, THREADS))
        with ProcessPoolExecutor(max(1, min(THREADS, 32)), mp_context=__import__("multiprocessing").get_context("spawn")) as ex:
            raw = list(ex.map(_start, [(name, i) for i in range(k)]))
        assert [[(r.depart, r.arrive, list(r.customers)) for r in s.routes] for s in sols[:k]] == raw, \
            "device start states differ from the oracle's"
        _CACHE[(name, n)] = (inst, consts, nbr, sols)
    return _CACHE[(name, n)]


def _device_descents(inst, consts, nbr, sols, depth, ids):
    work = [s.clone() for s in sols]
    pens = [P.PenaltyState() for _ in sols]
    stats = P.local_search_population(work, pens, P.SearchConfig(depth=depth, multi_move=True), nbr, consts, inst,
                                      [random.Random(i) for i in ids])
    info = _searcher(inst, consts, nbr, 0).pop.info()
    return work, pens, stats, info


def _oracle_descents(inst, consts, nbr, sols, depth, ids):
    oi = O.OracleInstance(inst, consts, nbr)
    ops = P.enabled_operators(inst)
    perms = [draw_permutations(random.Random(i), ops, depth + 1) for i in ids]
    return O.local_search_many_routes(oi, sols, [[1.0] * 4] * len(sols), depth, True, 0.5, 0.01, 1e4, perms,
                                      THREADS)


def _assert_same(work, pens, stats, want, which):
    for j, (routes, lam, st) in zip(which, want):
        assert G.routes_of(work[j]) == routes, f"individual {j}: routes differ"
        assert pens[j].lam == lam, f"individual {j}: penalties differ"
        assert stats[j]["passes"] == st["passes"] and stats[j]["accepted"] == st["accepted"], j
        assert stats[j]["cands"] == st["cands"], f"individual {j}: candidate counts differ"


FUZZ = list(range(int(os.environ.get("MDR_FUZZ_N", "64"))))


@pytest.mark.parametrize("seed", FUZZ)
def test_fuzz_large_cta_shape_bit_exact_vs_oracle(seed, monkeypatch):
    """The descent fuzz of test_gpu_parity with the large evaluator shape forced
    (the shape C4/C5 run): randomised variants, 2-120 customers, 1-6 depots,
    fleet limits, tight capacity/duration, theta 1-30, depth 1-300."""
    monkeypatch.setenv("MDR_CT", "32")
    r = random.Random(19000 + seed)
    variant = r.choice(["mdvrp", "mdvrptw", "mdovrp"])
    nc, nd = r.randint(2, 120), r.randint(1, 6)
    fleet = r.choice([None, None, 1, 2, 4])
    cap = r.choice([None, 15, 40, 1000])
    dur = r.choice([None, None, 150.0, 400.0]) if variant != "mdovrp" else None
    inst = W.make_instance(r, variant, n_customers=nc, n_depots=nd, capacity=cap, max_duration=dur, fleet=fleet)
    consts = P.ScalingConstants.from_instance(inst)
    nbr = P.build_neighbors(inst, P.NeighborConfig(r.choice([1, 3, 8, 30])), consts)
    count = r.randint(1, 8)
    sols = [W.random_solution(random.Random(seed * 100 + i), inst, scramble_depots=r.random() < 0.5)
            for i in range(count)]
    depth, mm = r.randint(1, 300), r.random() < 0.6
    lams = [[r.choice([0.01, 0.3, 1.0, 7.0]) for _ in range(4)] for _ in range(count)]
    ops = P.enabled_operators(inst)
    oi = O.OracleInstance(inst, consts, nbr)
    want = [O.local_search(oi, s, lams[i], depth, mm, 0.5, 0.01, 1e4, draw_permutations(random.Random(i), ops,
                                                                                      depth + 1))
            for i, s in enumerate(sols)]
    work = [s.clone() for s in sols]
    pens = [P.PenaltyState(lam=list(l)) for l in lams]
    stats = P.local_search_population(work, pens, P.SearchConfig(depth=depth, multi_move=mm), nbr, consts, inst,
                                      [random.Random(i) for i in range(count)])
    assert _searcher(inst, consts, nbr, 0).pop.info()["items_per_task"] == 32
    for i in range(count):
        routes, lam, st, _ = want[i]
        assert G.routes_of(work[i]) == routes, f"seed {seed} individual {i}"
        assert pens[i].lam == lam
        assert stats[i]["passes"] == st["passes"] and stats[i]["cands"] == st["cands"]


def test_c4_population_256_depth500_sample_vs_oracle():
    """BASELINE configs[3] exactly as bench.py times it: 256 complete descents in
    one device run; individuals 0, 16, ..., 240 compared with the oracle."""
    inst, consts, nbr, sols = appendix_a("C4", 256)
    ids = list(range(256))
    work, pens, stats, info = _device_descents(inst, consts, nbr, sols, 500, ids)
    assert info["items_per_task"] == 32, info  # the large shape the benchmark times
    which = list(range(0, 256, 16))
    want = _oracle_descents(inst, consts, nbr, [sols[j] for j in which], 500, which)
    _assert_same(work, pens, stats, want, which)
    # individuals 0 and 1 against the reference package's own descents (tests/golden/large.json)
    import json
    gold = json.load(open(os.path.join(G.GOLD, "large.json")))["C4"]
    for i in (0, 1):
        g = gold["descents"][str(i)]
        assert G.routes_of(sols[i]) == [(d, a, list(c)) for d, a, c in gold["starts"][i]]
        assert G.routes_of(work[i]) == [(d, a, list(c)) for d, a, c in g["final"]], f"individual {i} vs reference"
        assert [x.hex() for x in pens[i].lam] == g["lam"]
        assert stats[i]["passes"] == g["passes"] and stats[i]["accepted"] == g["accepted"]
        assert stats[i]["cands"] == g["cands"]


def test_c4_population_256_depth30_all_vs_oracle():
    inst, consts, nbr, sols = appendix_a("C4", 256)
    ids = list(range(256))
    work, pens, stats, info = _device_descents(inst, consts, nbr, sols, 30, ids)
    assert info["items_per_task"] == 32, info
    want = _oracle_descents(inst, consts, nbr, sols, 30, ids)
    _assert_same(work, pens, stats, want, ids)


def test_c5_population_64_depth20_vs_oracle():
    """BASELINE configs[4] shard (512 over 8 GPUs = 64 per GPU), no windows, theta 40."""
    inst, consts, nbr, sols = appendix_a("C5", 64)
    ids = list(range(64))
    work, pens, stats, info = _device_descents(inst, consts, nbr, sols, 20, ids)
    assert info["items_per_task"] == 32, info
    want = _oracle_descents(inst, consts, nbr, sols, 20, ids)
    _assert_same(work, pens, stats, want, ids)


def test_c4_start_states_equal_reference_golden_shape():
    """The C4 start states are what bench.py feeds: sanity of size and coverage."""
    inst, consts, nbr, sols = appendix_a("C4", 256)
    for s in sols[:8]:
        assert sorted(s.customer_list()) == list(range(inst.n_depots, inst.n_nodes))
    assert np.mean([len(s.routes) for s in sols]) > 60
