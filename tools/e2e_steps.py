"""Per-step phase times of the e2e path (local_search_population at C4, 256), to find outliers."""
import os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2605_05208_b200 as P
from paper_2605_05208_b200 import localsearch as LS
spec, inst, consts, nbr, sols = bench.make_workload("C4", list(range(256)))
cfg = P.SearchConfig(depth=500, multi_move=True)
T = {}
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*a, **k):
        t0 = time.perf_counter(); r = f(*a, **k); T[name] = T.get(name, 0) + time.perf_counter() - t0; return r
    setattr(obj, name, g)
wrap(LS.DeviceSearch, "run"); wrap(LS, "_finish"); wrap(LS, "draw_permutations")
from paper_2605_05208_b200.device import Population
wrap(Population, "upload"); wrap(Population, "local_search"); wrap(Population, "download"); wrap(Population, "route_attrs")
for step in range(14):
    work = [s.clone() for s in sols]
    pens = [P.PenaltyState() for _ in sols]
    rngs = [random.Random(i) for i in range(256)]
    T.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.local_search_population(work, pens, cfg, nbr, consts, inst, rngs)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"step {step}: total {1000*tot:.0f} ms  " + "  ".join(f"{k} {1000*v:.0f}" for k, v in T.items()), flush=True)
