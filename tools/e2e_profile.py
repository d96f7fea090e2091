"""Host-side cost breakdown of the e2e path (local_search_population, C4, 256)."""
import cProfile
import os
import pstats
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_05208_b200 as P  # noqa: E402

NPOP = int(sys.argv[1]) if len(sys.argv) > 1 else 256
spec, inst, consts, nbr, sols = bench.make_workload("C4", list(range(NPOP)))
cfg = P.SearchConfig(depth=500, multi_move=True)
run = lambda: P.local_search_population([s.clone() for s in sols], [P.PenaltyState() for _ in sols], cfg, nbr,  # noqa
                                        consts, inst, [random.Random(i) for i in range(NPOP)])
run()
pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
