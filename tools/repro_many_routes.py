import random, sys
sys.path.insert(0, ".")
import paper_2605_05208_b200 as P
from paper_2605_05208_b200 import workload as W
from paper_2605_05208_b200.model import Route, Solution
rng = random.Random(3)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
inst = W.make_instance(rng, "mdvrp", n_customers=n, n_depots=4)
c = P.ScalingConstants.from_instance(inst)
nb = P.build_neighbors(inst, P.NeighborConfig(20), c)
s = Solution([Route(i % 4, i % 4, [4 + i]) for i in range(n)])
print("routes", len(s.routes), flush=True)
P.local_search(s, P.PenaltyState(), P.SearchConfig(2, True), nb, c, inst, random.Random(0))
print("ok", flush=True)
