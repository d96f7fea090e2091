"""One C4 neighbour-list build and one batched IRI repair of 256 offspring
(the bench's repair workload) -- the command profiled by tools/prof_widen.sh."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_05208_b200.device import Population  # noqa: E402
from paper_2605_05208_b200.neighborhood import NeighborConfig, build_device  # noqa: E402
from paper_2605_05208_b200.session import session_for  # noqa: E402

spec, inst, consts, nbr, sols = bench.make_workload("C4", list(range(256)))
nb = build_device(inst, NeighborConfig(spec.theta), consts)
rs, pend = bench.repair_workload(sols, list(range(256)))
sess = session_for(inst, consts, None, 0)
J, K = Population.caps_for(rs, inst)
pop = Population(sess.dinst, len(rs), min(4094, J + max(len(u) for u in pend)), min(500, K + 32), 1 << 10)
pop.upload(rs, [[1.0] * 4] * len(rs))
st = pop.repair(3, pend)
print("neighbors kernel ms", nb.kernel_ms, "repair ref slot evals", sum(x["ref_slot_evals"] for x in st))
