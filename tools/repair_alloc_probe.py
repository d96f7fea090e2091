"""Time Population creation vs repair call for the C4 batched-engine shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2605_05208_b200.device import Population
from paper_2605_05208_b200.session import session_for
spec, inst, consts, nbr, sols = bench.make_workload("C4", list(range(64)))
rs, pend = bench.repair_workload(sols, list(range(64)))
sess = session_for(inst, consts, None, 0)
for J, K in ((162, 42), (262, 42), (400, 64)):
    t = time.perf_counter(); pop = Population(sess.dinst, 256, J, K, 1 << 10); t1 = time.perf_counter()
    pop.upload(rs, [[1.0] * 4] * len(rs)); t2 = time.perf_counter()
    pop.repair(3, pend); t3 = time.perf_counter()
    print(f"J {J} K {K}: create {1e3*(t1-t):.1f} ms upload {1e3*(t2-t1):.1f} ms repair {1e3*(t3-t2):.1f} ms")
    del pop
