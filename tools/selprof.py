"""k_select phase clocks (diagnostic library built with -DMDR_SEL_PROF): run one C4
population descent of --pop individuals and print the summed cycles per phase."""
import ctypes, os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2605_05208_b200 import _lib
from paper_2605_05208_b200.device import DeviceInstance, Population
from paper_2605_05208_b200.localsearch import draw_permutations, enabled_operators
pop_n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
spec, inst, consts, nbr, sols = bench.make_workload("C4", list(range(pop_n)))
ops = enabled_operators(inst)
perms = np.stack([draw_permutations(random.Random(i), ops, 501) for i in range(pop_n)])
d = DeviceInstance(inst, consts, nbr)
J, K = Population.caps_for(sols, inst)
pop = Population(d, pop_n, J, K, 1 << 15)
pop.upload(sols, [[1.0] * 4] * pop_n)
L = _lib.lib()
buf = (ctypes.c_ulonglong * 16)()
pop.local_search(perms, 500, True, 0.5, 0.01, 1e4)
L.mdr_debug_selprof(buf)
base = list(buf)
pop.upload(sols, [[1.0] * 4] * pop_n)
st = pop.local_search(perms, 500, True, 0.5, 0.01, 1e4)
L.mdr_debug_selprof(buf)
names = ["select followers", "apply", "incremental rebuild", "full rebuild", "fleet", "totals/adapt/etc"]
tot = sum(buf[i] - base[i] for i in range(6))
rounds = pop.timing()["rounds"] // 2
print(f"pop {pop_n}: rounds {rounds}, k_select CTA-cycles {tot:.3e}")
for i, n in enumerate(names):
    print(f"  {n:22s} {100 * (buf[i] - base[i]) / tot:5.1f}%  {(buf[i] - base[i]) / max(rounds, 1) / 1.965e3:8.1f} us-CTA per round")
act, full = buf[8] - base[8], buf[9] - base[9]
print(f"  active CTA-rounds {act}, full rebuilds {full} ({100 * full / max(act, 1):.1f}%), "
      f"{(buf[3] - base[3]) / max(full, 1) / 1.965e3:.1f} us each; mean CTA {tot / max(act, 1) / 1.965e3:.1f} us, "
      f"max CTA {buf[10] / 1.965e3:.1f} us; of a full rebuild, the compaction {(buf[11] - base[11]) / max(full, 1) / 1.965e3:.1f} us")
nb = buf[15] - base[15]
print(f"  staged rebuilds: batches {nb}; per batch: scan {(buf[12] - base[12]) / max(nb, 1) / 1.965e3:.2f} us, "
      f"stage {(buf[13] - base[13]) / max(nb, 1) / 1.965e3:.2f} us, fold {(buf[14] - base[14]) / max(nb, 1) / 1.965e3:.2f} us")
