"""Where the e2e write-back time goes: the download C call vs the host list building."""
import ctypes as C, os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2605_05208_b200 as P
from paper_2605_05208_b200 import _lib
from paper_2605_05208_b200.device import DeviceInstance, Population
spec, inst, consts, nbr, sols = bench.make_workload("C4", list(range(256)))
cfg = P.SearchConfig(depth=500, multi_move=True)
work = [s.clone() for s in sols]
P.local_search_population(work, [P.PenaltyState() for _ in sols], cfg, nbr, consts, inst, [random.Random(i) for i in range(256)])
pop = P.localsearch._searcher(inst, consts, nbr, 0).pop
import torch
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); r = pop.download(); t1 = time.perf_counter()
    a = pop.route_attrs(0, 256); t2 = time.perf_counter()
    print(f"download {1000*(t1-t0):.1f} ms, route_attrs {1000*(t2-t1):.1f} ms")
# the C call alone
B = pop.B; cap_r = B * pop.J_cap; cap_c = pop.n_cust + 16
bufs = [np.zeros(B + 1, np.int32), np.zeros(cap_r + 1, np.int32), np.zeros(cap_c, np.int32), np.zeros(cap_r, np.int32), np.zeros(cap_r, np.int32)]
extra = np.zeros(B * 4); nr, nc = C.c_int32(cap_r), C.c_int32(cap_c)
for rep in range(3):
    t0 = time.perf_counter()
    _lib.lib().mdr_pop_download(pop.handle, *[_lib.ptr(b, _lib.i32p) for b in bufs], _lib.ptr(extra, _lib.f64p), C.byref(nr), C.byref(nc), None)
    t1 = time.perf_counter()
    print(f"mdr_pop_download C call {1000*(t1-t0):.1f} ms")
