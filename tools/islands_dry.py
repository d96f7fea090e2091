"""torchrun --nproc-per-node N tools/islands_dry.py [backend]: run_islands on the
device path (gloo: ranks may share one GPU -- a functional check)."""
import os, sys, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2605_05208_b200 as P
from paper_2605_05208_b200 import workload as W

backend = sys.argv[1] if len(sys.argv) > 1 else "gloo"
local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
torch.cuda.set_device(local)
dist.init_process_group(backend)
inst = W.make_instance(random.Random(13), "mdvrptw", n_customers=40, n_depots=3, fleet=4, max_duration=700.0)
cfg = P.SolverConfig(generations=5, mu=5, theta=10, depth=60, multi_move=True, seed=3)
comm = torch.device("cuda", local) if backend == "nccl" else None
st = P.run_islands(inst, cfg, batch=16, exchange_every=2, device=local, comm_device=comm)
print(f"rank {dist.get_rank()}: generations {st.generations} offspring {st.offspring} migrants {st.migrants} "
      f"best {st.best_cost:.3f} global {st.global_best:.3f}", flush=True)
dist.destroy_process_group()
