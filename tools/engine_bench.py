"""Batched generation loop on an Appendix A config: phase times per generation."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_05208_b200 import engine as E  # noqa: E402
from paper_2605_05208_b200 import workload as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
gens = int(sys.argv[3]) if len(sys.argv) > 3 else 3
spec = W.CONFIGS[name]
inst, _ = W.appendix_a_instance(spec)
cfg = E.SolverConfig(generations=gens - 1, mu=20, theta=spec.theta, depth=500, multi_move=True, seed=1)
E.run_batched(inst, E.SolverConfig(generations=1, mu=4, theta=spec.theta, depth=20, seed=2), batch=batch)  # warm-up
t0 = time.perf_counter()
st = E.run_batched(inst, cfg, batch=batch)
wall = time.perf_counter() - t0
print(json.dumps(dict(config=name, depth=cfg.depth, mu=cfg.mu, batch=batch, generations=st.generations, offspring=st.offspring, wall_s=wall,
                      phase_s=st.phase_s, best_cost=st.best_cost, feasible=st.feasible_found,
                      offspring_per_s_loop=st.offspring / sum(st.phase_s.values()))))
