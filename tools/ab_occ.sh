# occupancy A/B: 16 warps x 128 regs (default) vs 20 warps x 96 regs vs 24 warps x 80 regs, pipe and k_eval_c forms
set -x
run() { # lib tag env
  env $3 MDR_LIB=$PWD/paper_2605_05208_b200/$1 timeout 600 python bench.py --config C4 --steps 2 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/occ_$2.jsonl 2> gpurun_out/occ_$2.err
}
run libmdr_sm100.so base X=1
run libmdr_o20.so o20 X=1
run libmdr_o20.so o20np MDR_NO_PIPE=1
run libmdr_o24.so o24 X=1
run libmdr_o24.so o24np MDR_NO_PIPE=1
for f in gpurun_out/occ_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); p=d['profile']['evaluators_ms']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', {k: round(v,1) for k,v in p.items()})" 2>&1 | tail -1; done
