set -x
for L in libmdr_sm100.so libmdr_g4.so; do
  for p in 256 32; do
    MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 600 python bench.py --config C4 --pop $p --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/g_${L%.so}_$p.jsonl 2> gpurun_out/g_${L%.so}_$p.err
  done
done
for f in gpurun_out/g_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', 'sel', round(pr['select_ms'],1), {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
