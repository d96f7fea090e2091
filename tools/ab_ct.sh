# evaluator shape at the strong-scaling shards: small (auto below 100k customers) vs forced large
set -x
for p in 64 32; do
  for ct in auto 32; do
    if [ $ct = auto ]; then unset MDR_CT; else export MDR_CT=$ct; fi
    timeout 600 python bench.py --config C4 --pop $p --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/ct_${p}_$ct.jsonl 2> gpurun_out/ct_${p}_$ct.err
  done
done
unset MDR_CT
for f in gpurun_out/ct_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', 'sel', round(pr['select_ms'],1), {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
