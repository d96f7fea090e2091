# strong-scaling shards on one B200 (C4 population 256 split over N GPUs = 256/N per GPU) + engine host phases
set -x
for p in 256 128 64 32; do
  timeout 600 python bench.py --config C4 --pop $p --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/shard_$p.jsonl 2> gpurun_out/shard_$p.err
done
timeout 900 python tools/engine_bench.py C4 256 3 > gpurun_out/engine_C4.json 2> gpurun_out/engine_C4.err
for p in 256 128 64 32; do python -c "
import json
d=json.loads(open('gpurun_out/shard_$p.jsonl').read().strip().splitlines()[-1]); pr=d['profile']
print($p, round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', 'rounds', pr['rounds_per_step'], 'select', round(pr['select_ms'],1), 'plan', round(pr['plan_ms'],1), {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
cat gpurun_out/engine_C4.json; tail -3 gpurun_out/engine_C4.err
