set -x
for L in libmdr_sm100.so libmdr_pad168.so; do
  for spec in "C5 128" "C3 128"; do
    set -- $spec
    MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 900 python bench.py --config $1 --pop $2 --steps 2 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/pad2_${L%.so}_$1.jsonl 2> gpurun_out/pad2_${L%.so}_$1.err
  done
done
for f in gpurun_out/pad2_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
