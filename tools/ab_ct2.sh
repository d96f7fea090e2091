set -x
for spec in "C2 64" "C3 128"; do
  set -- $spec
  for ct in auto 32; do
    if [ $ct = auto ]; then unset MDR_CT; else export MDR_CT=$ct; fi
    timeout 600 python bench.py --config $1 --pop $2 --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/ct2_$1_$ct.jsonl 2> gpurun_out/ct2_$1_$ct.err
  done
done
unset MDR_CT
for f in gpurun_out/ct2_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', 'sel', round(pr['select_ms'],1))"; done
