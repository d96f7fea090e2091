# C1 (one descent, launch-latency bound): HEAD-of-round libraries vs current, 20 steps each, twice
for rep in 1 2; do for L in libmdr_head.so libmdr_prev.so libmdr_sm100.so; do
  MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 600 python bench.py --config C1 --pop 1 --steps 20 --warmup 5 --no-cpu-baseline --no-numpy-ref --no-repair > gpurun_out/c1_$L.$rep.jsonl 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/c1_$L.$rep.jsonl').read().strip().splitlines()[-1])
print('$L', $rep, round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],3), 'ms', 'e2e', round(d['e2e']['value']/1e6,2))"
done; done > gpurun_out/c1_ab.txt
cat gpurun_out/c1_ab.txt
