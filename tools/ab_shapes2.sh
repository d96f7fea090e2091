set -x
run() { MDR_LIB=$PWD/paper_2605_05208_b200/$1 timeout 900 python bench.py --config $2 --pop $3 --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/s2_${1%.so}_$2.jsonl 2> gpurun_out/s2_${1%.so}_$2.err; }
run libmdr_sm100.so C4 256
run libmdr_tos32.so C4 256
run libmdr_sm100.so C5 128
run libmdr_nw24.so C5 128
run libmdr_sm100.so C3 128
run libmdr_nw24.so C3 128
for f in gpurun_out/s2_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
