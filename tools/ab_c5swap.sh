set -x
run() { env $3 MDR_LIB=$PWD/paper_2605_05208_b200/$1 timeout 900 python bench.py --config C5 --pop 128 --steps 2 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/c5s_$2.jsonl 2> gpurun_out/c5s_$2.err; }
run libmdr_sm100.so base X=1
run libmdr_yonw.so yo_pipe MDR_SWAP_SHAPE=0
run libmdr_yonw.so yo_c20 MDR_SWAP_SHAPE=1
run libmdr_yonw.so yo_c24 MDR_SWAP_SHAPE=2
for f in gpurun_out/c5s_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
