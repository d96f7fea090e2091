set -x
run() { env $3 MDR_LIB=$PWD/paper_2605_05208_b200/$1 timeout 600 python bench.py --config $4 --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/sw_$2_$4.jsonl 2> gpurun_out/sw_$2_$4.err; }
for c in C4 C2; do
  run libmdr_sm100.so base X=1 $c
  run libmdr_youter.so yo0 MDR_SWAP_SHAPE=0 $c
  run libmdr_youter.so yo1 MDR_SWAP_SHAPE=1 $c
  run libmdr_youter.so yo2 MDR_SWAP_SHAPE=2 $c
done
MDR_LIB=$PWD/paper_2605_05208_b200/libmdr_youter.so MDR_SWAP_SHAPE=1 timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "fuzz or depth30 or appendix" > gpurun_out/sw_tests.log 2>&1; echo "yo tests exit $?" >> gpurun_out/sw_tests.log
tail -2 gpurun_out/sw_tests.log
for f in gpurun_out/sw_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
