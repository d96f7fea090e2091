# A/B: pipelined relocate/swap evaluators (k_eval_p, default) vs k_eval_c (MDR_NO_PIPE=1); parity first
set -x
timeout 1200 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/ab_tests.log
for cfg in C4 C2 C3; do
  for v in pipe nopipe; do
    if [ $v = nopipe ]; then export MDR_NO_PIPE=1; else unset MDR_NO_PIPE; fi
    timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/ab_${cfg}_$v.jsonl 2> gpurun_out/ab_${cfg}_$v.err
  done
done
unset MDR_NO_PIPE
tail -3 gpurun_out/ab_tests.log
for f in gpurun_out/ab_*.jsonl; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); p=d['profile']['evaluators_ms']
print('$f', round(d['value']/1e9,3), 'G/s', {k: round(v,1) for k,v in p.items()})"; done
