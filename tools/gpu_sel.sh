# sorted-greedy follower selection in k_select: parity + shard benches
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_large_golden.py -q -m gpu -x -p no:cacheprovider > gpurun_out/sel_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/sel_tests.log
for p in 256 32; do
  timeout 600 python bench.py --config C4 --pop $p --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/sel_$p.jsonl 2> gpurun_out/sel_$p.err
done
tail -3 gpurun_out/sel_tests.log
for p in 256 32; do python -c "
import json
d=json.loads(open('gpurun_out/sel_$p.jsonl').read().strip().splitlines()[-1]); pr=d['profile']
print($p, round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', 'select', round(pr['select_ms'],1), {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
