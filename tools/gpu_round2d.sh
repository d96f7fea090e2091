# device route exchange + k_select 512 threads + per-op shapes: tests, shard bench, engine phases
set -x
timeout 900 python -m pytest tests/test_engine.py -q -m gpu -x -p no:cacheprovider > gpurun_out/xc_tests.log 2>&1; echo "engine tests exit $?" >> gpurun_out/xc_tests.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -q -m gpu -x -p no:cacheprovider > gpurun_out/sel2_tests.log 2>&1; echo "parity tests exit $?" >> gpurun_out/sel2_tests.log
for p in 256 32; do
  timeout 600 python bench.py --config C4 --pop $p --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/sel2_$p.jsonl 2> gpurun_out/sel2_$p.err
done
timeout 900 python tools/engine_bench.py C4 256 3 > gpurun_out/engine_C4.json 2> gpurun_out/engine_C4.err
tail -15 gpurun_out/xc_tests.log; tail -2 gpurun_out/sel2_tests.log
for p in 256 32; do python -c "
import json
d=json.loads(open('gpurun_out/sel2_$p.jsonl').read().strip().splitlines()[-1]); pr=d['profile']
print($p, round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', 'select', round(pr['select_ms'],1), {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
cat gpurun_out/engine_C4.json; tail -3 gpurun_out/engine_C4.err
