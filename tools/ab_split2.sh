set -x
MDR_REL_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_shapes.py -q -m gpu -x -p no:cacheprovider -k "fuzz or depth30" > gpurun_out/split_tests.log 2>&1; echo "split tests exit $?" >> gpurun_out/split_tests.log
for v in 0 1; do
  MDR_REL_SPLIT=$v timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/split_$v.jsonl 2> gpurun_out/split_$v.err
  MDR_REL_SPLIT=$v timeout 600 python bench.py --config C5 --pop 128 --steps 2 --warmup 1 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/split5_$v.jsonl 2> gpurun_out/split5_$v.err
done
tail -2 gpurun_out/split_tests.log
for f in split_0 split_1 split5_0 split5_1; do python -c "
import json
d=json.loads(open('gpurun_out/$f.jsonl').read().strip().splitlines()[-1]); pr=d['profile']
print('$f', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
