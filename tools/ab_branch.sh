set -x
timeout 1200 python -m pytest tests/test_gpu_shapes.py -q -m gpu -x -p no:cacheprovider > gpurun_out/br_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/br_tests.log
for p in 256 32 64; do
  for v in branch nobranch; do
    if [ $v = nobranch ]; then export MDR_REL_NOBRANCH=1; else unset MDR_REL_NOBRANCH; fi
    timeout 600 python bench.py --config C4 --pop $p --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/br_${p}_$v.jsonl 2> gpurun_out/br_${p}_$v.err
  done
done
unset MDR_REL_NOBRANCH
tail -2 gpurun_out/br_tests.log
for f in gpurun_out/br_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms')"; done
