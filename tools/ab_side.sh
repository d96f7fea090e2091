set -x
timeout 1500 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/side_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/side_tests.log
for L in libmdr_sm100.so libmdr_side1.so; do
  for spec in "C4 256" "C5 128" "C2 64"; do
    set -- $spec
    MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 900 python bench.py --config $1 --pop $2 --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/side_${L%.so}_$1.jsonl 2> gpurun_out/side_${L%.so}_$1.err
  done
done
tail -2 gpurun_out/side_tests.log
for f in gpurun_out/side_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
