set -x
MDR_TSPLIT=4 timeout 1200 python -m pytest tests/test_gpu_shapes.py -q -m gpu -x -p no:cacheprovider > gpurun_out/ts_tests.log 2>&1; echo "tsplit4 tests exit $?" >> gpurun_out/ts_tests.log
for p in 32 64 128; do
  for v in 1 def; do
    if [ $v = def ]; then unset MDR_TSPLIT; else export MDR_TSPLIT=$v; fi
    timeout 600 python bench.py --config C4 --pop $p --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/ts_${p}_$v.jsonl 2> gpurun_out/ts_${p}_$v.err
  done
done
export MDR_TSPLIT=2; timeout 600 python bench.py --config C4 --pop 32 --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/ts_32_2.jsonl 2> gpurun_out/ts_32_2.err
export MDR_TSPLIT=2; timeout 600 python bench.py --config C4 --pop 256 --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/ts_256_2.jsonl 2> gpurun_out/ts_256_2.err
unset MDR_TSPLIT; timeout 600 python bench.py --config C4 --pop 256 --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/ts_256_def.jsonl 2> gpurun_out/ts_256_def.err
tail -2 gpurun_out/ts_tests.log
for f in gpurun_out/ts_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms')"; done
