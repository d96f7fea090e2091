# A/B of evaluator register budgets: default (16 warps/SM, 128 regs) vs 12 warps x 168 regs vs 8 warps x 255 regs
set -x
for L in libmdr_sm100.so libmdr_cu12.so libmdr_cu8.so; do
  for cfg in C4 C5; do
    MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 900 python bench.py --config $cfg --pop $([ $cfg = C5 ] && echo 128 || echo 256) --steps 2 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/lib_${L%.so}_$cfg.jsonl 2> gpurun_out/lib_${L%.so}_$cfg.err
  done
done
MDR_LIB=$PWD/paper_2605_05208_b200/libmdr_cu12.so timeout 900 python -m pytest tests/test_gpu_shapes.py -q -m gpu -x -p no:cacheprovider > gpurun_out/lib_cu12_tests.log 2>&1; echo "cu12 tests exit $?" >> gpurun_out/lib_cu12_tests.log
tail -2 gpurun_out/lib_cu12_tests.log
for f in gpurun_out/lib_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); p=d['profile']['evaluators_ms']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', {k: round(v,1) for k,v in p.items()})" 2>&1 | tail -1; done
