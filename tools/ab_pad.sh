# RB stride 176 B (bank-conflict-free route staging reads) vs 160 B
set -x
for L in libmdr_sm100.so libmdr_nopad.so; do
  for spec in "C4 256" "C5 128" "C2 64"; do
    set -- $spec
    MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 900 python bench.py --config $1 --pop $2 --steps 2 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/pad_${L%.so}_$1.jsonl 2> gpurun_out/pad_${L%.so}_$1.err
  done
done
timeout 900 python -m pytest tests/test_gpu_shapes.py -q -m gpu -x -p no:cacheprovider -k "fuzz" > gpurun_out/pad_tests.log 2>&1; echo "pad tests exit $?" >> gpurun_out/pad_tests.log
tail -2 gpurun_out/pad_tests.log
for f in gpurun_out/pad_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); pr=d['profile']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
timeout 600 python tools/e2e_profile.py 64 > gpurun_out/e2e_prof64.txt 2>&1
timeout 600 python tools/e2e_profile.py 256 > gpurun_out/e2e_prof256.txt 2>&1
head -40 gpurun_out/e2e_prof64.txt; head -40 gpurun_out/e2e_prof256.txt
