# per-operator evaluator shapes (large): parity + C4/C5 bench; k_select phase clocks
set -x
timeout 1200 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/shp_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/shp_tests.log
timeout 600 python bench.py --config C4 --steps 3 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/shp_C4.jsonl 2> gpurun_out/shp_C4.err
timeout 900 python bench.py --config C5 --pop 128 --steps 2 --warmup 1 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/shp_C5.jsonl 2> gpurun_out/shp_C5.err
MDR_LIB=$PWD/paper_2605_05208_b200/libmdr_selprof.so timeout 600 python tools/selprof.py 32 > gpurun_out/selprof.txt 2>&1
MDR_LIB=$PWD/paper_2605_05208_b200/libmdr_selprof.so timeout 600 python tools/selprof.py 256 >> gpurun_out/selprof.txt 2>&1
tail -3 gpurun_out/shp_tests.log
for c in C4 C5; do python -c "
import json
d=json.loads(open('gpurun_out/shp_$c.jsonl').read().strip().splitlines()[-1]); pr=d['profile']
print('$c', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', 'select', round(pr['select_ms'],1), {k: round(v,1) for k,v in pr['evaluators_ms'].items()})"; done
cat gpurun_out/selprof.txt
