# A/B of the intra-route drains (k_eval_g): HEAD vs per-region specialisation (+ queue prefetch, + 16 warps)
set -x
run() {  # tag lib cfg pop [env]
  env $5 MDR_LIB=$PWD/paper_2605_05208_b200/$2 timeout 900 python bench.py --config $3 --pop $4 --steps 3 --warmup 3 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/g_$1_$3.jsonl 2> gpurun_out/g_$1_$3.err
}
for cfg in "C4 256" "C5 64" "C4 32"; do
  set -- $cfg
  run head libmdr_head.so $1 $2
  run spec libmdr_sm100.so $1 $2
  run nopf libmdr_nopf.so $1 $2
  run m2 libmdr_m2.so $1 $2
  run gen libmdr_sm100.so $1 $2 MDR_G_GENERIC=1
  run head2 libmdr_head.so $1 $2
  run spec2 libmdr_sm100.so $1 $2
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_large_golden.py -q -m gpu -x -p no:cacheprovider > gpurun_out/g_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/g_tests.log
tail -2 gpurun_out/g_tests.log
for f in gpurun_out/g_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); p=d['profile']['evaluators_ms']
print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G/s', d.get('parity_checked',{}).get('bit_exact'), {k: round(v,1) for k,v in p.items()})" 2>&1 | tail -1; done
MDR_LIB=$PWD/paper_2605_05208_b200/libmdr_selprof.so timeout 600 python tools/selprof.py 32 > gpurun_out/selprof.txt 2>&1
MDR_LIB=$PWD/paper_2605_05208_b200/libmdr_selprof.so timeout 600 python tools/selprof.py 256 >> gpurun_out/selprof.txt 2>&1
cat gpurun_out/selprof.txt
