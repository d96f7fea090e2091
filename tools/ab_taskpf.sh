# thread 0 claims the CTA's next task while the current one runs (current) vs claiming at the boundary (prev)
set -x
timeout 1500 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py tests/test_large_golden.py -q -m gpu -x -p no:cacheprovider > gpurun_out/s_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/s_tests.log
run() {  # tag lib cfg pop
  MDR_LIB=$PWD/paper_2605_05208_b200/$2 timeout 900 python bench.py --config $3 --pop $4 --steps 5 --warmup 3 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/s_$1_$3_$4.jsonl 2> gpurun_out/s_$1_$3_$4.err
}
for cfg in "C4 256" "C4 32" "C5 64" "C2 64"; do
  set -- $cfg
  for rep in 1 2; do
    run prev$rep libmdr_prev.so $1 $2
    run cur$rep libmdr_sm100.so $1 $2
  done
done
for f in gpurun_out/s_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1].ljust(26), round(d['value']/1e9,4), 'G/s', round(d['ms_per_step'],2), 'ms')" 2>&1 | tail -1; done | sort > gpurun_out/s_summary.txt
