# round-batch graph kept across calls (current) vs re-captured per call (prev); full GPU suite on current
set -x
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/s_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/s_tests.log
tail -2 gpurun_out/s_tests.log
run() {  # tag lib cfg pop
  MDR_LIB=$PWD/paper_2605_05208_b200/$2 timeout 900 python bench.py --config $3 --pop $4 --steps 10 --warmup 3 --no-cpu-baseline --no-numpy-ref --no-repair > gpurun_out/s_$1_$3_$4.jsonl 2> gpurun_out/s_$1_$3_$4.err
}
for cfg in "C1 1" "C2 64" "C4 32" "C3 128" "C4 256"; do
  set -- $cfg
  for rep in 1 2; do
    run prev$rep libmdr_prev.so $1 $2
    run cur$rep libmdr_sm100.so $1 $2
  done
done
for f in gpurun_out/s_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1].ljust(26), round(d['value']/1e9,4), 'G/s', round(d['ms_per_step'],2), 'ms e2e', round(d['e2e']['value']/1e9,4), (d.get('parity_checked') or {}).get('bit_exact'))" 2>&1 | tail -1; done | sort > gpurun_out/s_summary.txt
