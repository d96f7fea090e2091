# confirm the adopted k_select form (staged route rebuild, warp follower selection, 96-register CTAs) vs HEAD
set -x
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/s_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/s_tests.log
tail -2 gpurun_out/s_tests.log
bash tools/selprof_ab.sh
run() {  # tag lib cfg pop
  MDR_LIB=$PWD/paper_2605_05208_b200/$2 timeout 900 python bench.py --config $3 --pop $4 --steps 3 --warmup 3 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/s_$1_$3_$4.jsonl 2> gpurun_out/s_$1_$3_$4.err
}
for cfg in "C4 32" "C4 256" "C5 64" "C2 64"; do
  set -- $cfg
  for rep in 1 2; do
    run prev$rep libmdr_prev.so $1 $2
    run min1$rep libmdr_rbmin1.so $1 $2
    run new$rep libmdr_sm100.so $1 $2
  done
done
for f in gpurun_out/s_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1].ljust(26), round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', round(d['profile'].get('select_ms',0),1))" 2>&1 | tail -1; done | sort > gpurun_out/s_summary.txt
