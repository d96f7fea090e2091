# relocate families in the pipelined form (MDR_REL_FAM_PIPE bit 0 granular, bit 1 boundary) vs k_eval_c
set -x
run() {  # tag env cfg pop
  env $2 timeout 900 python bench.py --config $3 --pop $4 --steps 3 --warmup 3 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair > gpurun_out/s_$1_$3_$4.jsonl 2> gpurun_out/s_$1_$3_$4.err
}
for cfg in "C4 256" "C4 32"; do
  set -- $cfg
  for rep in 1 2; do
    run p0$rep MDR_REL_FAM_PIPE=0 $1 $2
    run p1$rep MDR_REL_FAM_PIPE=1 $1 $2
    run p2$rep MDR_REL_FAM_PIPE=2 $1 $2
    run p3$rep MDR_REL_FAM_PIPE=3 $1 $2
  done
done
for f in gpurun_out/s_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); e=d['profile']['evaluators_ms']
print('$f'.split('/')[-1].ljust(26), round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],1), 'ms', (d.get('parity_checked') or {}).get('bit_exact'), {k: round(v,1) for k,v in e.items()})" 2>&1 | tail -1; done | sort > gpurun_out/s_summary.txt
MDR_REL_FAM_PIPE=3 timeout 900 python -m pytest tests/test_gpu_shapes.py -q -m gpu -x -p no:cacheprovider > gpurun_out/s_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/s_tests.log
