# device rounds per host poll (one CUDA graph launch each): 8 (default) vs 16 vs 32
run() {  # tag rps cfg pop
  MDR_RPS=$2 timeout 900 python bench.py --config $3 --pop $4 --steps 5 --warmup 3 --no-cpu-baseline --no-numpy-ref --no-repair > gpurun_out/r_$1_$3_$4.jsonl 2> gpurun_out/r_$1_$3_$4.err
}
for cfg in "C1 1" "C2 64" "C4 32" "C4 256"; do
  set -- $cfg
  for rep in 1 2; do
    for r in 8 4 2 16; do run rps${r}_$rep $r $1 $2; done
  done
done
for f in gpurun_out/r_*.jsonl; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1].ljust(28), round(d['value']/1e9,4), 'G/s', round(d['ms_per_step'],2), 'ms e2e', round(d['e2e']['value']/1e9,4))" 2>&1 | tail -1; done | sort > gpurun_out/r_summary.txt
cat gpurun_out/r_summary.txt
