# bench line for every BASELINE config (one B200): C1 single descent, C2/C3/C4 at their populations,
# C5 at its per-GPU share (512 over 8 GPUs = 64)
out=gpurun_out/sweep.jsonl; : > $out
for spec in "C1 1" "C2 64" "C3 128" "C4 256" "C5 64"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --pop $2 --steps 2 --warmup 3 --no-repair >> $out 2> gpurun_out/sweep_$1.err || echo "{\"config\": \"$1\", \"failed\": true}" >> $out
done
cat $out | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if d.get('failed'): print(d); continue
    print(d['config']['workload'][:40], 'value %.3g e2e %.3g desc/s %.1f cpu %.3g l2 %.2f' % (d['value'], d['e2e']['value'], d['descents_per_s'], (d['cpu_baseline'] or {}).get('value', 0), d['roofline']['l2']['frac']))
"
