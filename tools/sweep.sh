# bench line for every BASELINE config on one B200: C1 single descent, C2/C3/C4 at their populations,
# C5 at its 8-GPU shard (512 / 8 = 64) and the C4 strong-scaling shards (256 / N for N = 2, 4, 8)
out=gpurun_out/sweep.jsonl; : > $out
for spec in "C1 1" "C2 64" "C3 128" "C4 256" "C5 64" "C4 128" "C4 64" "C4 32"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --pop $2 --steps 2 --warmup 3 --no-repair --no-numpy-ref >> $out 2> gpurun_out/sweep_$1_$2.err || echo "{\"config\": \"$1\", \"failed\": true}" >> $out
done
cat $out | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if d.get('failed'): print(d); continue
    c = d['cpu_baseline'] or {}
    print(d['config']['workload'][:3], 'pop', d['config']['population'], 'value %.4g e2e %.4g desc/s %.1f cpu %.3g e2e/cpu %.0f parity %s' % (
        d['value'], d['e2e']['value'], d['descents_per_s'], c.get('value', 0), d['e2e']['value'] / c['value'] if c else 0,
        (d.get('parity_checked') or {}).get('bit_exact')))
"
