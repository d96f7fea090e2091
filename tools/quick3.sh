for c in C2 C3; do for E in MDR_X=1 MDR_NO_STAGED=1; do
 timeout 600 env $E MDR_ROUND_LOG=gpurun_out/rounds_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['profile']; print('$c $E value %.4g ms/step %.1f eval %.1f geval %.1f sel %.1f plan %.1f rounds %d'%(d['value'], d['ms_per_step'],p['eval_ms'],p['geval_ms'],p['select_ms'],p['plan_ms'],p['rounds_per_step']))
    elif 'rror' in l: print(l.strip()[:300])
"
done; done
