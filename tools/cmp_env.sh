# A/B of environment settings on C2 / C3 (one step each): bash tools/cmp_env.sh "MDR_X=1" "MDR_GDIV=3" ...
for E in "$@"; do for c in C2 C3; do
  timeout 300 env $E python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --no-repair 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['profile']
        print('$E $c value %.4g  ms/step %.1f  eval %.1f geval %.1f select %.1f'%(d['value'],d['ms_per_step'],p['eval_ms'],p.get('geval_ms',0),p['select_ms']))
    elif 'rror' in l: print(l.strip()[:300])
"
done; done
