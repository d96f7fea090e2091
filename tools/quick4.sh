for E in MDR_X=1 MDR_CARVEOUT=25 MDR_CARVEOUT=40; do
 timeout 600 env $E python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['profile']; print('$E value %.4g ms/step %.1f eval %.1f geval %.1f'%(d['value'], d['ms_per_step'],p['eval_ms'],p['geval_ms']))
    elif 'rror' in l: print(l.strip()[:300])
"
done
