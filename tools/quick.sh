# GPU parity suite + one C4 bench step (dev loop); extra args: env assignments for an A/B run
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1 | cut -c1-80
run() {
timeout 600 env "$@" python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['profile']
        print('value %.4g  ms/step %.0f  eval %.0f geval %.0f select %.0f plan %.0f (ms/step) frac %.3f rounds %d'%(d['value'],d['ms_per_step'],p['eval_ms'],p.get('geval_ms',0),p['select_ms'],p['plan_ms'],d['roofline']['frac'],p['rounds_per_step']))
    elif 'rror' in l: print(l.strip()[:300])
"
}
run MDR_X=1
for v in "$@"; do echo "== $v"; run $v; done
