# A/B of two library builds on the given configs (1 step each, two alternations)
# usage: bash tools/ab.sh "C2 C4 C5" libA.so libB.so
CFGS=$1; shift
for rep in 1 2; do
for C in $CFGS; do
for L in "$@"; do
  printf "%s %-28s " $C $L
  MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 300 python bench.py --config $C --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-repair 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['profile']
        print('value %.4g  ms/step %.1f  eval %.1f geval %.1f select %.1f'%(d['value'],d['ms_per_step'],p['eval_ms'],p.get('geval_ms',0),p['select_ms']))
    elif 'rror' in l: print(l.strip()[:300])
"
done; done; done
