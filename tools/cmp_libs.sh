# quick A/B of library variants on C4 (1 step)
for L in libmdr_sm100.so libmdr_sm100_g2.so libmdr_sm100_g3.so libmdr_sm100_g4.so; do
  echo "== $L"
  MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 300 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['profile']
        print('value %.4g  ms/step %.0f  eval %.0f geval %.0f select %.0f'%(d['value'],d['ms_per_step'],p['eval_ms'],p.get('geval_ms',0),p['select_ms']))
    elif 'rror' in l: print(l.strip()[:300])
"
done
