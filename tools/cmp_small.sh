# A/B of library variants on the small configs (C2, C3) and C4, one step each
for L in libmdr_sm100.so libmdr_sm100_g2.so libmdr_sm100_g3.so libmdr_sm100_g4.so; do
  for c in C2 C3 C4; do
  MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 300 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-repair 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['profile']
        print('$L $c value %.4g  ms/step %.1f  eval %.1f geval %.1f select %.1f'%(d['value'],d['ms_per_step'],p['eval_ms'],p.get('geval_ms',0),p['select_ms']))
    elif 'rror' in l: print(l.strip()[:300])
"
  done
done
