timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1 | cut -c1-80
for c in C2 C3 C4; do for g in 1; do
 if [ $g = 0 ]; then E="MDR_NO_GRAPH=1"; else E="MDR_X=1"; fi
 timeout 600 env $E python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$c graph=$g value %.4g e2e %.4g ms/step %.1f'%(d['value'], d['e2e']['value'], d['ms_per_step']))
    elif 'rror' in l: print(l.strip()[:300])
"
done; done
