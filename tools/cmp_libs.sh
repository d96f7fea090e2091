# quick A/B of library variants on C4 (1 step)
for L in libmdr_sm100.so libmdr_sm100_mb2.so libmdr_sm100_mb3.so; do
  echo "== $L"
  MDR_LIB=$PWD/paper_2605_05208_b200/$L timeout 300 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value %.3e  ms/step %.0f  eval_avg_ms %.3f  frac %.3f'%(d['value'],d['ms_per_step'],d['roofline']['eval_avg_launch_ms'],d['roofline']['frac']))
    elif 'Error' in l or 'error' in l: print(l.strip())
"
done
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
