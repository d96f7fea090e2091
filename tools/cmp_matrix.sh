# lib x env matrix on C4 (one step each)
run() { MDR_LIB=$PWD/paper_2605_05208_b200/$1 timeout 300 env $2 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-repair 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); p=d['profile']
        print('$1 $2 value %.4g  ms/step %.0f  eval %.0f geval %.0f select %.0f'%(d['value'],d['ms_per_step'],p['eval_ms'],p.get('geval_ms',0),p['select_ms']))
"; }
run libmdr_sm100.so MDR_X=1
run libmdr_sm100.so MDR_FORCE_OVERLAP=1
run libmdr_sm100_g3.so MDR_X=1
run libmdr_sm100_g3.so MDR_FORCE_OVERLAP=1
run libmdr_sm100_g4.so MDR_X=1
run libmdr_sm100_g4.so MDR_FORCE_OVERLAP=1
run libmdr_sm100_g2.so MDR_X=1
run libmdr_sm100_g2.so MDR_NO_OVERLAP=1
