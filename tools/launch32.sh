CMD="python bench.py --config C4 --pop 32 --steps 1 --warmup 0 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 2400 --csv --log-file gpurun_out/launches_p32.csv $CMD > gpurun_out/ncu_l32.log 2>&1
echo rc=$?
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/launches_p32.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
tot=collections.Counter(); cnt=collections.Counter()
for r in rows[1:]:
    try: v=float(r[vi].replace(',',''))
    except: continue
    n=r[ki].split('(')[0].replace('void ','')
    tot[n]+=v; cnt[n]+=1
T=sum(tot.values())
for k,v in tot.most_common(): print(f"{k:40s} n={cnt[k]:5d} share={100*v/T:5.1f}% avg={v/cnt[k]/1e3:8.1f} us")
PY
