# source-level look at the relocate boundary kernel (summarised on the box)
CMD="python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_eval_c<[^,]*1, [^,]*0, [^,]*8, [^,]*32, [^,]*3, [^,]*2>" -s 100 -c 1 -o /tmp/prof_bnd $CMD > gpurun_out/ncu_bnd.log 2>&1
echo rc=$?
python tools/ncu_lines.py /tmp/prof_bnd.ncu-rep 0 60 > gpurun_out/bnd_lines.txt 2>&1
python tools/ncu_summary.py /tmp/prof_bnd.ncu-rep > gpurun_out/bnd_summary.txt 2>&1
ncu -i /tmp/prof_bnd.ncu-rep --page source --csv --print-source=sass > /tmp/bnd_sass.csv 2>/dev/null
python - <<'PY' > gpurun_out/bnd_mix.txt
import csv, collections, re
rows=list(csv.reader(open('/tmp/bnd_sass.csv')))
h=rows[1]; ie=h.index("Instructions Executed"); ws=h.index("Warp Stall Sampling (All Samples)")
cnt=collections.Counter(); st=collections.Counter(); tot=0; stot=0; full=collections.Counter()
for r in rows[2:]:
    if len(r) < len(h): continue
    try: n=float(r[ie]); s=float(r[ws] or 0)
    except ValueError: continue
    m=re.match(r'(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?', r[1].strip())
    if not m: continue
    cnt[m.group(2)]+=n; st[m.group(2)]+=s; tot+=n; stot+=s; full[m.group(2)+(m.group(3) or '')]+=n
print("total warp inst %.3e" % tot)
for k,v in cnt.most_common(25): print(f"{k:10s} {100*v/tot:5.1f}% inst {100*st[k]/max(stot,1):5.1f}% stall")
for k,v in full.most_common(25): print(f"{k:24s} {100*v/tot:5.1f}%")
PY
rm -f /tmp/prof_bnd.ncu-rep
head -30 gpurun_out/bnd_mix.txt
