# source-level look at the intra-route swap drain (k_eval_g, queue region 2) on C5 and C4 (summarised on the box)
for spec in "C5 64 0" "C4 256 1"; do
  set -- $spec
  CMD="python bench.py --config $1 --pop $2 --steps 1 --warmup 0 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_eval_g<[^,]*$3, [^,]*1>" -s 300 -c 1 -o /tmp/prof_g $CMD > gpurun_out/ncu_g_$1.log 2>&1
  echo rc=$?
  python tools/ncu_lines.py /tmp/prof_g.ncu-rep 0 60 > gpurun_out/g_lines_$1.txt 2>&1
  python tools/ncu_summary.py /tmp/prof_g.ncu-rep > gpurun_out/g_summary_$1.txt 2>&1
  rm -f /tmp/prof_g.ncu-rep
done
head -40 gpurun_out/g_summary_C5.txt
