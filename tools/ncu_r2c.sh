# round-2 captures of every staged evaluator kernel (C4, C5), mid-descent rounds; the reports are
# summarised on the box (ncu_roofline.py / ncu_summary.py) and deleted, only the summaries come back
export NCU_ROOFLINE_OUT=$PWD/gpurun_out/ncu_roofline.json
cp profiles/ncu_roofline.json $NCU_ROOFLINE_OUT 2>/dev/null
for CFG in C4 C5; do
  POP=$([ $CFG = C5 ] && echo "--pop 128" || echo "")
  CMD="python bench.py --config $CFG $POP --steps 1 --warmup 0 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair"
  timeout 600 $CMD > gpurun_out/plain3_$CFG.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_eval_[cp]" -s 200 -c 8 -o /tmp/prof3_$CFG $CMD > gpurun_out/ncu3_$CFG.log 2>&1
  echo "$CFG rc=$?"
  W=$([ $CFG = C5 ] && echo 0 || echo 1)
  python tools/ncu_roofline.py $CFG /tmp/prof3_$CFG.ncu-rep "k_eval_c<$W, 0, \d+, 32, \d+, 1>" relocate_granular > /dev/null
  python tools/ncu_roofline.py $CFG /tmp/prof3_$CFG.ncu-rep "k_eval_c<$W, 0, \d+, 32, \d+, 2>" relocate_boundary > /dev/null
  python tools/ncu_roofline.py $CFG /tmp/prof3_$CFG.ncu-rep "k_eval_c<$W, 0, \d+, 32, \d+, 0>" relocate > /dev/null
  python tools/ncu_roofline.py $CFG /tmp/prof3_$CFG.ncu-rep "k_eval_[cp]<$W, 1, " swap > /dev/null
  python tools/ncu_roofline.py $CFG /tmp/prof3_$CFG.ncu-rep "k_eval_c<$W, 2, " two_opt_star > /dev/null
  python tools/ncu_summary.py /tmp/prof3_$CFG.ncu-rep > gpurun_out/r2_ncu_${CFG}_summary.txt 2>&1
  ncu -i /tmp/prof3_$CFG.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread > gpurun_out/r2_ncu_${CFG}_kernels.csv 2>&1
  rm -f /tmp/prof3_$CFG.ncu-rep
done
