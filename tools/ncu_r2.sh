# round-2 baseline captures: C4 and C5 full-set capture of one round's evaluators (source-level), C5 launch list
for CFG in C4 C5; do
  CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-repair"
  timeout 400 $CMD > gpurun_out/plain_$CFG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 300 -c 6 -o gpurun_out/prof_r2_$CFG $CMD > gpurun_out/ncu_r2_$CFG.log 2>&1
  echo "$CFG full_rc=$?"
done
CMD="python bench.py --config C5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-repair"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 2000 -c 1200 --csv --log-file gpurun_out/launches_r2_C5.csv $CMD > gpurun_out/ncu_launch_C5.log 2>&1
echo launch_rc=$?
tail -1 gpurun_out/plain_C4.log | cut -c1-300; tail -1 gpurun_out/plain_C5.log | cut -c1-300
