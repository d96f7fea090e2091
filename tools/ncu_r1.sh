set -x
CMD="python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 40 -c 1 -o gpurun_out/prof_eval_r1 $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo ncu2_rc=$?
tail -2 gpurun_out/plain.log | cut -c1-600
