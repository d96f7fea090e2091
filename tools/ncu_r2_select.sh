# k_select at the strong-scaling shard (C4 population 32 = 256/8): early round and tail round captures
CMD="python bench.py --config C4 --pop 32 --steps 1 --warmup 0 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair"
timeout 300 $CMD > gpurun_out/plain_sel32.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_select -s 30 -c 1 -o gpurun_out/prof_sel32_early $CMD > gpurun_out/ncu_sel32a.log 2>&1
echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_select -s 700 -c 1 -o gpurun_out/prof_sel32_tail $CMD > gpurun_out/ncu_sel32b.log 2>&1
echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 1600 --csv --log-file gpurun_out/launches_C4_p32.csv $CMD > gpurun_out/ncu_launch32.log 2>&1
echo rc=$?
