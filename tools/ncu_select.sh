CMD="python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_sel.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_select -s 100 -c 2 -o gpurun_out/prof_sel $CMD > gpurun_out/ncu_sel.log 2>&1
echo rc=$?
