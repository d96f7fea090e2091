# full-set capture of k_select on a config (default C2): early rounds (many followers) and a later one
CFG=${1:-C2}
CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-repair"
timeout 300 $CMD > gpurun_out/plain_sel.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_select -s 20 -c 3 -o gpurun_out/prof_sel_$CFG $CMD > gpurun_out/ncu_sel.log 2>&1
echo rc=$?
