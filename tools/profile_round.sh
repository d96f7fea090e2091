# round-1 evidence: plain bench, ncu launch list (shares) and a full-set capture of 16 consecutive
# evaluation-phase launches (= exactly two rounds: 3 staged, 2 enumerators, 3 generic drains each)
CMD="python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_prof.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1600 --csv --log-file gpurun_out/launches_final.csv $CMD > gpurun_out/ncu_launch_final.log 2>&1
echo launch_rc=$?
timeout 300 $CMD > gpurun_out/plain_prof2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 300 -c 16 -o gpurun_out/prof_final $CMD > gpurun_out/ncu_final.log 2>&1
echo full_rc=$?
