# launch list + full capture of one round's evaluation kernels (C4 bench, 1 step)
TAG=${1:-x}
CMD="python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 300 -c 6 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1800 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo ncu2_rc=$?
tail -1 gpurun_out/plain_$TAG.log | cut -c1-200
