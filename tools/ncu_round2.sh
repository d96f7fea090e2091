# full capture of one round's evaluation kernels (C4 bench, 1 step)
TAG=${1:-x}
CMD="python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 300 -c 6 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
