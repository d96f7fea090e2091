# usage: bash tools/ncu_eval.sh TAG  -- full ncu capture of one k_eval launch (C4 bench, 1 step)
TAG=${1:-x}
CMD="python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval -s 40 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
tail -1 gpurun_out/plain_$TAG.log | cut -c1-300
