# round-2 captures of the current evaluators (C4, C5): staged evaluators only, a mid-descent round
for CFG in C4 C5; do
  POP=$([ $CFG = C5 ] && echo "--pop 128" || echo "")
  CMD="python bench.py --config $CFG $POP --steps 1 --warmup 0 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair"
  timeout 600 $CMD > gpurun_out/plain2_$CFG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_eval_c -s 150 -c 3 -o gpurun_out/prof2_$CFG $CMD > gpurun_out/ncu2_$CFG.log 2>&1
  echo "$CFG rc=$?"
done
CMD="python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline --no-numpy-ref --no-e2e --no-repair"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 2000 -c 1600 --csv --log-file gpurun_out/launches2_C4.csv $CMD > gpurun_out/ncu_launch2.log 2>&1
echo launch rc=$?
