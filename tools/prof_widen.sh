# widened rows: plain run, then an ncu launch list and a full capture of k_neighbors / k_repair
timeout 300 python tools/prof_widen.py > gpurun_out/widen_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/widen_launches.csv \
  python tools/prof_widen.py > gpurun_out/widen_launch.log 2>&1
echo launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_neighbors|k_repair" -c 2 \
  -o gpurun_out/prof_widen python tools/prof_widen.py > gpurun_out/widen_full.log 2>&1
echo full_rc=$?
