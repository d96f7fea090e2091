for L in selprof; do
  echo "== $L"; MDR_LIB=$PWD/paper_2605_05208_b200/libmdr_$L.so timeout 600 python tools/selprof.py 32 2>&1 | tail -9
done > gpurun_out/selprof_ab.txt
cat gpurun_out/selprof_ab.txt
