# 1000-case descent and repair fuzz on the current kernels (small and large evaluator shapes)
MDR_FUZZ_N=1000 timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_repair.py -q -m gpu -k "fuzz" -p no:cacheprovider > gpurun_out/fuzz1000.log 2>&1; echo "fuzz exit $?" >> gpurun_out/fuzz1000.log
tail -3 gpurun_out/fuzz1000.log
