set -x
timeout 600 python tools/e2e_steps.py > gpurun_out/e2e_steps.txt 2>&1
timeout 1500 python -m pytest tests/test_engine.py tests/test_population.py tests/test_scalar_oracles.py tests/test_formats.py tests/test_dropin.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/fix_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/fix_tests.log
tail -14 gpurun_out/e2e_steps.txt; tail -3 gpurun_out/fix_tests.log
