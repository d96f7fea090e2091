# round-2: drop-in boundary tests, on_feasible replay, full GPU suite, bench
set -x
timeout 900 python -m pytest tests/test_dropin.py "tests/test_gpu_parity.py::test_on_feasible_per_state_and_attrs" -q -m gpu -p no:cacheprovider > gpurun_out/gpu_dropin.log 2>&1; echo "dropin exit $?" >> gpurun_out/gpu_dropin.log
timeout 2400 python -m pytest tests -q -m gpu --durations=10 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-numpy-ref > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
tail -30 gpurun_out/gpu_dropin.log; tail -8 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; cut -c1-400 gpurun_out/bench.jsonl; tail -3 gpurun_out/bench.err
