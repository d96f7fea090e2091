# round-2: the new device rows (population selection, feasibility, construction) + full GPU suite + bench
set -x
timeout 600 python -m pytest tests/test_population.py tests/test_scalar_oracles.py tests/test_host_inputs.py tests/test_large_golden.py -q -m gpu -x -p no:cacheprovider > gpurun_out/gpu_new.log 2>&1; echo "new exit $?" >> gpurun_out/gpu_new.log
timeout 2400 python -m pytest tests -q -m gpu --durations=15 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
tail -5 gpurun_out/gpu_new.log; tail -30 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; cut -c1-1500 gpurun_out/bench.jsonl; tail -3 gpurun_out/bench.err; cut -c1-600 gpurun_out/bench_ref.jsonl; tail -3 gpurun_out/bench_ref.err
