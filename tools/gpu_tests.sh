# GPU parity suite + smoke + one default bench line (round dev loop)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-repair > gpurun_out/bench_quick.jsonl 2> gpurun_out/bench_quick.err
tail -25 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; cut -c1-600 gpurun_out/bench_quick.jsonl; tail -3 gpurun_out/bench_quick.err
