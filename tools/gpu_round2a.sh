# round-2 first GPU pass: the full GPU suite (incl. large-shape / C4 / C5 parity), smoke, quick bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu --durations=25 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_quick.jsonl 2> gpurun_out/bench_quick.err
tail -40 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; cut -c1-900 gpurun_out/bench_quick.jsonl; tail -3 gpurun_out/bench_quick.err
