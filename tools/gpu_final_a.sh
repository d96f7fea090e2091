# full GPU suite + smoke + default bench line + reference arm, then the evaluator captures
set -x
timeout 2400 python -m pytest tests -q -m gpu --durations=10 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
bash tools/ncu_r2c.sh
tail -4 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; cut -c1-300 gpurun_out/bench.jsonl; tail -3 gpurun_out/bench.err
