# closing run after the graph cache: GPU suite, smoke, driver-shaped bench + reference arm, ncu captures, sweep
set -x
timeout 2400 python -m pytest tests -q -m gpu --durations=10 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_final.jsonl 2> gpurun_out/bench_final.err
timeout 1800 python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/bench_ref_final.jsonl 2> gpurun_out/bench_ref_final.err
timeout 300 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err
rm -f gpurun_out/sweep.jsonl
bash tools/sweep.sh > gpurun_out/sweep.txt 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; cut -c1-300 gpurun_out/bench_final.jsonl; cut -c1-200 gpurun_out/bench_default.jsonl
