set -x
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.jsonl 2> gpurun_out/bench_ref.err
bash tools/sweep.sh > gpurun_out/sweep.txt 2>&1
tail -2 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log | tail -2; cut -c1-400 gpurun_out/bench_default.jsonl; cut -c1-300 gpurun_out/bench_ref.jsonl; cat gpurun_out/sweep.txt
