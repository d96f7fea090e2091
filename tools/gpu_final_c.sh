# round-2 final numbers: driver-shaped bench + reference arm, all-config sweep with shards, 1000-case fuzz
set -x
timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_final.jsonl 2> gpurun_out/bench_final.err
timeout 1800 python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/bench_ref_final.jsonl 2> gpurun_out/bench_ref_final.err
bash tools/sweep.sh
bash tools/fuzz1000.sh
cut -c1-300 gpurun_out/bench_final.jsonl; tail -3 gpurun_out/bench_final.err
