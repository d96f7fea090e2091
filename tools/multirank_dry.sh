# functional check of the N>1 bench flow on one box: 2 ranks sharing the GPU over gloo (not a scaling number)
set -x
MDR_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config C4 --steps 2 --warmup 1 --no-cpu-baseline --no-numpy-ref --no-repair > gpurun_out/mr.jsonl 2> gpurun_out/mr.err; echo "mr exit $?"
MDR_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 --no-numpy-ref > gpurun_out/mr_ref.jsonl 2> gpurun_out/mr_ref.err; echo "mr ref exit $?"
cut -c1-700 gpurun_out/mr.jsonl; tail -5 gpurun_out/mr.err; cut -c1-300 gpurun_out/mr_ref.jsonl; tail -3 gpurun_out/mr_ref.err
