set -x
timeout 600 python bench.py --config C4 --pop 64 --steps 4 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-repair > gpurun_out/e2e64.jsonl 2> gpurun_out/e2e64.err
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
python -c "
import json
d=json.loads(open('gpurun_out/e2e64.jsonl').read().strip().splitlines()[-1])
print('device ms/step', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], d['e2e']['steps_ms'])"
