set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_engine.py tests/test_dropin.py tests/test_session.py -q -m gpu -x -p no:cacheprovider > gpurun_out/pack_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/pack_tests.log
timeout 600 python tools/e2e_profile.py 256 > gpurun_out/e2e_prof256.txt 2>&1
timeout 900 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-numpy-ref --no-repair > gpurun_out/pack_bench.jsonl 2> gpurun_out/pack_bench.err
tail -2 gpurun_out/pack_tests.log; head -22 gpurun_out/e2e_prof256.txt
python -c "
import json
d=json.loads(open('gpurun_out/pack_bench.jsonl').read().strip().splitlines()[-1])
print('device', d['value']/1e9, d['ms_per_step'], 'e2e', d['e2e']['value']/1e9, d['e2e']['ms_per_step'], d['e2e']['steps_ms'])"
