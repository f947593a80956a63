python -m pytest tests/test_gpu_parity.py tests/test_gpu_b256.py tests/test_group_api.py -m gpu -q > gpurun_out/g23_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/g23_pytest.log; grep FAILED gpurun_out/g23_pytest.log | head
python bench.py --model vgg16_b256 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/vgg.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/vgg.json').read().strip().splitlines()[-1]); print(round(d['value']), d['ms_per_step'])
print([(x['launch'], x['kernel'], x['ms'], x['frac']) for x in d['per_launch'][:3]]); print(d['plans']['fused20'])"
