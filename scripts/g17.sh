python bench.py --model vgg16_b256 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/vgg.json 2>gpurun_out/vgg.err; echo rc=$?
MRB200_NO_DENSE_TC=1 python bench.py --model vgg16_b256 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/vgg_simt.json 2>/dev/null
python bench.py --model dqn_b256 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/dqn.json 2>/dev/null
python - <<'PY'
import json
for f in ['vgg','vgg_simt','dqn']:
    d=json.loads(open('gpurun_out/%s.json'%f).read().strip().splitlines()[-1])
    print(f, d['config']['workload'], round(d['value']), round(d['ms_per_step'],3))
    for x in d['per_launch']:
        if 'dense' in x['kernel']: print('   ', x['launch'], x['kernel'], x['ms'], x['roof_ms'], x['frac'])
PY
