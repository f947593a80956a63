python -m pytest tests/test_gpu_b256.py tests/test_gpu_parity.py tests/test_group_api.py -m gpu -q -k "mobilenet" > gpurun_out/g21_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/g21_pytest.log
for v in new old; do
  if [ $v = old ]; then L=_ab/old/libmrb200.so; else L=paper_1904_08368_b200/_lib/libmrb200.so; fi
  MRB200_LIB=$L python bench.py --model mobilenet_v1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/mb_$v.json 2>/dev/null
done
python - <<'PY'
import json
for v in ['new','old']:
    d=json.loads(open('gpurun_out/mb_%s.json'%v).read().strip().splitlines()[-1])
    dw=[x for x in d['bf16']['per_launch'] if x['kernel']=='dwconv']
    dwi=[x for x in d['per_launch'] if x['kernel']=='dwconv']
    print(v, 'bf16', round(d['bf16']['value']), round(d['bf16']['ms_per_step'],4), 'dw ms', round(sum(x['ms'] for x in dw),3), [x['frac'] for x in dw], 'int8', round(d['value']), 'dw int8 ms', round(sum(x['ms'] for x in dwi),3))
PY
