python -m pytest tests/test_gpu_b256.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/g25_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/g25_pytest.log
for r in 1 2; do
for cfg in "cur:paper_1904_08368_b200/_lib/libmrb200.so:1" "cur_nosplit:paper_1904_08368_b200/_lib/libmrb200.so:0" "late:_ab/late/libmrb200.so:1"; do
  n=${cfg%%:*}; rest=${cfg#*:}; L=${rest%%:*}; SP=${rest#*:}
  MRB200_LIB=$L MRB200_SPLIT_B=$SP python bench.py --no-cpu-baseline --steps 100 --warmup 10 > gpurun_out/abx_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/abx_$n.json').read().strip().splitlines()[-1]); print('$n', $r, round(d['ms_per_step'],4), round(d['bf16']['ms_per_step'],4))"
done; done
python -c "
import json
a=json.loads(open('gpurun_out/abx_cur_nosplit.json').read().strip().splitlines()[-1]); b=json.loads(open('gpurun_out/abx_cur.json').read().strip().splitlines()[-1])
for x,y in zip(a['per_launch'],b['per_launch']):
    if abs(y['ms_event']/x['ms_event']-1)>0.03: print(x['launch'], x['ms_event'], y['ms_event'], b['plans'].get(x['launch'][1:],'')[:100])"
