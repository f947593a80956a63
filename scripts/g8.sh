python -m pytest tests/test_gpu_parity.py tests/test_gpu_b256.py -m gpu -q -x --deselect tests/test_gpu_b256.py::test_c5_batch4096_seeded_subset_matches_reference > gpurun_out/g8_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/g8_pytest.log
bash tests/ab_env.sh 3 "pipe=MRB200_RES_PIPE=1" "nopipe=MRB200_RES_PIPE=0"
python - <<'PY'
import json
def load(n):
    return json.loads(open('gpurun_out/abe_%s_1.json'%n).read().strip().splitlines()[-1])
b,m=load('nopipe'),load('pipe')
for x,y in zip(b['per_launch'],m['per_launch']):
    print(x['launch'][:20].ljust(20), x['kernel'][:22].ljust(22), x['ms_event'], y['ms_event'], round(y['ms_event']/x['ms_event'],3))
PY
