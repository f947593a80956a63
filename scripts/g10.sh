python -m pytest tests/test_gpu_parity.py tests/test_gpu_b256.py tests/test_group_api.py -m gpu -q -x --deselect tests/test_gpu_b256.py::test_c5_batch4096_seeded_subset_matches_reference > gpurun_out/g10_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/g10_pytest.log
bash tests/ab_env.sh 2 "p4=X=0" "p9=MRB200_STEM_POOL9=1"
python -c "
import json
for n in ['p9','p4']:
    d=json.loads(open('gpurun_out/abe_%s_1.json'%n).read().strip().splitlines()[-1]); print(n, d['per_launch'][1]['ms_event'], d['plans']['fused21'][:80])"
BENCH_ARGS="--model mobilenet_v1" bash tests/ab_env.sh 1 "mb=X=0"
