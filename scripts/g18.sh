python -m pytest tests -m gpu -q -x > gpurun_out/g18_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/g18_pytest.log
bash tests/ab_env.sh 3 "fuse=X=0" "nofuse=MRB200_NO_SUM_FUSE=1"
python -c "
import json
for n in ['nofuse','fuse']:
    d=json.loads(open('gpurun_out/abe_%s_1.json'%n).read().strip().splitlines()[-1])
    print(n, [(x['kernel'], x['ms_event']) for x in d['per_launch'][-3:]])"
