bash tests/ab_env.sh 2 "cur=X=0" "trs2=MRB200_TRS_MIN=2"
python - <<'PY'
import json
b=json.loads(open('gpurun_out/abe_cur_1.json').read().strip().splitlines()[-1]); m=json.loads(open('gpurun_out/abe_trs2_1.json').read().strip().splitlines()[-1])
for x,y in zip(b['per_launch'],m['per_launch']):
    if abs(y['ms_event']/x['ms_event']-1)>0.02: print(x['launch'], x['ms_event'], y['ms_event'], round(y['ms_event']/x['ms_event'],3), m['plans'].get(x['launch'][1:],'')[:90])
PY
