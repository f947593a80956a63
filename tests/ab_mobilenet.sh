#!/bin/bash
# A/B of library variants on MobileNet-v1 (bench.py --model mobilenet_v1): int8 and bf16
# images/s plus the depthwise launches' summed per-launch ms.  usage: tests/ab_mobilenet.sh NAME...
for n in "$@"; do
  MRB200_LIB=_ab/$n/libmrb200.so python bench.py --model mobilenet_v1 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/mb_$n.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/mb_$n.json').read().strip().splitlines()[-1]); print('$n', round(d['value']), round(d['bf16']['value']), round(sum(L['ms'] for L in d['bf16']['per_launch'] if L['kernel']=='dwconv'),4), round(sum(L['ms'] for L in d['per_launch'] if L['kernel']=='dwconv'),4))"
done
