#!/bin/bash
# A/B timing of environment settings with one library (bench.py int8 line):
#   tests/ab_env.sh ROUNDS "NAME=ENV1=v1,ENV2=v2" "NAME2=..." ...  -> gpurun_out/abe_<name>_<round>.json
rounds=$1; shift
for r in $(seq 1 $rounds); do
  for spec in "$@"; do
    n=${spec%%=*}; envs=${spec#*=}
    env $(echo $envs | tr ',' ' ') python bench.py --no-cpu-baseline --no-bf16 --steps 200 --warmup 10 ${BENCH_ARGS} \
      > gpurun_out/abe_${n}_$r.json 2> gpurun_out/abe_${n}_$r.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/abe_${n}_$r.json').read().strip().splitlines()[-1]); print('$n', $r, round(d['ms_per_step'],4), round(d['value']))"
  done
done
