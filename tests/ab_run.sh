#!/bin/bash
# A/B timing of library variants under _ab/<name>/libmrb200.so (bench.py int8 line).
# usage: tests/ab_run.sh ROUNDS NAME...   -> gpurun_out/ab_<name>_<round>.json
rounds=$1; shift
for r in $(seq 1 $rounds); do
  for n in "$@"; do
    MRB200_LIB=_ab/$n/libmrb200.so python bench.py --no-cpu-baseline --no-bf16 --steps 200 --warmup 10 \
      > gpurun_out/ab_${n}_$r.json 2> gpurun_out/ab_${n}_$r.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab_${n}_$r.json').read().strip().splitlines()[-1]); print('$n', $r, round(d['ms_per_step'],4), round(d['value']))"
  done
done
