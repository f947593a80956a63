#!/bin/bash
# Round-end measurement bundle (run on the B200 via gpurun, one GPU):
#   bench line, launch list (ncu, after the same command ran clean), DRAM traffic per
#   kernel family, one --set full capture of the first conv launches, side benches.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err || exit 1
python bench.py --no-cuda-graph --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_nograph.json 2>/dev/null || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --no-cuda-graph --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
for p in int8 fp32; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/traffic_$p.csv python tests/profile_run.py $p 256 1 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -c 3 -o gpurun_out/conv_full \
    python tests/profile_run.py int8 256 1 > gpurun_out/ncu_full.log 2>&1
python bench.py --batch 4096 --no-cpu-baseline --no-bf16 --steps 20 --warmup 3 > gpurun_out/bench_b4096.json 2>/dev/null
python bench.py --model mobilenet_v1 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/bench_mbv1.json 2>/dev/null
echo done
