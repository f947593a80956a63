#!/bin/bash
# Round-end measurement bundle (run on the B200 via gpurun, one GPU):
#   bench line (C2 headline), C5 strong-scaling line (batch 4096 through the shard path),
#   launch list (ncu, after the same command ran clean), DRAM traffic per kernel family,
#   ncu --set full of EVERY tcgen05 conv launch of one int8 step (20) + the other
#   kernel families, side benches of the other BASELINE configs.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err || exit 1
python bench.py --global-batch 4096 --no-cpu-baseline --no-bf16 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2>/dev/null
python bench.py --no-cuda-graph --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_nograph.json 2>/dev/null || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --no-cuda-graph --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tests/profile_run.py int8 256 1 > gpurun_out/profile_run.log 2>&1 || exit 1
for p in int8 fp32; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/traffic_$p.csv python tests/profile_run.py $p 256 1 > /dev/null 2>&1
done
ncu --set full --clock-control none -k regex:"k_conv_tc|k_dense_tc|k_sum_hw|k_input" -c 25 \
    -o gpurun_out/conv_full python tests/profile_run.py int8 256 1 > gpurun_out/ncu_full.log 2>&1
# reports are large: keep their raw pages (what profiles/ summarises), not the reports
ncu -i gpurun_out/conv_full.ncu-rep --page raw --csv > gpurun_out/conv_full_raw.csv && rm -f gpurun_out/conv_full.ncu-rep
python tests/profile_model.py mobilenet_v1 fp32 256 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none -k regex:"k_dw3x3" -c 13 -o gpurun_out/dw_full \
    python tests/profile_model.py mobilenet_v1 fp32 256 1 > gpurun_out/ncu_dw.log 2>&1
ncu -i gpurun_out/dw_full.ncu-rep --page raw --csv > gpurun_out/dw_full_raw.csv && rm -f gpurun_out/dw_full.ncu-rep
python bench.py --model mobilenet_v1 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/bench_mbv1.json 2>/dev/null
python bench.py --model vgg16_b256 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_vgg.json 2>/dev/null
python bench.py --model dqn_b256 --no-cpu-baseline --steps 100 --warmup 5 > gpurun_out/bench_dqn.json 2>/dev/null
echo done
