set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_b256.py > gpurun_out/g1_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/g1_pytest.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/g1_bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['bf16']['value'])"
python tests/profile_run.py int8 256 1 > gpurun_out/g1_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 1 -c 1 -o gpurun_out/g1_l1ga python tests/profile_run.py int8 256 1 > gpurun_out/g1_ncu.log 2>&1; echo ncu rc=$?
