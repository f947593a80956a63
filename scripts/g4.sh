python -m pytest tests -m gpu -q --deselect tests/test_gpu_b256.py::test_c5_batch4096_seeded_subset_matches_reference > gpurun_out/g4_pytest.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/g4_pytest.log | grep -E "passed|failed|FAIL|Error" | head -30
python -m pytest tests/test_gpu_b256.py -m gpu -q -s --deselect tests/test_gpu_b256.py::test_c5_batch4096_seeded_subset_matches_reference 2>&1 | grep -E "int8 b|bf16 b|passed|failed" | head -20
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g4_bench.json 2> gpurun_out/g4_bench.err; echo bench rc=$?
python -c "
import json;d=json.load(open('gpurun_out/g4_bench.json'));print(d['value'],d['ms_per_step'],d['bf16']['value'])
for x in d['per_launch'][-3:]: print(x)
print(d['plans']['fused0'])"
