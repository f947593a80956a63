python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_b256.py::test_c5_batch4096_seeded_subset_matches_reference > gpurun_out/g5_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/g5_pytest.log
python tests/profile_run.py int8 256 2 > gpurun_out/g5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dense|sum_hw" --csv --log-file gpurun_out/g5_dense.csv python tests/profile_run.py int8 256 2 > /dev/null 2>&1
grep -E "dense|sum_hw" gpurun_out/g5_dense.csv | awk -F'","' '{print $5, $NF}' | head -20
