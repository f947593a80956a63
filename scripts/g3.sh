python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_b256.py > gpurun_out/g3_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g3_pytest.log
bash tests/ab_run.sh 3 base pre
