python -m pytest tests -m gpu -q > gpurun_out/g12_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/g12_pytest.log
grep -E "FAILED" gpurun_out/g12_pytest.log | head
