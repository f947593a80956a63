MRB200_SYNC_DEBUG=1 python tests/sanitize_run.py > gpurun_out/g13_plain.log 2>&1; echo plain rc=$?; cat gpurun_out/g13_plain.log | tail -5
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "combine" > gpurun_out/g13_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/g13_pytest.log
