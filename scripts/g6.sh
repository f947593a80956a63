python tests/profile_run.py int8 256 1 > gpurun_out/g6_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dense_tc -c 1 -o gpurun_out/g6_dense python tests/profile_run.py int8 256 1 > gpurun_out/g6_ncu.log 2>&1; echo rc=$?
