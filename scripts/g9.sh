python tests/profile_run.py int8 256 1 > gpurun_out/g9_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 2 -c 1 -o gpurun_out/g9_l1gb python tests/profile_run.py int8 256 1 > gpurun_out/g9_ncu.log 2>&1; echo rc=$?
