python tests/profile_run.py int8 256 1 > gpurun_out/g11_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -c 1 -o gpurun_out/g11_p4 python tests/profile_run.py int8 256 1 > gpurun_out/g11_ncu.log 2>&1; echo rc=$?
MRB200_STEM_POOL9=1 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -c 1 -o gpurun_out/g11_p9 python tests/profile_run.py int8 256 1 > gpurun_out/g11_ncu9.log 2>&1; echo rc=$?
