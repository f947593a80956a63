python tests/profile_model.py mobilenet_v1 fp32 256 1 > gpurun_out/g16_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dw3x3 -s 1 -c 1 -o gpurun_out/g16_dw python tests/profile_model.py mobilenet_v1 fp32 256 1 > gpurun_out/g16_ncu.log 2>&1; echo rc=$?
