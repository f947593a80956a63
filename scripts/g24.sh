MRB200_LIB=_ab/tl/libmrb200.so MRB200_TC_DBG=2052 python tests/profile_run.py int8 256 1 2> gpurun_out/g24_nomma.log >/dev/null; echo rc=$?
MRB200_LIB=_ab/tl/libmrb200.so MRB200_TC_DBG=2049 python tests/profile_run.py int8 256 1 2> gpurun_out/g24_noepi.log >/dev/null; echo rc=$?
