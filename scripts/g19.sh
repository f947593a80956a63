bash tests/ab_env.sh 2 "cur=X=0" "tl=MRB200_LIB=_ab/tl/libmrb200.so"
MRB200_LIB=_ab/tl/libmrb200.so MRB200_TC_DBG=2048 python tests/profile_run.py int8 256 1 2> gpurun_out/g19_tl.log >/dev/null; echo tl rc=$?
