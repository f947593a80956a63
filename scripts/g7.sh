python tests/profile_run.py int8 256 2 > gpurun_out/g7_plain.log 2>&1 || exit 1
for d in 0 1 2 4 7 8; do
MRB200_DENSE_DBG=$d ncu --metrics gpu__time_duration.sum,smsp__cycles_active.avg,sm__cycles_elapsed.avg --clock-control none -k regex:"k_dense_tc" --csv --log-file gpurun_out/g7_$d.csv python tests/profile_run.py int8 256 2 > /dev/null 2>&1
echo "dbg=$d"; grep -E "k_dense_tc" gpurun_out/g7_$d.csv | awk -F'","' '{print $(NF-2), $NF}' | tail -3
done
