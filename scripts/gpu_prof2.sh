# launch list (first NLAUNCH launches of one C2 solve) + ncu --set full of the three hot kernels
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 300 python scripts/diag.py C2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-8000} --csv --log-file gpurun_out/launches_${TAG}.csv \
    python scripts/diag.py C2 > gpurun_out/ncu_ll.log 2>&1
echo "ll rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k5_|k4_cg}" -s ${SKIP:-600} -c ${NFULL:-6} -o gpurun_out/prof_${TAG} \
    python scripts/diag.py C2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
