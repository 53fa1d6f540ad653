# launch list (ncu gpu__time_duration per launch) of one C2 solve (+ optional full capture of a kernel)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 300 python scripts/diag.py ${CONFIG:-C2} > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-40000} --csv --log-file gpurun_out/launches_${TAG:-x}.csv \
    python scripts/diag.py ${CONFIG:-C2} > gpurun_out/ncu_ll.log 2>&1
echo "ll rc=$?"; cat gpurun_out/plain.log
if [ -n "$FULL" ]; then
ncu --set full --clock-control none --import-source on -k regex:"$FULL" -s ${SKIP:-50} -c ${NFULL:-3} -o gpurun_out/prof_${TAG:-x} \
    python scripts/diag.py ${CONFIG:-C2} > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
fi
