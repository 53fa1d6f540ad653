# bench line + launch list of the bench command + one ncu --set full capture of the k4 kernels
mkdir -p gpurun_out
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
export GPCG_TRACE_OFF=1
timeout 300 python scripts/diag.py C2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1
echo "ll rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k4_" -s 300 -c 6 -o gpurun_out/prof_${TAG} \
    python scripts/diag.py C2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
