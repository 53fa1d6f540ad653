# bench line + paper-setting runs + launch list (one C2 solve) + ncu --set full of the persistent kernels
mkdir -p gpurun_out
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 900 python scripts/paper_setting.py --out gpurun_out/paper_setting.json > gpurun_out/paper_setting.log 2>&1; echo "paper rc=$?"
export GPCG_TRACE_OFF=1
timeout 300 python scripts/diag.py C2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python scripts/diag.py C2 > gpurun_out/ncu_ll.log 2>&1
echo "ll rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_" -s 60 -c 2 -o gpurun_out/prof_${TAG} \
    python scripts/diag.py C2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
