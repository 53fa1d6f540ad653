# diag A/B (tile vs column march), launch list and one ncu --set full capture of the tile kernels (C2)
mkdir -p gpurun_out
timeout 300 python scripts/diag.py C0 C1 C2 > gpurun_out/diag_tile.log 2>&1
GPCG_TILE=0 timeout 300 python scripts/diag.py C0 C1 C2 > gpurun_out/diag_march.log 2>&1
grep -h "solve" gpurun_out/diag_tile.log gpurun_out/diag_march.log
export GPCG_TRACE_OFF=1
timeout 300 python scripts/diag.py C2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/launches_C2.csv \
    python scripts/diag.py C2 > gpurun_out/ncu_ll.log 2>&1
echo "ll rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k3_ -s 400 -c 6 -o gpurun_out/prof_k3_C2 \
    python scripts/diag.py C2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
