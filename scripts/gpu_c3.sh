# C3 (8000^2, 64M unknowns) on one B200 + ncu traffic of fixed-length CG calls on C2 and C3
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 900 python scripts/diag.py C3 > gpurun_out/diag_c3.log 2>&1; echo "c3 rc=$?"; grep -E "solve|Error" gpurun_out/diag_c3.log
timeout 300 python scripts/cg_traffic.py 64 > gpurun_out/cg_traffic_plain.log 2>&1 && cat gpurun_out/cg_traffic_plain.log && \
timeout 600 ncu --set full --clock-control none -k regex:"k6_cg_loop" -c 1 -o gpurun_out/prof_cgtraffic python scripts/cg_traffic.py 64 > gpurun_out/ncu_cgtraffic.log 2>&1
echo "ncu rc=$?"
