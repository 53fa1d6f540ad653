# C3-scale (64M unknowns, HBM-bound) ncu captures: one fixed-length CG call (16 iterations) and one GP phase
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 600 python scripts/cg_traffic.py 16 C3 > gpurun_out/c3_plain.log 2>&1 && cat gpurun_out/c3_plain.log && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k6_" -c 2 -o gpurun_out/prof_c3 python scripts/cg_traffic.py 16 C3 > gpurun_out/ncu_c3.log 2>&1
echo "ncu rc=$?"
