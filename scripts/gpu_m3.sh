# 3-D plane march: C4s timing (depth 2 / depth 3 / generic) + ncu of the depth-3 cauchy sweep
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
echo "depth2";  timeout 300 python scripts/diag.py C4s C4s 2>&1 | tail -1
echo "depth3"; GPCG_LIB=build_variants/libgpcg_m3d3.so timeout 300 python scripts/diag.py C4s C4s 2>&1 | tail -1
GPCG_LIB=build_variants/libgpcg_m3d3.so timeout 600 ncu --set full --clock-control none -k regex:"k7_" -c 3 -o gpurun_out/prof_m3d3 python scripts/diag.py C4s > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/prof_m3d3.ncu-rep
