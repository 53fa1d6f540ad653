export GPCG_TRACE_OFF=1
timeout 600 python -m pytest tests -m gpu -x -q -k "stencil3d" 2>&1 | tail -1
timeout 300 python scripts/diag.py C4s C4s 2>&1 | tail -1 | cut -c1-150
mkdir -p gpurun_out; timeout 600 ncu --set full --clock-control none -k regex:"k7_" -c 3 -o gpurun_out/prof_m3b python scripts/diag.py C4s > /dev/null 2>&1; python scripts/ncu_summary.py gpurun_out/prof_m3b.ncu-rep; rm -f gpurun_out/prof_m3b.ncu-rep
