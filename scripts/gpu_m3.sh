export GPCG_TRACE_OFF=1
echo "default"; timeout 300 python scripts/diag.py C4s C4s 2>&1 | tail -1 | cut -c1-170
echo "async cauchy"; GPCG_LIB=build_variants/libgpcg_m3async.so timeout 300 python scripts/diag.py C4s C4s 2>&1 | tail -1 | cut -c1-170
GPCG_LIB=build_variants/libgpcg_m3async.so timeout 600 python -m pytest tests -m gpu -x -q -k "stencil3d" 2>&1 | tail -1
for v in "" build_variants/libgpcg_m3async.so; do GPCG_LIB=$v timeout 600 ncu --set full --clock-control none -k regex:"k7_cauchy" -c 2 -o gpurun_out/prof_cy python scripts/diag.py C4s > /dev/null 2>&1; python scripts/ncu_summary.py gpurun_out/prof_cy.ncu-rep | tail -2; rm -f gpurun_out/prof_cy.ncu-rep; done
