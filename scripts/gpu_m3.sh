export GPCG_TRACE_OFF=1
for v in "" build_variants/libgpcg_m3mb3.so build_variants/libgpcg_m3mb4.so; do echo "lib=$v"; GPCG_LIB=$v timeout 300 python scripts/diag.py C4s C4s 2>&1 | tail -1 | cut -c1-150; done
GPCG_LIB=build_variants/libgpcg_m3mb4.so timeout 600 python -m pytest tests -m gpu -x -q -k "stencil3d" 2>&1 | tail -1
