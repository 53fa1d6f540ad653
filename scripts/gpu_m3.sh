# 3-D plane march: parity tests, C4s timing (march TY=8 / TY=16 / generic)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "stencil3d" 2>&1 | tail -3
export GPCG_TRACE_OFF=1
echo "TY=8";  timeout 300 python scripts/diag.py C4s C4s 2>&1 | tail -1
echo "TY=16"; GPCG_LIB=build_variants/libgpcg_m3ty16.so timeout 300 python scripts/diag.py C4s C4s 2>&1 | tail -1
echo "generic"; GPCG_GENERIC=1 timeout 300 python scripts/diag.py C4s C4s 2>&1 | tail -1
