mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "solve_parity or kernel_families or golden or edge" 2>&1 | tail -1
export GPCG_TRACE_OFF=1
for i in 1 2; do timeout 300 python scripts/diag.py C2 2>&1 | tail -1; done
