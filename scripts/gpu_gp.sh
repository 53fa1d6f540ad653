mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "solve_parity or kernel_families or golden or edge or gp_cap or determinism" 2>&1 | tail -1
export GPCG_TRACE_OFF=1
for i in 1 2; do timeout 300 python scripts/diag.py C2 C3_1600 2>&1 | tail -2 | cut -c1-160; done
