mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "solve_parity or kernel_families or golden or edge or gp_cap or path_switches or slab" 2>&1 | tail -1
export GPCG_TRACE_OFF=1
timeout 300 python scripts/diag.py C2 C3_1600 2>&1 | tail -2 | cut -c1-160
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cg_block_flags" -c 5 --csv python scripts/diag.py C2 2>/dev/null | grep -o '"[0-9,.]*"$' | head -5
