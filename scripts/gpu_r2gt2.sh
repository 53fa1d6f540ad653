# r2i: per-CTA GP sweep times vs SM occupancy / band (diagnostic build)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
GPCG_LIB=build_variants/diagt.so timeout 300 python scripts/gp_step_times.py C3 3
