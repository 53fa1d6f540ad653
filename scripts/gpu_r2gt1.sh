# r2h: where a persistent GP step's time goes (globaltimer stamps per CTA, diagnostic build)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
GPCG_LIB=build_variants/diagt.so timeout 300 python scripts/gp_step_times.py C3 3
GPCG_LIB=build_variants/diagt.so timeout 300 python scripts/gp_step_times.py C2 3
GPCG_LIB=build_variants/diagt.so timeout 300 python scripts/gp_step_times.py C2 20
