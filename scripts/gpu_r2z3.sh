# r2z3: upper bound of a cheaper bounds stream -- GP steps on C3 with the scalar-bounds sweeps
# (diagnostic build: wrong bounds, per-step time only)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 300 python scripts/gp_ab.py C3 100 3
GPCG_LIB=build_variants/forcesb.so timeout 300 python scripts/gp_ab.py C3 100 3
GPCG_LIB=build_variants/forcesb.so timeout 300 python scripts/gp_ab.py C3 100 1
