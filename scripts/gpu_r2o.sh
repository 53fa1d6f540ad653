# r2o: GP block rows / stages A/B (GPCG_GP_BR, GPCG_GP_NST, GPCG_GP_MINB)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "solve_parity and (C0 or C1 or c3_family)" > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2o_pytest.log
for V in default br8 br6 br4n2 default; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C3 100000 2 2>&1 | tail -1
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C2 100000 3 2>&1 | tail -1
done
