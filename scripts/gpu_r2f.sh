# r2f: compact free-row list (tests, a4 microbenchmark), GP-loop A/B (warps / CTAs per SM)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "compact or spmv or c4 or golden" > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2f_pytest.log | tail -20
timeout 600 python scripts/a4_compact.py C4 C4s 2>&1 | tail -6
for V in default w8m2 w4m4 w4m6 old_nst4minb2; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C3 300 2>&1 | tail -1
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C2 300 2>&1 | tail -1
done
