# r2r: CG sweep compute skip for all-active warp blocks; BJ-ILU(2) solves three tiles per warp
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "not c3_full" > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2r_pytest.log | tail -5
for V in default head; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  GPCG_LIB=$L timeout 600 python scripts/diag.py C3 C2 2>&1 | grep solve
  GPCG_LIB=$L GPCG_PRECOND=3 timeout 600 python scripts/diag.py C2 C3_1600 2>&1 | grep solve
done
