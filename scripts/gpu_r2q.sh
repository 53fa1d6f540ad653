# r2q: speculative GP sweep without the mask_prev stream (previous mask from y, l, u)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "not c3_full" > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2q_pytest.log | tail -5
for V in default head default head; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C3 100000 2 2>&1 | tail -1
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C2 100000 3 2>&1 | tail -1
done
