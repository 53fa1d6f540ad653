# r2z5: spec sweep fp64 trims (face sums folded, boundary faces behind a warp-uniform test, no ||g||^2)
# vs head; and the streamed previous mask (mpload)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
for V in default head mpload default; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo "== $V"; GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C2 100 3
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C3 100 3
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "not c3_full" > gpurun_out/r2z5_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2z5_pytest.log | tail -3
timeout 600 python scripts/diag.py C2 C3 2>&1 | grep solve
