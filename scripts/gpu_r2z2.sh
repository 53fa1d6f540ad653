# r2z2: branch-free emitted row in the speculative GP sweep (GPCG_GP_BRANCHFREE=1) vs default
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
for V in default bfree; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo "== $V"; GPCG_LIB=$L timeout 600 python scripts/diag.py C2 C3 2>&1 | grep solve
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C2 100 3
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C3 100 3
done
GPCG_LIB=build_variants/bfree.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "golden or slab" > gpurun_out/r2z2_pytest.log 2>&1; echo "pytest(bfree) rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2z2_pytest.log | tail -3
