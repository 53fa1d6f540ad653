# r2y: grid barrier variants (0 = poll the counter, 1 = generation flag, 2 = flag + nanosleep)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
for V in default gbar1 gbar2; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo "== $V"; GPCG_LIB=$L timeout 600 python scripts/diag.py C2 C3 2>&1 | grep solve
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C2 100 3
done
GPCG_LIB=build_variants/gbar1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "golden or slab" > gpurun_out/r2y_pytest.log 2>&1; echo "pytest(gbar1) rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2y_pytest.log | tail -3
