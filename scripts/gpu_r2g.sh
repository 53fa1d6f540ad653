# r2g: two-column speculative GP sweep (spec_sweep7): parity + A/B against spec_sweep6
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 120 python scripts/diag.py C0 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "not c3_full" > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2g_pytest.log | tail -20
for V in default spec6 spec7nst3; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C3 100000 2 2>&1 | tail -1
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C2 100000 3 2>&1 | tail -1
done
timeout 300 python scripts/slab_timing.py C2 1 2 2>&1 | tail -2
timeout 600 python scripts/diag.py C3 2>&1 | tail -1
