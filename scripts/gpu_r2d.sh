# r2d: multi-slab persistent GP + CG loops (tests, timings) and GP sweep A/B (branch-free sums, stages / CTAs)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 1800 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "not c3_full" > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2d_pytest.log | tail -20
timeout 600 python scripts/slab_timing.py C2 1 2 4 2>&1 | tail -4
timeout 600 python scripts/slab_timing.py C3_1600 1 2 2>&1 | tail -3
for V in default bf0 old_nst4minb2; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo "== $V"; GPCG_LIB=$L timeout 600 python scripts/diag.py C3 C2 2>&1 | grep -E "solve|rror"
done
