# r2w: spec_sweep6 with fewer instructions per row (row pointers, shared bound / sign tests, hoisted
# boundary face); C2 one slab through the multi-slab kernels (GPCG_MS_ONE)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "not c3_full" > gpurun_out/r2w_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2w_pytest.log | tail -5
for V in default head; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo "== $V"; GPCG_LIB=$L timeout 600 python scripts/diag.py C3 C2 2>&1 | grep solve
done
echo "== MS_ONE"; GPCG_MS_ONE=1 timeout 600 python scripts/slab_timing.py C2 1 2 2>&1 | grep slabs
