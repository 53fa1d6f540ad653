# r2x3: cross-rank protocol polling variants (GPCG_XR_POLL 0 / 1 / 2 (default); local fence scope A/B)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 1500 python -m pytest tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "cross_rank or persistent" > gpurun_out/r2x3_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2x3_pytest.log | tail -20
echo "XRANK_EMU=0"; GPCG_XRANK_EMU=0 timeout 900 python scripts/slab_timing.py C2 2 8 2>&1 | tee gpurun_out/r2x3_slab_timing_C2.txt
for V in default xr_poll0 xr_poll1 xr_poll2_fgpu; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo "XRANK_EMU=1 $V"; GPCG_LIB=$L GPCG_XRANK_EMU=1 timeout 900 python scripts/slab_timing.py C2 2 8
done 2>&1 | tee -a gpurun_out/r2x3_slab_timing_C2.txt
for E in 0 1; do echo "XRANK_EMU=$E"; GPCG_XRANK_EMU=$E timeout 1200 python scripts/slab_timing.py C3 8; done 2>&1 | tee gpurun_out/r2x3_slab_timing_C3.txt
