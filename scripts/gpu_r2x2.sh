# r2x2: hierarchical cross-rank protocol (local barrier, one leader per rank forwards the rank's
# partials and arrives on every rank's cross counter), emulated in one launch (GPCG_XRANK_EMU=1)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 1500 python -m pytest tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2x2_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2x2_pytest.log | tail -20
for E in 0 1; do echo "XRANK_EMU=$E"; GPCG_XRANK_EMU=$E timeout 900 python scripts/slab_timing.py C2 2 4 8; done 2>&1 | tee gpurun_out/r2x2_slab_timing_C2.txt
echo "XRANK_EMU=1, local fence at gpu scope (A/B)"; GPCG_LIB=build_variants/xr_fgpu.so GPCG_XRANK_EMU=1 timeout 900 python scripts/slab_timing.py C2 2 4 8 2>&1 | tee -a gpurun_out/r2x2_slab_timing_C2.txt
for E in 0 1; do echo "XRANK_EMU=$E"; GPCG_XRANK_EMU=$E timeout 1200 python scripts/slab_timing.py C3 8; done 2>&1 | tee gpurun_out/r2x2_slab_timing_C3.txt
