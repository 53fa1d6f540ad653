# r2x5: cross-rank protocol emulated in one launch: gpu scope (the emulation's ranks share a device)
# vs system scope (GPCG_XRANK_SYS=1, what ranks on several devices run)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 1500 python -m pytest tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "cross_rank or persistent" > gpurun_out/r2x5_pytest.log 2>&1; echo "pytest rc=$?"
GPCG_XRANK_SYS=1 timeout 1500 python -m pytest tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider -k "cross_rank" >> gpurun_out/r2x5_pytest.log 2>&1; echo "pytest (sys scope) rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2x5_pytest.log | tail -20
for E in 0 1; do echo "XRANK_EMU=$E"; GPCG_XRANK_EMU=$E timeout 900 python scripts/slab_timing.py C2 2 4 8; done 2>&1 | tee gpurun_out/r2x5_slab_timing_C2.txt
echo "XRANK_EMU=1 XRANK_SYS=1"; GPCG_XRANK_SYS=1 GPCG_XRANK_EMU=1 timeout 900 python scripts/slab_timing.py C2 2 8 2>&1 | tee -a gpurun_out/r2x5_slab_timing_C2.txt
for E in 1; do echo "XRANK_EMU=$E"; GPCG_XRANK_EMU=$E timeout 1200 python scripts/slab_timing.py C3 2 8; done 2>&1 | tee gpurun_out/r2x5_slab_timing_C3.txt
