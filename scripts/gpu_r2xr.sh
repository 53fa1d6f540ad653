# r2xr: host side of the cross-rank loops (GPCG_XRANK; neighbour tables shared with the slabs of one
# device), entry barrier under system scope in the emulation: full GPU suite, C2 / C3 slab timing
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2xr_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2xr_pytest.log | tail -20
for E in 0 1; do echo "XRANK_EMU=$E"; GPCG_XRANK_EMU=$E timeout 900 python scripts/slab_timing.py C2 2 8; done 2>&1 | tee gpurun_out/r2xr_slab_timing_C2.txt
echo "XRANK_EMU=1 XRANK_SYS=1"; GPCG_XRANK_SYS=1 GPCG_XRANK_EMU=1 timeout 900 python scripts/slab_timing.py C2 2 8 2>&1 | tee -a gpurun_out/r2xr_slab_timing_C2.txt
