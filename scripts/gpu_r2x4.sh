# r2x4: cross-rank protocol, final form (partials stored into every mailbox by each CTA; leader-only
# system-scope fence / arrivals / poll, go flag), emulated in one launch (GPCG_XRANK_EMU=1)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 1500 python -m pytest tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2x4_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2x4_pytest.log | tail -20
for E in 0 1; do echo "XRANK_EMU=$E"; GPCG_XRANK_EMU=$E timeout 900 python scripts/slab_timing.py C2 2 4 8; done 2>&1 | tee gpurun_out/r2x4_slab_timing_C2.txt
for E in 0 1; do echo "XRANK_EMU=$E"; GPCG_XRANK_EMU=$E timeout 1200 python scripts/slab_timing.py C3 2 8; done 2>&1 | tee gpurun_out/r2x4_slab_timing_C3.txt
