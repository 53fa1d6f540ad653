# GPU tests + diag of every config family + A/B of the GP sweeps (k5 g-free vs k4 stored g)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head -5
GPCG_TRACE=0 timeout 600 python scripts/diag.py C0 C1 C2 C3_1600 C4_128 C4 C4s 2>&1 | grep -E "solve|Error|error"
for T in 63 127; do echo "GPCG_TILE=$T"; GPCG_TILE=$T GPCG_TRACE=0 timeout 300 python scripts/diag.py C2 2>&1 | grep -E "solve|Error"; done
