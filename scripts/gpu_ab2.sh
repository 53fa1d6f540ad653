# GPU tests + A/B: persistent CG (k6) vs graph chunks, on C2 and the C3 1600^2 member
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head -5
for P in 1 0; do echo "GPCG_GP_SPEC=$P"; GPCG_GP_SPEC=$P GPCG_TRACE=0 timeout 300 python scripts/diag.py C0 C2 C3_1600 2>&1 | grep -E "solve|Error|error"; done
