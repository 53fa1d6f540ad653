# tests + A/B of CG kernels on C2 (k4 default vs k3 tile vs k2 march)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for T in 15 7 3; do echo "GPCG_TILE=$T"; GPCG_TILE=$T GPCG_TRACE=0 timeout 300 python scripts/diag.py C0 C2 2>&1 | grep solve; done
