# GPU tests + a quick C2 diag + bench (one gpurun call)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
GPCG_TRACE=0 timeout 300 python scripts/diag.py C0 C1 C2 > gpurun_out/diag.log 2>&1; grep solve gpurun_out/diag.log
if [ -n "$BENCH" ]; then timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-600; fi
