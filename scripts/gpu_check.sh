set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
GPCG_TRACE=0 timeout 300 python scripts/diag.py c0 c1 c2 > gpurun_out/diag_tile.log 2>&1
GPCG_TILE=0 GPCG_TRACE= timeout 300 python scripts/diag.py c0 c1 c2 > gpurun_out/diag_march.log 2>&1
grep -h solve gpurun_out/diag_*.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench.log
