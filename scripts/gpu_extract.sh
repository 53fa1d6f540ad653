mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
timeout 900 python scripts/extraction_ablation.py --out gpurun_out/extraction_ablation.json > gpurun_out/ablation.log 2>&1; echo "ablation rc=$?"; cut -c1-260 gpurun_out/ablation.log
