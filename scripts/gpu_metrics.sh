mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "stencil3d" 2>&1 | tail -1
timeout 900 python scripts/metrics_all.py --out gpurun_out/metrics_c4s.json C4s > gpurun_out/metrics.log 2>&1; echo "metrics rc=$?"
