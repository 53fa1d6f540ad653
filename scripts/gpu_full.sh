# full GPU suite + preconditioner comparison + paper-setting runs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
timeout 900 python scripts/precond_compare.py --out gpurun_out/precond_compare.json > gpurun_out/precond.log 2>&1; echo "precond rc=$?"; cut -c1-250 gpurun_out/precond.log
timeout 900 python scripts/paper_setting.py --out gpurun_out/paper_setting.json > gpurun_out/paper_setting.log 2>&1; echo "paper rc=$?"; cut -c1-200 gpurun_out/paper_setting.log
