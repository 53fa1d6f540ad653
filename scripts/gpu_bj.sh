mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "bjilu" 2>&1 | tail -1
timeout 300 python scripts/precond_compare.py C2 2>&1 | grep bj
