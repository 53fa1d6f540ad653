timeout 300 python -m pytest tests -m gpu -x -q -k "bjilu and C0" 2>&1 | tail -30
