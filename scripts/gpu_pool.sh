mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_pool.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_pool.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
