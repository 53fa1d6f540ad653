# end-of-session measurement: full GPU suite, smoke, bench line, preconditioner + paper-setting JSON
TAG=${TAG:-r1h}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-200
timeout 900 python scripts/precond_compare.py --out gpurun_out/precond_compare.json > gpurun_out/precond.log 2>&1; echo "precond rc=$?"
timeout 900 python scripts/paper_setting.py --out gpurun_out/paper_setting.json > gpurun_out/paper_setting.log 2>&1; echo "paper rc=$?"
