# r2fin: end-of-session validation of HEAD: smoke, full GPU suite, C3 bench line, C2 bench line
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2fin_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2fin_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2fin_pytest.log
timeout 1200 python bench.py > gpurun_out/r2fin_bench_C3.json 2> gpurun_out/r2fin_bench_C3.err; echo "bench C3 rc=$?"
timeout 900 python bench.py --config C2 --steps 10 > gpurun_out/r2fin_bench_C2.json 2> gpurun_out/r2fin_bench_C2.err; echo "bench C2 rc=$?"
timeout 900 python bench.py --config C4 --steps 10 > gpurun_out/r2fin_bench_C4.json 2> gpurun_out/r2fin_bench_C4.err; echo "bench C4 rc=$?"
