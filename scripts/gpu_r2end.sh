# r2end: final validation of HEAD: smoke, full GPU suite, default bench line (C3)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2end_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/r2end_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2end_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2end_pytest.log
timeout 1200 python bench.py > gpurun_out/r2end_bench_C3.json 2> gpurun_out/r2end_bench_C3.err; echo "bench rc=$?"
