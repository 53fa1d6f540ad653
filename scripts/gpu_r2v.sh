mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2v_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2v_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2v_pytest.log
timeout 900 python bench.py > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2v_bench.json
