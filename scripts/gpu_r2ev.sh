# r2ev (run as r2f, outputs tagged r2f): round-2 evidence refresh -- full GPU test suite, the default bench line (C3), the C2 bench
# line, then the profiling set of gpu_prof_r2.sh (launch list, ncu --set full of both loops, traffic)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2f_pytest.log | tail -3
timeout 1800 python bench.py > gpurun_out/r2f_bench_C3.json 2> gpurun_out/r2f_bench_C3.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r2f_bench_C3.json
timeout 900 python bench.py --config C2 > gpurun_out/r2f_bench_C2.json 2> gpurun_out/r2f_bench_C2.err; echo "bench C2 rc=$?"
TAG=r2f bash scripts/gpu_prof_r2.sh
