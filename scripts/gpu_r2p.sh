# r2p: full GPU suite on the tuned GP sweeps (6-row blocks, 2 stages), C2 bench line, slab timings
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|\[C3\]" gpurun_out/r2p_pytest.log | tail -8
timeout 900 python bench.py --config C2 --steps 10 --warmup 3 > gpurun_out/r2p_bench_C2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2p_bench_C2.log | cut -c1-600
timeout 300 python scripts/slab_timing.py C2 1 2 4 2>&1 | tail -3
timeout 300 python scripts/gp_ab.py C3 100000 2 2>&1 | tail -1
