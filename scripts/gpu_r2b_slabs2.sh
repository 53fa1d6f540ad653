# r2b_slabs2: GP items per CTA chosen per slab geometry (C3 two slabs: 2 items of 364 rows per CTA)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_slabs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2b_slabs2_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2b_slabs2_pytest.log | tail -3
timeout 1200 python scripts/slab_timing.py C3 1 2 2>&1 | grep slabs
timeout 900 python scripts/slab_timing.py C2 1 2 2>&1 | grep slabs
