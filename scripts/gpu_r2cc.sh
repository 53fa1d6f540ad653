# r2cc: compact-space CG vectors over the free-row list (k_cg_init_c / k_cg_iter_c): tests, C4 / C4s timing, launch list
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "compact or hessvec_free or c4 or golden or spec or stencil3d" > gpurun_out/r2cc_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2cc_pytest.log | tail -20
timeout 900 python scripts/spec_ab.py C4 C4s 2>&1 | tee gpurun_out/r2cc_c4.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2cc_launches.csv python scripts/spec_ab.py C4 > gpurun_out/r2cc_ncu.log 2>&1; echo "ncu rc=$?"
gzip -f gpurun_out/r2cc_launches.csv
