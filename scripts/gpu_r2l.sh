# r2l: full GPU suite, C3 bench, preconditioners (incl. BJ-ILU(2)), paper-setting runs, solve-wide
# DRAM traffic on C3, compact free-row a4 microbenchmark, multi-slab timings
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2l_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|\[C3\]|\[parity\]" gpurun_out/r2l_pytest.log | tail -12
timeout 1500 python bench.py --steps 3 --warmup 1 > gpurun_out/r2l_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2l_bench.log
timeout 900 python scripts/precond_compare.py --out gpurun_out/precond_compare_r2.json C1 C2 C3_1600 2>&1 | tail -12
timeout 900 python scripts/paper_setting.py --out gpurun_out/paper_setting_r2.json 2>&1 | tail -16
timeout 600 python scripts/a4_compact.py C4 C4s 2>&1 | tail -4
timeout 300 python scripts/slab_timing.py C2 1 2 4 2>&1 | tail -3
timeout 600 python scripts/diag.py C3 > gpurun_out/r2l_diag_c3.log 2>&1; cat gpurun_out/r2l_diag_c3.log
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k6_" --csv --log-file /tmp/r2l_launches_c3.csv python scripts/diag.py C3 > gpurun_out/r2l_ncu_ll.log 2>&1; echo "ncu ll rc=$?"
python scripts/traffic_summary.py /tmp/r2l_launches_c3.csv gpurun_out/r2l_diag_c3.log C3 r2l > gpurun_out/traffic_C3_r2l.json; cat gpurun_out/traffic_C3_r2l.json
