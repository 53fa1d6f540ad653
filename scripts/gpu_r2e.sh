# r2e: recalibrated C3 (c = 0.01045): full GPU suite, bench on C3, solve-wide DRAM traffic of the
# persistent loops, ncu --set full of one CG call and one GP phase
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|\[C3\]" gpurun_out/r2e_pytest.log | tail -10
timeout 1500 python bench.py --steps 3 --warmup 1 > gpurun_out/r2e_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2e_bench.log
timeout 300 python scripts/slab_timing.py C2 1 2 4 2>&1 | tail -3
timeout 600 python scripts/diag.py C3 > gpurun_out/r2e_diag_c3.log 2>&1; cat gpurun_out/r2e_diag_c3.log
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k6_" --csv --log-file gpurun_out/r2e_launches_c3.csv python scripts/diag.py C3 > gpurun_out/r2e_ncu_ll.log 2>&1; echo "ncu ll rc=$?"
python scripts/traffic_summary.py gpurun_out/r2e_launches_c3.csv gpurun_out/r2e_diag_c3.log C3 r2e > gpurun_out/traffic_C3.json; cat gpurun_out/traffic_C3.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_cg_loop" -s 5 -c 1 -o gpurun_out/r2e_cg_c3 python scripts/diag.py C3 > gpurun_out/r2e_ncu_cg.log 2>&1; echo "ncu cg rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_gp_loop" -s 5 -c 1 -o gpurun_out/r2e_gp_c3 python scripts/diag.py C3 > gpurun_out/r2e_ncu_gp.log 2>&1; echo "ncu gp rc=$?"
for r in r2e_cg_c3 r2e_gp_c3; do python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1; cat gpurun_out/${r}_summary.txt; done
