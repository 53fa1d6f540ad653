# r2a: C3 under the paper's uncapped GP phase: solve timing, full-size certificate test, goldens,
# short bench on C3, ncu DRAM traffic of one CG call / one GP phase on C3
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; grep -m1 "model name" /proc/cpuinfo
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 600 python scripts/diag.py C3 C2 > gpurun_out/r2a_diag.log 2>&1; cat gpurun_out/r2a_diag.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -k "c3_full or golden" -p no:cacheprovider > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/r2a_tests.log
timeout 900 python bench.py --steps 2 --warmup 1 > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/r2a_bench.log
timeout 600 python scripts/cg_traffic.py 16 C3 > gpurun_out/r2a_cgtraffic_plain.log 2>&1; cat gpurun_out/r2a_cgtraffic_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_cg_loop" -c 1 -o gpurun_out/r2a_cg_c3 python scripts/cg_traffic.py 16 C3 > gpurun_out/r2a_ncu_cg.log 2>&1; echo "ncu cg rc=$?"
timeout 600 python scripts/gp_traffic.py 16 C3 > gpurun_out/r2a_gptraffic_plain.log 2>&1; cat gpurun_out/r2a_gptraffic_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_gp_loop" -c 1 -o gpurun_out/r2a_gp_c3 python scripts/gp_traffic.py 16 C3 > gpurun_out/r2a_ncu_gp.log 2>&1; echo "ncu gp rc=$?"
for r in r2a_cg_c3 r2a_gp_c3; do python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.txt 2>&1; ncu -i gpurun_out/$r.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/${r}_dram.csv 2>&1; cat gpurun_out/${r}_dram.csv; done
