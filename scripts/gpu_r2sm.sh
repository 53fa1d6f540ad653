# r2sm: smoke (C0 + the CSR path) and ncu --set full of one compact CG iteration (k_cg_iter_c) on C4
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2sm_smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/r2sm_smoke.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,lts__t_sector_hit_rate.pct
timeout 900 ncu --set full --clock-control none -k regex:k_cg_iter_c -c 1 -o /tmp/r2sm_cg -f python scripts/spec_ab.py C4 > /dev/null 2>&1; echo "ncu rc=$?"
ncu -i /tmp/r2sm_cg.ncu-rep --page raw --csv --metrics $M > gpurun_out/r2sm_ncu_cg_iter_c_C4_raw.csv 2>&1
ncu -i /tmp/r2sm_cg.ncu-rep --page details > gpurun_out/r2sm_ncu_cg_iter_c_C4_details.txt 2>&1
