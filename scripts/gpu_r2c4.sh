# r2c4: where a C4 solve's time goes: traced solve, ncu launch list of 4 solves (spec_ab.py), ncu --set full of k_spec
mkdir -p gpurun_out
GPCG_TRACE=1 timeout 600 python scripts/diag.py C4 > gpurun_out/r2c4_trace.txt 2>&1; echo "diag rc=$?"
tail -3 gpurun_out/r2c4_trace.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2c4_launches.csv python scripts/spec_ab.py C4 > gpurun_out/r2c4_ncu.log 2>&1; echo "ncu rc=$?"
gzip -f gpurun_out/r2c4_launches.csv
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,lts__t_sector_hit_rate.pct
timeout 900 ncu --set full --clock-control none -k regex:k_spec -c 2 -o /tmp/r2c4_spec -f python scripts/spec_ab.py C4 > /dev/null 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/r2c4_spec.ncu-rep --page raw --csv --metrics $M > gpurun_out/r2c4_ncu_spec_raw.csv 2>&1
ncu -i /tmp/r2c4_spec.ncu-rep --page details > gpurun_out/r2c4_ncu_spec_details.txt 2>&1
