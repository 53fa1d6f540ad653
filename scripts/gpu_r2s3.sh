# r2s3: k_spec with g' = A y' - b (bit for bit the search + accept sweeps) for the GP steps and the
# CG phase's step of the generic operators: full GPU suite, C4 / C4s A/B, ncu of k_spec
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s3_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2s3_pytest.log | tail -20
for S in 0 1; do GPCG_GP_SPEC=$S timeout 900 python scripts/spec_ab.py C4 C4s; done 2>&1 | tee gpurun_out/r2s3_spec_ab.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,lts__t_sector_hit_rate.pct
timeout 900 ncu --set full --clock-control none -k regex:k_spec -c 2 -o /tmp/r2s3_spec -f python scripts/spec_ab.py C4 > /dev/null 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/r2s3_spec.ncu-rep --page raw --csv --metrics $M > gpurun_out/r2s3_ncu_spec_C4_raw.csv 2>&1
ncu -i /tmp/r2s3_spec.ncu-rep --page details > gpurun_out/r2s3_ncu_spec_C4_details.txt 2>&1
