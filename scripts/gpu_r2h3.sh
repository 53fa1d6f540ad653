# r2h3: compact-output reduced HVP with the chosen row groups (4 lanes x 2 rows, 64 registers):
# parity tests, a4 microbenchmark (events no longer include the host's launch latency), ncu
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "hessvec_free or compact or spmv" > gpurun_out/r2h3_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2h3_pytest.log | tail -20
timeout 900 python scripts/a4_compact.py C4 C4s 2>&1 | tail -4
cp gpurun_out/a4_compact.json gpurun_out/r2h3_a4_compact.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,launch__grid_size,launch__occupancy_limit_registers
for C in C4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hessvec_free --launch-skip 35 -c 1 \
    -o /tmp/r2h3_ncu_hvf_$C -f python scripts/a4_compact.py $C > gpurun_out/r2h3_ncu_$C.log 2>&1; echo "ncu $C rc=$?"
  ncu -i /tmp/r2h3_ncu_hvf_$C.ncu-rep --page raw --csv --metrics $M > gpurun_out/r2h3_ncu_hvf_${C}_raw.csv 2>&1
  ncu -i /tmp/r2h3_ncu_hvf_$C.ncu-rep --page details > gpurun_out/r2h3_ncu_hvf_${C}_details.txt 2>&1
done
