# r2h2: compact-output reduced HVP: parity tests, random-gather ceiling microbenchmark, row-group
# variants A/B, ncu --set full of one launch each (text summaries only: the reports exceed the
# 64 MiB return limit)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "hessvec_free or compact or spmv" > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2h_pytest.log | tail -20
./scripts/micro/gather.bin 6546.2 | tee gpurun_out/r2h_gather.txt
for V in default hvf_minb4 hvf_l4u2m4 hvf_l4u4m4 hvf_l8u2m6 hvf_l8u4m5; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo $V; GPCG_LIB=$L timeout 600 python scripts/a4_compact.py C4 2>&1 | grep '"cg_mode": 2' | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['hvp_us'], r['hvp_free_us'], r['frac_alg_free'])"
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,launch__grid_size,launch__occupancy_limit_registers
for C in C4 C4s; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hessvec_free --launch-skip 35 -c 1 \
    -o /tmp/r2h_ncu_hvf_$C -f python scripts/a4_compact.py $C > gpurun_out/r2h_ncu_$C.log 2>&1; echo "ncu $C rc=$?"
  ncu -i /tmp/r2h_ncu_hvf_$C.ncu-rep --page raw --csv --metrics $M > gpurun_out/r2h_ncu_hvf_${C}_raw.csv 2>&1
  ncu -i /tmp/r2h_ncu_hvf_$C.ncu-rep --page details > gpurun_out/r2h_ncu_hvf_${C}_details.txt 2>&1
  ncu -i /tmp/r2h_ncu_hvf_$C.ncu-rep --page source --csv > gpurun_out/r2h_ncu_hvf_${C}_source.csv 2>&1
  gzip -f gpurun_out/r2h_ncu_hvf_${C}_source.csv
done
ls -la gpurun_out
