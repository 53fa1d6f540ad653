# round-2 evidence set (C3, the bench workload): the bench command's own ncu launch list (cold,
# serialised per-launch times -> device-time shares), one ncu --set full capture each of the
# persistent CG and GP loops (CSV exports only), and the solve-wide DRAM traffic per unit
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
TAG=${TAG:-r2z}
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu bench rc=$?"
python scripts/ncu_summary.py /tmp/launches_bench.csv > gpurun_out/${TAG}_launches_bench_C3_summary.txt 2>&1; cat gpurun_out/${TAG}_launches_bench_C3_summary.txt | head -20
gzip -c /tmp/launches_bench.csv > gpurun_out/${TAG}_launches_bench_C3.csv.gz
for K in k6_cg_loop k6_gp_loop; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 4 -c 1 -o /tmp/prof_$K python scripts/diag.py C3 > gpurun_out/${TAG}_ncu_$K.log 2>&1; echo "ncu $K rc=$?"
  python scripts/ncu_summary.py /tmp/prof_$K.ncu-rep > gpurun_out/${TAG}_ncu_full_${K}_C3.txt 2>&1; cat gpurun_out/${TAG}_ncu_full_${K}_C3.txt
  ncu -i /tmp/prof_$K.ncu-rep --page details > gpurun_out/${TAG}_ncu_full_${K}_C3_details.txt 2>&1
  ncu -i /tmp/prof_$K.ncu-rep --page raw --csv 2>/dev/null | gzip -c > gpurun_out/${TAG}_ncu_full_${K}_C3_raw.csv.gz
done
timeout 600 python scripts/diag.py C3 > gpurun_out/${TAG}_diag_c3.log 2>&1; cat gpurun_out/${TAG}_diag_c3.log
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k6_" --csv --log-file /tmp/ll_c3.csv python scripts/diag.py C3 > gpurun_out/${TAG}_ncu_ll.log 2>&1; echo "ncu ll rc=$?"
python scripts/traffic_summary.py /tmp/ll_c3.csv gpurun_out/${TAG}_diag_c3.log C3 ${TAG} > gpurun_out/traffic_C3_${TAG}.json; cat gpurun_out/traffic_C3_${TAG}.json
