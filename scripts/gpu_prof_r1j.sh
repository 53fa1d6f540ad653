mkdir -p gpurun_out
TAG=r1j
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 900 --csv \
  --log-file gpurun_out/launches_bench_${TAG}.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
echo "ll rc=$?"
python scripts/ncu_summary.py gpurun_out/launches_bench_${TAG}.csv > gpurun_out/launches_bench_${TAG}_summary.txt; cat gpurun_out/launches_bench_${TAG}_summary.txt
gzip -f gpurun_out/launches_bench_${TAG}.csv
export GPCG_TRACE_OFF=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_" -s 60 -c 2 -o gpurun_out/prof_${TAG} python scripts/diag.py C2 > /dev/null 2>&1; echo "full rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep > gpurun_out/ncu_full_${TAG}_C2.txt; cat gpurun_out/ncu_full_${TAG}_C2.txt
rm -f gpurun_out/prof_${TAG}.ncu-rep
