# ncu launch list of the bench command itself: one full timed C2 solve (skip create + 3 warm-up
# solves + the first timed one; ~860 launches per solve), per-launch durations
mkdir -p gpurun_out
TAG=${TAG:-r1h}
timeout 600 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_plain.log 2>&1; echo "plain rc=$?"
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -s 3500 -c 900 --csv \
  --log-file gpurun_out/launches_bench_${TAG}.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_bench.log
python scripts/ncu_summary.py gpurun_out/launches_bench_${TAG}.csv > gpurun_out/launches_bench_${TAG}_summary.txt; cat gpurun_out/launches_bench_${TAG}_summary.txt
gzip -f gpurun_out/launches_bench_${TAG}.csv
timeout 300 python scripts/precond_compare.py C2 2>&1 | grep bj
