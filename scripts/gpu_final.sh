# round measurement: full GPU suite, bench line, launch list, ncu --set full of the persistent loops
# (C2) and of the CSR / 3-D generic sweeps (C4, C4s), preconditioner comparison, paper-setting runs.
# ncu reports are summarised on the box (scripts/ncu_summary.py) and only the C2 one is kept.
TAG=${TAG:-r1g}
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
fi
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-300
timeout 900 python scripts/precond_compare.py --out gpurun_out/precond_compare.json > gpurun_out/precond.log 2>&1; echo "precond rc=$?"
timeout 900 python scripts/paper_setting.py --out gpurun_out/paper_setting.json > gpurun_out/paper_setting.log 2>&1; echo "paper rc=$?"
export GPCG_TRACE_OFF=1
timeout 300 python scripts/diag.py C2 C4 C4s > gpurun_out/plain.log 2>&1; echo "diag rc=$?"; cat gpurun_out/plain.log | cut -c1-250
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python scripts/diag.py C2 > gpurun_out/ncu_ll.log 2>&1; echo "ll rc=$?"
python scripts/ncu_summary.py gpurun_out/launches_${TAG}.csv > gpurun_out/launches_${TAG}_summary.txt 2>&1
gzip -f gpurun_out/launches_${TAG}.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_" -s 60 -c 2 -o gpurun_out/prof_${TAG} \
    python scripts/diag.py C2 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep > gpurun_out/ncu_full_${TAG}_C2.txt 2>&1
for c in C4 C4s; do
timeout 900 ncu --set full --clock-control none -k regex:"k_(accept|search|cg_iter|cauchy|cg_init)" -c 6 -o gpurun_out/prof_${TAG}_$c \
    python scripts/diag.py $c > gpurun_out/ncu_$c.log 2>&1; echo "$c rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_${TAG}_$c.ncu-rep > gpurun_out/ncu_full_${TAG}_$c.txt 2>&1
rm -f gpurun_out/prof_${TAG}_$c.ncu-rep
done
du -sh gpurun_out
