# r2cc2: compact-space CG + adaptive chunks (CG: 4, 8, 16, ...; GP graph: a 2-step graph for each phase's first launch)
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2cc2_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2cc2_pytest.log | tail -20
timeout 900 python scripts/spec_ab.py C4 C4s 2>&1 | tee gpurun_out/r2cc2_c4.txt
timeout 900 python scripts/a4_compact.py C4 C4s 2>&1 | tail -4
cp gpurun_out/a4_compact.json gpurun_out/r2cc2_a4_compact.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2cc2_launches.csv python scripts/spec_ab.py C4 > gpurun_out/r2cc2_ncu.log 2>&1; echo "ncu rc=$?"
gzip -f gpurun_out/r2cc2_launches.csv
