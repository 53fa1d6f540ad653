mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "csr or c4 or dense or spmv or slab or golden or extract" 2>&1 | tail -3
export GPCG_TRACE_OFF=1
echo "vector"; timeout 300 python scripts/diag.py C4 C4 2>&1 | tail -1
echo "scalar"; GPCG_CSR_SCALAR=1 timeout 300 python scripts/diag.py C4 C4 2>&1 | tail -1
timeout 900 python scripts/metrics_all.py --oracle-budget 0 --out gpurun_out/metrics_c4.json C4 > /dev/null 2>&1; python -c "import json; r=json.load(open('gpurun_out/metrics_c4.json'))['rows'][0]; print('a4', r['a4_hvp_us_median'], r['a4_alg_gbs'], 'solve', r['solve_s'])"
timeout 900 ncu --set full --clock-control none -k regex:"k_(accept|search|cauchy)" -c 3 -o gpurun_out/prof_csrv python scripts/diag.py C4 > /dev/null 2>&1; python scripts/ncu_summary.py gpurun_out/prof_csrv.ncu-rep
