mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "spmv or c4 or dense or csr or extract or slab" 2>&1 | tail -1
export GPCG_TRACE_OFF=1
timeout 900 python scripts/metrics_all.py --oracle-budget 0 --out gpurun_out/metrics_c4.json C4 > /dev/null 2>&1; python -c "import json; r=json.load(open('gpurun_out/metrics_c4.json'))['rows'][0]; print(r['a4_hvp_us_median'], r['a4_alg_gbs'], r['solve_s'])"
timeout 300 python scripts/diag.py C4 C4 2>&1 | tail -1
