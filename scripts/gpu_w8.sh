export GPCG_TRACE_OFF=1
for v in "" build_variants/libgpcg_w8.so; do echo "lib=$v"; GPCG_LIB=$v timeout 900 python scripts/metrics_all.py --oracle-budget 0 C2 C3 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l); print(r['config'], 'solve', round(r['solve_s'],4), 'hvps', round(r['hvp_per_s']), 'cg_us', round(r['cg_us_per_iter'] or 0,1), 'a4_us', round(r['a4_hvp_us_median'],1), 'outer', r['outer'], 'gp', r['gp_iters'], 'cg', r['cg_iters'])"; done
