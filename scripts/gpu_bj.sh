set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "bj or BJ or pcg or precond" 2>&1 | tail -3
timeout 300 python scripts/precond_compare.py C2 C3_1600 2>&1 | grep bj
GPCG_PRECOND=2 timeout 600 ncu --set full --clock-control none -k regex:"pcg2_solve" -s 40 -c 1 -o gpurun_out/prof_bj8 python scripts/diag.py C2 > /dev/null 2>&1; python scripts/ncu_summary.py gpurun_out/prof_bj8.ncu-rep
