# BJ-ILU(0): parity tests, preconditioner comparison (variants), ncu capture of the two PCG kernels
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "bjilu and C0" 2>&1 | tail -3 | grep -q "passed" || {
  timeout 300 python -m pytest tests -m gpu -x -q -k "bjilu and C0" 2>&1 | tail -15; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "bj or BJ or pcg or precond" 2>&1 | tail -5
timeout 300 python scripts/precond_compare.py C2 C3_1600 2>&1 | grep bj
echo "no L2 window"; GPCG_BJ_L2=0 timeout 300 python scripts/precond_compare.py C2 2>&1 | grep bj
echo "column-march matvec"; GPCG_BJ_MATVEC=1 timeout 300 python scripts/precond_compare.py C2 2>&1 | grep bj
GPCG_PRECOND=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pcg2_solve|pcg2_matvec" -s 40 -c 2 -o gpurun_out/prof_bj7 python scripts/diag.py C2 > gpurun_out/ncu_bj7.log 2>&1; tail -1 gpurun_out/ncu_bj7.log
