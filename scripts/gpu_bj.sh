# BJ-ILU(0): parity tests, preconditioner comparison, and an ncu capture of the solve kernel
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "bjilu and C0" 2>&1 | tail -3 | grep -q "passed" || {
  GPCG_PRECOND=2 timeout 300 compute-sanitizer --print-limit 5 python scripts/diag.py C0 2>&1 | head -40; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "bj or BJ or pcg or precond" 2>&1 | tail -5
timeout 300 python scripts/precond_compare.py C2 C3_1600 2>&1 | tail -8
for u in 16; do echo "unroll $u"; GPCG_LIB=build_variants/libgpcg_bj$u.so timeout 300 python scripts/precond_compare.py C2 2>&1 | grep bj; done
GPCG_PRECOND=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pcg2_solve|k_pcg2_matvec" -s 40 -c 2 -o gpurun_out/prof_bj4 python scripts/diag.py C2 > gpurun_out/ncu_bj4.log 2>&1; tail -3 gpurun_out/ncu_bj4.log
