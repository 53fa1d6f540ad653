# launch list of a few BJ-ILU PCG iterations on C2 (per-kernel durations)
mkdir -p gpurun_out
GPCG_PRECOND=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 80 --csv --log-file gpurun_out/bj_ll.csv python scripts/diag.py C2 > gpurun_out/bj_ll.log 2>&1
tail -2 gpurun_out/bj_ll.log
GPCG_PRECOND=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pcg2_matvec" -s 40 -c 1 -o gpurun_out/prof_bj5 python scripts/diag.py C2 > gpurun_out/ncu_bj5.log 2>&1; tail -2 gpurun_out/ncu_bj5.log
