# C3 family: outer / GP / CG counts vs grid size (is the 8000^2 convergence algorithmic?)
export GPCG_TRACE_OFF=1
for c in C3_800 C3_1600 C3_2400 C3_3200 C3_4800; do timeout 600 python scripts/diag.py $c 2>&1 | tail -1 | cut -c1-200; done
