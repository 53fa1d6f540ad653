export GPCG_TRACE_OFF=1
for c in 2 1; do echo "CG CTAs/SM=$c"; GPCG_CG_CTAS_PER_SM=$c timeout 300 python scripts/diag.py C2 C3_1600 2>&1 | tail -2 | cut -c1-150; done
for c in 2 1; do echo "GP CTAs/SM=$c"; GPCG_GP_CTAS_PER_SM=$c timeout 300 python scripts/diag.py C2 C3_1600 2>&1 | tail -2 | cut -c1-150; done
