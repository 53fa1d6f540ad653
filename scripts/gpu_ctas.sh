export GPCG_TRACE_OFF=1
for c in 4 3 2; do echo "CG CTAs/SM=$c"; GPCG_CG_CTAS_PER_SM=$c timeout 300 python scripts/diag.py C2 2>&1 | tail -1 | cut -c1-160; done
for c in 3 2; do echo "GP CTAs/SM=$c"; GPCG_GP_CTAS_PER_SM=$c timeout 300 python scripts/diag.py C2 2>&1 | tail -1 | cut -c1-160; done
