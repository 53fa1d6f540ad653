# CTAs-per-SM sweep of the persistent CG / GP kernels on C2 (diag timing)
export GPCG_TRACE=0
for c in 4 3 2; do echo "CG_CTAS_PER_SM=$c"; GPCG_CG_CTAS_PER_SM=$c timeout 300 python scripts/diag.py C2 2>&1 | grep -E "solve|Error"; done
for c in 3 2; do echo "GP_CTAS_PER_SM=$c"; GPCG_GP_CTAS_PER_SM=$c timeout 300 python scripts/diag.py C2 2>&1 | grep -E "solve|Error"; done
