# r2ct: C3 GP step vs CTAs per SM of the GP bands (power-capped step; GPCG_GP_CTAS_PER_SM), and C2
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
for C in 0 2 1; do for R in 1 2; do
  if [ $C = 0 ]; then timeout 600 python scripts/gp_ab.py C3 1000; else GPCG_GP_CTAS_PER_SM=$C timeout 600 python scripts/gp_ab.py C3 1000; fi | sed "s/^/ctas=$C rep=$R /"
done; done 2>&1 | tee gpurun_out/r2ct.txt
for C in 0 2; do if [ $C = 0 ]; then timeout 600 python scripts/gp_ab.py C2 1000; else GPCG_GP_CTAS_PER_SM=$C timeout 600 python scripts/gp_ab.py C2 1000; fi | sed "s/^/ctas=$C /"; done 2>&1 | tee -a gpurun_out/r2ct.txt
