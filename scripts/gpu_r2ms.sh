# r2ms: C2 one slab vs two slabs (multi-slab persistent loops) under the CG band knobs
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
for I in 1 2 4; do for C in 0 2 3; do
  echo "CG_ITEMS_PER_CTA=$I CG_CTAS_PER_SM=$C"
  if [ $C = 0 ]; then GPCG_CG_ITEMS_PER_CTA=$I timeout 600 python scripts/slab_timing.py C2 1 2; else GPCG_CG_CTAS_PER_SM=$C GPCG_CG_ITEMS_PER_CTA=$I timeout 600 python scripts/slab_timing.py C2 1 2; fi
done; done 2>&1 | tee gpurun_out/r2ms_c2.txt
