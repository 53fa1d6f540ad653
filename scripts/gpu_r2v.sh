# r2v: C2 GP CTAs per SM; C2 1- vs 2-slab per-iteration times with CG items per CTA 1 / 2
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
for C in 1 2 3; do
  echo "gp ctas/sm=$C"; GPCG_GP_CTAS_PER_SM=$C timeout 600 python scripts/diag.py C2 2>&1 | grep solve
done
for I in 1 2; do
  echo "cg ipc=$I"; GPCG_CG_ITEMS_PER_CTA=$I timeout 600 python scripts/slab_timing.py C2 1 2 2>&1 | grep slabs
done
