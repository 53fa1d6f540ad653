# r2t: CG items per CTA sweep beyond 8
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
for I in 8 12 16 24 32; do
  echo "ipc=$I"; GPCG_CG_ITEMS_PER_CTA=$I timeout 600 python scripts/diag.py C3 2>&1 | grep solve
done
