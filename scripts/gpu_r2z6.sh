# r2z6: GP sweep occupancy / block shape: 4 CTAs per SM with 4-row blocks (64 registers) and 3 stages of 4 rows
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
for V in default m4b4 m3b4n3 default; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo "== $V"; GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C2 100 3
  GPCG_LIB=$L timeout 300 python scripts/gp_ab.py C3 100 3
done
