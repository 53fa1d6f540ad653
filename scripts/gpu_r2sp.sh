# r2sp: k_spec / k_cauchy register budget (CTAs per SM) A/B on C4
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
for V in default spec_m4 spec_m6 spec_m8; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo $V; GPCG_LIB=$L timeout 600 python scripts/spec_ab.py C4 C4
done 2>&1 | tee gpurun_out/r2sp.txt
