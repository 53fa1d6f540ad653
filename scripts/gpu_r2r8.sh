# r2r8: CsrOp rows of <= 8 entries loaded whole before the callbacks (GPCG_CSR_ROW8) A/B on C4
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
for V in default row8 default row8; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo $V; GPCG_LIB=$L timeout 600 python scripts/spec_ab.py C4
done 2>&1 | tee gpurun_out/r2r8.txt
GPCG_LIB=build_variants/row8.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "c4 or dense or spec or compact or golden" 2>&1 | tail -2
