# r2h: spec_sweep7 fault bisection: dbg1 = pipeline only (no row work), dbg2 = box A only
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
for V in dbg3 dbg4; do
  echo "== $V"
  GPCG_LIB=build_variants/$V.so timeout 120 python scripts/diag.py C0 2>&1 | tail -1
done
