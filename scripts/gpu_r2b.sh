# r2b: full GPU test suite (new goldens, C3 full-size certificate, ILU(2) parity) + GP-sweep A/B on C3 / C2
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|\[C3\]|\[parity\]" gpurun_out/r2b_pytest.log | tail -40
for V in default spec5 nst3 nst3minb3; do
  if [ $V = default ]; then L=""; else L=build_variants/$V.so; fi
  echo "== $V"; GPCG_LIB=$L timeout 600 python scripts/diag.py C3 C2 C2 2>&1 | grep -E "solve|rror"
done
