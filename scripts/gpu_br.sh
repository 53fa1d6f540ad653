export GPCG_TRACE_OFF=1
echo "BR=4"; timeout 300 python scripts/diag.py C2 C3_1600 2>&1 | tail -2 | cut -c1-150
echo "BR=8"; GPCG_LIB=build_variants/libgpcg_br8.so timeout 300 python scripts/diag.py C2 C3_1600 2>&1 | tail -2 | cut -c1-150
GPCG_LIB=build_variants/libgpcg_br8.so timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
