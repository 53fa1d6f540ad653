# A/B of CG-sweep occupancy builds (NST stages, MINB CTAs/SM register budget) on C2 / C3_1600
export GPCG_TRACE=0
echo "default"; timeout 300 python scripts/diag.py C2 C3_1600 2>&1 | grep -E "solve|Error"
for v in 3_5 3_6 2_6; do echo "variant $v"; GPCG_LIB=build_variants/libgpcg_$v.so timeout 300 python scripts/diag.py C2 C3_1600 2>&1 | grep -E "solve|Error"; done
