# r2h: compact-output reduced HVP (gpcg_hessvec_free, CSR-vector row groups + free bits): parity
# tests, a4 microbenchmark on C4 / C4s, A/B of row-group variants, ncu --set full of one launch each
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "hessvec_free or compact or spmv" > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2h_pytest.log | tail -20
timeout 900 python scripts/a4_compact.py C4 C4s 2>&1 | tail -6
cp gpurun_out/a4_compact.json gpurun_out/r2h_a4_compact.json
for V in hvf_u2 hvf_u8 hvf_l4 hvf_minb4; do echo $V; GPCG_LIB=build_variants/$V.so timeout 600 python scripts/a4_compact.py C4 2>&1 | grep '"cg_mode": 2' ; done
for C in C4 C4s; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hessvec_free --launch-skip 35 -c 1 \
    -o gpurun_out/r2h_ncu_hvf_$C -f python scripts/a4_compact.py $C > gpurun_out/r2h_ncu_$C.log 2>&1; echo "ncu $C rc=$?"
done
