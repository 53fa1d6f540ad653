# r2s2: speculative GP step of the generic operators (k_spec: CSR / 3-D), full GPU suite + C4 / C4s A/B
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s2_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2s2_pytest.log | tail -20
for S in 0 1; do GPCG_GP_SPEC=$S timeout 900 python scripts/spec_ab.py C4 C4s; done 2>&1 | tee gpurun_out/r2s2_spec_ab.txt
