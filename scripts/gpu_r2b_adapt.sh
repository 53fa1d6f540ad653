# r2b_adapt: adaptive chunk ranges for the speculative GP sweep (GPCG_GP_ADAPT) -- parity, determinism, A/B
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 120 python scripts/gp_ab.py C3 100 3 || { echo "adaptive C3 failed"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "adaptive_ranges or golden" > gpurun_out/r2b_adapt_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r2b_adapt_pytest.log | tail -8
for A in 0 1; do
  echo "adapt=$A"; GPCG_GP_ADAPT=$A timeout 300 python scripts/gp_ab.py C3 100 3
done
for C in 24 96; do
  echo "adapt chunk=$C"; GPCG_GP_CHUNK=$C timeout 300 python scripts/gp_ab.py C3 100 3
done
GPCG_LIB=build_variants/diagt.so timeout 300 python scripts/gp_step_times.py C3 3
for A in 0 1; do
  echo "full solves adapt=$A"; GPCG_GP_ADAPT=$A timeout 600 python scripts/diag.py C3 C2 2>&1 | grep solve
done
