# r2j: dynamic item claiming in the speculative GP sweep (GPCG_GP_DYN) x items per CTA
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 120 python scripts/gp_ab.py C2 100 3 || { echo "dyn C2 failed"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "dynamic_items or golden" > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r2j_pytest.log | tail -8
for D in 0 1; do
  for I in 4 8 16; do
    echo "dyn=$D ipc=$I"; GPCG_GP_DYN=$D GPCG_GP_ITEMS_PER_CTA=$I timeout 300 python scripts/gp_ab.py C3 100 3
  done
done
GPCG_GP_DYN=0 GPCG_GP_ITEMS_PER_CTA=1 timeout 300 python scripts/gp_ab.py C3 100 3
for D in 0 1; do
  echo "full solves dyn=$D"; GPCG_GP_DYN=$D timeout 600 python scripts/diag.py C3 C2 2>&1 | grep solve
done
