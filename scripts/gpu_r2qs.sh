# (the quiet-item skipping this script measured was not kept: scripts/patches/gp_quiet_item_skip.patch)
# r2qs (run as r2g): exact skipping of quiet GP items (GPCG_GP_SKIP) x GP items per CTA
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "quiet_item or golden" > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error|assert" gpurun_out/r2g_pytest.log | tail -8
for I in 1 4 8 16; do
  for K in 0 1; do
    echo "ipc=$I skip=$K"; GPCG_GP_ITEMS_PER_CTA=$I GPCG_GP_SKIP=$K timeout 300 python scripts/gp_ab.py C3 100000 3
  done
done
for I in 1 8 16; do
  echo "full solves ipc=$I"; GPCG_GP_ITEMS_PER_CTA=$I timeout 600 python scripts/diag.py C3 C2 2>&1 | grep solve
done
