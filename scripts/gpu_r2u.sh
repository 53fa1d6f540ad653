# r2u: CG ipc=16 default in pw mode; GP items per CTA sweep
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
GPCG_GP_ITEMS_PER_CTA=4 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "golden or c2" > gpurun_out/r2u_pytest.log 2>&1; echo "pytest(gp ipc 4) rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2u_pytest.log | tail -5
for I in 1 2 4 8; do
  echo "gp ipc=$I"; GPCG_GP_ITEMS_PER_CTA=$I timeout 600 python scripts/diag.py C3 C2 2>&1 | grep solve
done
