# r2s: CG items per CTA (shorter segments, round-robin) in the per-warp-box (large grid) mode
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "box_layouts or golden or c2" > gpurun_out/r2s_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2s_pytest.log | tail -5
for I in 1 2 4 8; do
  echo "ipc=$I"; GPCG_CG_ITEMS_PER_CTA=$I timeout 600 python scripts/diag.py C3 2>&1 | grep solve
done
