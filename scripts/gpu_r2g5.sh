# r2g5: k5_spec in the 2-D GP graph chunks (the ranks' path): GPU suite, C3 proxy of the ranks' path
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2g5_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2g5_pytest.log | tail -20
for S in 2 8; do
  GPCG_FORCE_NCCL=1 timeout 1500 python bench.py --slabs $S --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2g5_slabs$S.json 2> gpurun_out/r2g5_slabs$S.err; echo "slabs $S rc=$?"
done
