# tests + A/B of kernel variants: GPCG_TILE bit sets x GPCG_GP_GRAPH (see gpcg.cu)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for GG in ${GPGRAPH:-1 0}; do
for T in ${TILES:-63 15}; do echo "GPCG_TILE=$T GPCG_GP_GRAPH=$GG"; GPCG_GP_GRAPH=$GG GPCG_TILE=$T GPCG_TRACE=0 timeout 300 python scripts/diag.py ${CONFIGS:-C0 C2} 2>&1 | grep -E "solve|Error|error"; done
done
