# r2nc: the ranks' graph-chunk path (deferred reductions through a 1-rank NCCL communicator,
# GPCG_FORCE_NCCL=1) on C3 split into 2 / 8 slabs of one GPU: per-step costs of the N > 1 default path
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
for S in 2 8; do
  GPCG_FORCE_NCCL=1 timeout 1500 python bench.py --slabs $S --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2nc_slabs$S.json 2> gpurun_out/r2nc_slabs$S.err; echo "slabs $S rc=$?"
  tail -2 gpurun_out/r2nc_slabs$S.err
done
