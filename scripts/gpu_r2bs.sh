# r2bs: bench.py multi-slab path (--slabs 2, C2) and --xrank at N = 1 (pool off): the JSON line and its labels
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 900 python bench.py --config C2 --slabs 2 --steps 3 --no-cpu-baseline > gpurun_out/r2bs_slabs2.json 2> gpurun_out/r2bs_slabs2.err; echo "slabs2 rc=$?"
timeout 900 python bench.py --config C2 --xrank --steps 3 --no-cpu-baseline > gpurun_out/r2bs_xrank1.json 2> gpurun_out/r2bs_xrank1.err; echo "xrank1 rc=$?"
tail -2 gpurun_out/r2bs_slabs2.err
