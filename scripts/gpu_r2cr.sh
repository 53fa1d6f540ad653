# r2cr: one-slab CSR create (arrays uploaded as given, device-side validation), compact CG timing
# accounting, generic-operator GP roofline in bench: GPU suite, C4 bench line
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2cr_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2cr_pytest.log | tail -20
timeout 900 python bench.py --config C4 --steps 10 > gpurun_out/r2cr_bench_C4.json 2> gpurun_out/r2cr_bench_C4.err; echo "bench C4 rc=$?"
tail -3 gpurun_out/r2cr_bench_C4.err
