# the ghost-depth regression test on the current build, and on a build with 2 ghost rows (must fail)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_slabs.py -m gpu -q -k first_outer > gpurun_out/ghost3.log 2>&1; echo "3 ghosts rc=$?"; tail -2 gpurun_out/ghost3.log
sed -i 's/layout_slabs(h, re - rb, nsl, 3)/layout_slabs(h, re - rb, nsl, 2)/' paper_cs_0101018_b200/csrc/gpcg.cu && python -m paper_cs_0101018_b200._build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_slabs.py -m gpu -q -k first_outer > gpurun_out/ghost2.log 2>&1; echo "2 ghosts rc=$? (expected failures)"; grep -E "passed|failed" gpurun_out/ghost2.log | tail -1
