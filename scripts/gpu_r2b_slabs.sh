# r2b_slabs: multi-slab persistent loops vs one slab, per free point (CG) and per step (GP); C2 and C3
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 900 python scripts/slab_timing.py C2 1 2 4 2>&1 | grep slabs
timeout 1200 python scripts/slab_timing.py C3 1 2 2>&1 | grep slabs
