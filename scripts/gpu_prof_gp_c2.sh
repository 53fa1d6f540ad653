# ncu --set full of one k6_gp_loop launch on C2 (L2-resident): where the GP step's time goes
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
TAG=${TAG:-r2x}
python -c "import paper_cs_0101018_b200._build as b; b.build()"
timeout 300 python scripts/gp_ab.py C2 100 3 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_gp_loop" -s 1 -c 1 -o /tmp/prof_gp python scripts/gp_ab.py C2 100 3 > gpurun_out/${TAG}_ncu_gp.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/prof_gp.ncu-rep > gpurun_out/${TAG}_gp_c2_summary.txt 2>&1; cat gpurun_out/${TAG}_gp_c2_summary.txt
ncu -i /tmp/prof_gp.ncu-rep --page raw --csv > gpurun_out/${TAG}_gp_c2_raw.csv 2>&1
ncu -i /tmp/prof_gp.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_gp_c2_sass.csv 2>&1
ncu -i /tmp/prof_gp.ncu-rep --page details > gpurun_out/${TAG}_gp_c2_details.txt 2>&1
gzip -f gpurun_out/${TAG}_gp_c2_sass.csv gpurun_out/${TAG}_gp_c2_raw.csv
ls -la gpurun_out | tail -5
