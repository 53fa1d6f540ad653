# r2b_power: SM clock / power / throttle reasons sampled (nvidia-smi, 100 ms) during GP-only work
# (first outer iterations of C3 with long GP phases) and during a whole C3 solve
mkdir -p gpurun_out
export GPCG_TRACE_OFF=1
python -c "import paper_cs_0101018_b200._build as b; b.build()"
Q="clocks.sm,clocks.max.sm,power.draw,power.limit,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,temperature.gpu"
nvidia-smi --query-gpu=$Q --format=csv,noheader,nounits -lms 100 > gpurun_out/r2b_power_gp.csv & P=$!
timeout 300 python scripts/gp_ab.py C3 100000 4
kill $P
nvidia-smi --query-gpu=$Q --format=csv,noheader,nounits -lms 100 > gpurun_out/r2b_power_solve.csv & P=$!
timeout 300 python scripts/diag.py C3 2>&1 | grep solve
kill $P
nvidia-smi --query-gpu=$Q --format=csv,noheader,nounits -lms 100 > gpurun_out/r2b_power_idle.csv & P=$!
sleep 3
kill $P
for f in gp solve idle; do
python - "$f" <<'PY'
import sys, numpy as np
rows=[l.split(',') for l in open(f"gpurun_out/r2b_power_{sys.argv[1]}.csv") if l.strip()]
sm=np.array([float(r[0]) for r in rows]); pw=np.array([float(r[2]) for r in rows]); lim=float(rows[0][3])
cap=np.mean([r[4].strip().lower().startswith('active') for r in rows])
busy=pw>0.5*lim
print(f"{sys.argv[1]:6s} samples {len(rows)}: SM MHz median {np.median(sm):.0f} (busy samples {np.median(sm[busy]) if busy.any() else 0:.0f}), "
      f"power median {np.median(pw):.0f} W (busy {np.median(pw[busy]) if busy.any() else 0:.0f} W) of limit {lim:.0f} W, sw_power_cap in {100*cap:.0f} % of samples, max temp {max(float(r[6]) for r in rows):.0f} C")
PY
done
