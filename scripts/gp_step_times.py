"""Where a persistent GP step's time goes (diagnostic build with -DGPCG_DIAG_TIMES): per step of
the last k6_gp_loop launch, each CTA's globaltimer stamps -- step start, sweep done, grid barrier
passed, sums formed -- summarised over the steps: sweep time per CTA (min / median / max), the
wait of the first-finishing CTA for the last one, barrier latency after the last arrival, and
the reduction.

usage: GPCG_LIB=build_variants/diagt.so python scripts/gp_step_times.py CONFIG [MAX_IT]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

prob = P.get(sys.argv[1])
max_it = int(sys.argv[2]) if len(sys.argv) > 2 else 3
s = gpcg.Solver.from_problem(prob, device="cuda")
x0 = torch.from_numpy(prob.x0).cuda()
rc, x, st = s.solve(x0, prob.tol, max_it=max_it)
buf = np.zeros((64, 512, 5), dtype=np.uint64)
lib = gpcg.load()
assert lib.gpcg_diag_gp_times(buf.ctypes.data_as(C.POINTER(C.c_ulonglong))) == 0
s.close()
t = buf.astype(np.float64)
ok = (t[:, :, 0] > 0).sum(axis=1)
ncta = int(ok.max())
rows = []
for k in range(64):
    if ok[k] < ncta:
        continue
    a = t[k, :ncta]
    if np.any(a[:, 3] == 0) or np.any(a[:, 3] < a[:, 0]):
        continue
    start, done, passed, summed = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
    sweep = (done - start) / 1e3
    rows.append(dict(step_us=(summed.max() - start.min()) / 1e3, sweep_min=sweep.min(), sweep_med=np.median(sweep),
                     sweep_max=sweep.max(), finish_spread=(done.max() - done.min()) / 1e3,
                     barrier_after_last=(passed.max() - done.max()) / 1e3, pass_spread=(passed.max() - passed.min()) / 1e3,
                     reduce=np.median(summed - passed) / 1e3, start_spread=(start.max() - start.min()) / 1e3))
# per-CTA sweep time (median over steps) against its SM's CTA count, band and segment
good = [k for k in range(64) if ok[k] >= ncta and np.all(t[k, :ncta, 3] > 0)]
sw = np.median(np.stack([(t[k, :ncta, 1] - t[k, :ncta, 0]) / 1e3 for k in good]), axis=0)
sm = t[good[0], :ncta, 4].astype(int)
per_sm = np.bincount(sm, minlength=sm.max() + 1)
nb = s_nb = None
print("CTAs per SM:", np.bincount(per_sm[per_sm > 0]))
for c in (1, 2, 3, 4):
    sel = per_sm[sm] == c
    if sel.any():
        print(f"  CTAs on SMs with {c} CTAs: {sel.sum():4d}  sweep us min {sw[sel].min():7.1f} median {np.median(sw[sel]):7.1f} max {sw[sel].max():7.1f}")
order = np.argsort(sw)[::-1][:12]
print("slowest CTAs (blockIdx, sm, us):", [(int(i), int(sm[i]), round(float(sw[i]), 1)) for i in order])
print("fastest CTAs (blockIdx, sm, us):", [(int(i), int(sm[i]), round(float(sw[i]), 1)) for i in np.argsort(sw)[:6]])
print("sweep us by blockIdx % 39 (band at C3):", np.round([np.median(sw[np.arange(ncta) % 39 == b]) for b in range(39)], 0).tolist())
print(f"{prob.name}: {len(rows)} complete steps of the last launch, {ncta} CTAs (us, median over steps)")
for key in rows[0]:
    v = np.array([r[key] for r in rows])
    print(f"  {key:20s} median {np.median(v):9.2f}  min {v.min():9.2f}  max {v.max():9.2f}")
