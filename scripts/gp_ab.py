"""GP-step time of the persistent GP loop on a fixed amount of work: the first GP phase from x0,
capped at CAP steps, one outer iteration (A/B of libgpcg.so builds via GPCG_LIB).

usage: python scripts/gp_ab.py CONFIG [CAP] [MAX_IT]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

prob = P.get(sys.argv[1])
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 300
max_it = int(sys.argv[3]) if len(sys.argv) > 3 else 1
s = gpcg.Solver.from_problem(prob, device="cuda")
s.set_params(gp_cap=cap, cg_cap=1, refine_cap=1)
x0 = torch.from_numpy(prob.x0).cuda()
best = None
for rep in range(3):
    rc, x, st = s.solve(x0, prob.tol, max_it=max_it)
    us = 1e3 * st["t_gp_ms"] / max(st["gp_iters"], 1)
    best = us if best is None else min(best, us)
print(f"{sys.argv[1]} GP phase: {st['gp_iters']} steps ({st['gp_spec_rejected']} rejected) best {best:.1f} us/step "
      f"lib={os.environ.get('GPCG_LIB') or 'default'}", flush=True)
