"""One GP phase of a fixed number of steps for an ncu traffic capture of the persistent GP loop
(bench roofline `traffic` of k6_gp_loop): the first GP phase from x0, capped at CAP steps
(gpcg_params.gp_cap), one outer iteration; `ncu -k regex:k6_gp_loop -c 1` sees exactly the
phase whose step count and rejected speculative sweeps are printed here.

usage: python scripts/gp_traffic.py [CAP] [CONFIG]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

CAP = int(sys.argv[1]) if len(sys.argv) > 1 else 16
prob = P.get(sys.argv[2] if len(sys.argv) > 2 else "C3")
s = gpcg.Solver.from_problem(prob, device="cuda")
s.set_params(gp_cap=CAP, cg_cap=1, refine_cap=1)
x0 = torch.from_numpy(prob.x0).cuda()
rc, x, st = s.solve(x0, prob.tol, max_it=1)
torch.cuda.synchronize()
print(f"gp_iters={st['gp_iters']} (cap {CAP}) gp_spec_rejected={st['gp_spec_rejected']} "
      f"t_gp_ms={st['t_gp_ms']:.3f} us/step={1e3 * st['t_gp_ms'] / max(st['gp_iters'], 1):.2f} n={prob.n}",
      flush=True)
