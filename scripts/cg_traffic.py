"""Fixed-length CG calls for an ncu traffic capture of the CG sweep (bench roofline
`traffic`): C2, one outer iteration, every CG call capped at CAP iterations with the
progress test effectively off (eta2 = 1e-10), so `ncu -k regex:k6_cg_loop -c 1` sees a
launch of exactly CAP iterations (checked: the first call's count is printed).

usage: python scripts/cg_traffic.py [CAP] [CONFIG]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

CAP = int(sys.argv[1]) if len(sys.argv) > 1 else 64
prob = P.get(sys.argv[2] if len(sys.argv) > 2 else "C2")
s = gpcg.Solver.from_problem(prob, device="cuda")
s.set_params(cg_cap=CAP, eta2=1e-10, refine_cap=1)
x0 = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
rc, x, st = s.solve(x0, prob.tol, max_it=1)
torch.cuda.synchronize()
print(f"cg_calls={st['cg_calls']} cg_iters={st['cg_iters']} (cap {CAP}) n_free={st['n_free']} "
      f"t_cg_timed_ms={st['t_cg_timed_ms']:.3f} us/iter={1e3 * st['t_cg_timed_ms'] / max(st['cg_iters_timed'], 1):.2f}",
      flush=True)
