"""One reduced HVP (gpcg_hessvec) on C3 (8000^2) at the free set of a 2-outer-iteration solve:
the k4_hessvec launch ncu profiles (scripts/gpu_hv_prof.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

prob = P.get(sys.argv[1] if len(sys.argv) > 1 else "C3")
s = gpcg.Solver.from_problem(prob, device="cuda")
x0 = torch.from_numpy(prob.x0).cuda()
rc, x, st = s.solve(x0, prob.tol, max_it=2, allow_error=True)
s.project(x)
v = torch.from_numpy(2.0 * P.uniform(99, 1, prob.n) - 1.0).cuda()
y = torch.empty_like(v)
for _ in range(3):
    s.hessvec(v, y, reduced=True)
torch.cuda.synchronize()
print("free", st["n_free"], "n", prob.n)
