"""C3 family: effect of the GP-phase cap (gpcg_params.gp_cap, reading R13) on the outer
iteration count.  usage: python scripts/c3_gpcap.py C3_3200 100 1000 100000"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

name = sys.argv[1]
prob = P.get(name)
for cap in [int(c) for c in sys.argv[2:]]:
    s = gpcg.Solver.from_problem(prob, device="cuda")
    s.set_params(gp_cap=cap)
    x0 = torch.from_numpy(prob.x0).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc, x, st = s.solve(x0, prob.tol, max_it=500, allow_error=True)
    torch.cuda.synchronize()
    print(f"{name} gp_cap={cap}: rc={rc} {time.perf_counter() - t0:.2f}s outer={st['outer_iters']} "
          f"gp={st['gp_iters']} cg={st['cg_iters']} pg={st['pg_norm']:.3e} q={st['q']:.15g}", flush=True)
    s.close()
