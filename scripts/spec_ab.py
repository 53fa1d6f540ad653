"""GP phase of the generic operators with and without the speculative h = 0 sweep (k_spec):
solve time, GP steps, GP-phase time per step.  Run once per setting of GPCG_GP_SPEC (read at
create).  usage: GPCG_GP_SPEC=0|1 python scripts/spec_ab.py C4 C4s"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

for name in sys.argv[1:]:
    prob = P.get(name)
    x0 = torch.from_numpy(prob.x0).cuda()
    with gpcg.Solver.from_problem(prob, device="cuda") as s:
        s.solve(x0, prob.tol)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc, x, st = s.solve(x0, prob.tol)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
    print(f"{name} GPCG_GP_SPEC={os.environ.get('GPCG_GP_SPEC', '1')}: solve {min(ts) * 1e3:.2f} ms rc={rc} "
          f"outer={st['outer_iters']} gp={st['gp_iters']} cg={st['cg_iters']} | GP phase {st['t_gp_ms']:.2f} ms "
          f"({1e3 * st['t_gp_ms'] / max(st['gp_iters'], 1):.1f} us/step) | q={st['q']:.15g}", flush=True)
