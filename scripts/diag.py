"""One traced GPCG solve per config on cuda:0 (GPCG_TRACE=1 prints per-phase lines to stderr)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GPCG_TRACE", "1")
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

for name in sys.argv[1:]:
    t0 = time.time()
    prob = P.get(name)
    t1 = time.time()
    s = gpcg.Solver.from_problem(prob, device="cuda")
    x0 = torch.from_numpy(prob.x0).cuda()
    torch.cuda.synchronize()
    t2 = time.time()
    rc, x, st = s.solve(x0, prob.tol)
    torch.cuda.synchronize()
    t3 = time.time()
    print(f"{name}: gen {t1-t0:.2f}s create {t2-t1:.2f}s solve {t3-t2:.3f}s rc={rc} {st}", flush=True)
    s.close()
