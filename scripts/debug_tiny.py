import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_cs_0101018_b200 import problems as P, gpcg
from tests.test_gpu_parity import ragged_stencil
from oracle import oracle as O
for nx, ny in [(1, 1), (1, 2), (3, 1), (5, 3)]:
    prob = ragged_stencil(nx, ny, 40 + nx + ny)
    A = O.problem_csr(prob)
    with gpcg.Solver.from_problem(prob) as s:
        px, pg2, na, nnb = s.project(prob.x0)
        pref = O.project(prob.l, prob.u, prob.x0)
        g = O.gradient(A, prob.b, pref)
        print(nx, ny, "pg2", pg2, "ref", np.sum(O.proj_grad(pref, g, prob.l, prob.u)**2), "na", na, flush=True)
        rc, x, st = s.solve(prob.x0, -1e-12, allow_error=True)
        print("  rc", rc, gpcg.last_error(), st["outer_iters"], st["gp_iters"], flush=True)
