"""One traced GPCG solve per config on cuda:0 (GPCG_TRACE=1 prints per-phase lines to stderr)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if not os.environ.get("GPCG_TRACE_OFF"):
    os.environ.setdefault("GPCG_TRACE", "1")
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

for name in sys.argv[1:]:
    t0 = time.time()
    prob = P.get(name)
    t1 = time.time()
    s = gpcg.Solver.from_problem(prob, device="cuda")
    if os.environ.get("GPCG_PRECOND"):
        s.set_params(precond=int(os.environ["GPCG_PRECOND"]))
    x0 = torch.from_numpy(prob.x0).cuda()
    torch.cuda.synchronize()
    t2 = time.time()
    rc, x, st = s.solve(x0, prob.tol)
    torch.cuda.synchronize()
    t3 = time.time()
    cg_us = 1e3 * st["t_cg_timed_ms"] / max(st["cg_iters_timed"], 1)
    gp_us = 1e3 * st["t_gp_ms"] / max(st["gp_iters"], 1)
    print(f"{name}: solve {t3-t2:.3f}s rc={rc} outer={st['outer_iters']} gp={st['gp_iters']} cg={st['cg_iters']} "
          f"| CG {cg_us:.1f} us/iter (steady) | GP {gp_us:.1f} us/step | t_cg {st['t_cg_ms']:.0f} ms "
          f"t_gp {st['t_gp_ms']:.0f} ms | q={st['q']:.15g} free={st['n_free']} launches={st['kernel_launches']}",
          flush=True)
    s.close()
