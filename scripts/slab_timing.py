"""Per-iteration CG / GP times of one problem split into S row slabs on one GPU (the multi-slab
persistent loops with fused halo writes, SlabLink in march_tma.cuh) against one slab.

usage: python scripts/slab_timing.py CONFIG S1 S2 ...
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

prob = P.get(sys.argv[1])
x0 = torch.from_numpy(prob.x0).cuda()
for slabs in [int(a) for a in sys.argv[2:]]:
    s = gpcg.Solver.from_problem(prob, device="cuda", slabs=slabs)
    s.solve(x0, prob.tol)                               # warm-up
    torch.cuda.synchronize()
    t0 = time.time()
    rc, x, st = s.solve(x0, prob.tol)
    torch.cuda.synchronize()
    t1 = time.time()
    cg_us = 1e3 * st["t_cg_timed_ms"] / max(st["cg_iters_timed"], 1)
    # per free point and iteration: the CG sweep skips all-active blocks, so the per-iteration time
    # follows the free-set sizes along the path, which differs with the slab count (rounding)
    cg_ps = 1e9 * st["t_cg_timed_ms"] / max(st["cg_free_iters_timed"], 1)
    gp_us = 1e3 * st["t_gp_ms"] / max(st["gp_iters"], 1)
    print(f"{prob.name} slabs={slabs}: solve {t1 - t0:.3f}s rc={rc} outer={st['outer_iters']} gp={st['gp_iters']} "
          f"cg={st['cg_iters']} | CG {cg_us:.1f} us/iter ({cg_ps:.2f} ps per free point) | GP {gp_us:.1f} us/step | launches={st['kernel_launches']} "
          f"q={st['q']:.15g}", flush=True)
    s.close()
