"""Time gpcg_hessvec (full and reduced) with CUDA events on the configured workloads."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

reps = 50
for name in (sys.argv[1:] or ["C2"]):
    prob = P.get(name)
    stream = torch.cuda.current_stream()
    s = gpcg.Solver.from_problem(prob, device="cuda", stream=stream)
    v = torch.rand(prob.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(v)
    x = torch.from_numpy(prob.x0).cuda() + 0.01 * torch.rand(prob.n, dtype=torch.float64, device="cuda")
    s.project(x)
    for reduced in (False, True):
        for _ in range(5):
            s.hessvec(v, y, reduced)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            s.hessvec(v, y, reduced)
        e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        gbs = (16.0 * prob.n) / (us * 1e-6) / 1e9
        print(f"{name} hessvec reduced={reduced}: {us:.2f} us/launch, {gbs:.1f} GB/s (16 B/pt)", flush=True)
    for _ in range(3):
        s.project(x)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(10):
        s.project(x)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{name} project: {e0.elapsed_time(e1) * 1e3 / 10:.2f} us/call (includes D2D copies + sync)", flush=True)
    s.close()
