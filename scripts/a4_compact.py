"""a4 microbenchmark for the small-free regime: one reduced HVP
gpcg_hessvec(reduced=1) at the SOLUTION's free set of C4 (CSR) and C4s (3-D stencil), through
the masked full-length kernel (cg_mode 0) and the compacted free-row list (cg_mode 2 / 3),
L2 flushed before every rep (the call enqueued while the flush runs, so the events time the
GPU work and not the host's launch latency), CUDA events around each call (the call clears y off F with a
memset, then runs the free-row kernels over F), and the compact-output product
gpcg_hessvec_free (|F| outputs in the reduced space, no clear) for the free-row modes.  Also one
solve per mode (CG in place over F vs masked full-length).

usage: python scripts/a4_compact.py [C4 C4s]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
out = []
flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 1 GB: keeps the GPU busy while the host enqueues the call
for name in (sys.argv[1:] or ["C4", "C4s"]):
    prob = P.get(name)
    stream = torch.cuda.current_stream()
    x0 = torch.from_numpy(prob.x0).cuda()
    for mode in (0, 2):
        s = gpcg.Solver.from_problem(prob, device="cuda", stream=stream)
        s.set_params(cg_mode=mode)
        s.solve(x0, prob.tol)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc, x, st = s.solve(x0, prob.tol)
        torch.cuda.synchronize()
        ts = time.perf_counter() - t0
        m = st["n_free"]
        v = torch.rand(prob.n, dtype=torch.float64, device="cuda")
        y = torch.empty_like(v)
        for _ in range(5):
            s.hessvec(v, y, True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tt = []
        for _ in range(30):
            torch.cuda.synchronize()
            flush.zero_()              # no sync: the host enqueues the call while the flush runs
            e0.record(stream)
            s.hessvec(v, y, True)
            e1.record(stream)
            torch.cuda.synchronize()
            tt.append(e0.elapsed_time(e1) * 1e3)
        us = sorted(tt)[len(tt) // 2]
        if prob.kind == "csr":
            z = prob.val.size / prob.n
            alg = (8.0 + 12.0 * z + 16.0 + 4.0) * m          # 112 m at z = 7
            what = "SURVEY 8(d) CSR: m (8 row_ptr + 12 z col/val + 16 p/write + 4 free-list)"
        else:
            alg = (4.0 + 6 * 8.0 + 8.0 + 8.0) * m            # list + 6 face weights + x + y per free row
            what = "3-D stencil: m (4 free-list + 48 face weights + 8 x + 8 y)"
        zero = 8.0 * prob.n
        # the compact-output product (gpcg_hessvec_free: |F| outputs, no n-long clear)
        us_free = None
        if mode != 0:
            yc = torch.empty(max(s.free_count(), 1), dtype=torch.float64, device="cuda")
            for _ in range(5):
                s.hessvec_free(v, yc)
            tf = []
            for _ in range(30):
                torch.cuda.synchronize()
                flush.zero_()          # no sync: the host enqueues the call while the flush runs
                e0.record(stream)
                s.hessvec_free(v, yc)
                e1.record(stream)
                torch.cuda.synchronize()
                tf.append(e0.elapsed_time(e1) * 1e3)
            us_free = sorted(tf)[len(tf) // 2]
        r = {"config": name, "cg_mode": mode, "n": prob.n, "n_free": m, "solve_s": ts, "rc": rc,
             "cg_iters": st["cg_iters"], "hvp_us": us, "alg_bytes": alg, "alg_what": what,
             "frac_alg": alg / (us * 1e-6) / 1e9 / peak, "zero_fill_bytes": zero,
             "frac_alg_plus_zero_fill": (alg + zero) / (us * 1e-6) / 1e9 / peak, "peak_gbs": peak,
             "hvp_free_us": us_free,
             "frac_alg_free": (alg / (us_free * 1e-6) / 1e9 / peak) if us_free else None}
        print(json.dumps(r), flush=True)
        out.append(r)
        s.close()
json.dump(out, open("gpurun_out/a4_compact.json", "w"), indent=1)
