"""BASELINE.json's metric on every config (SURVEY.md 8(d) row d): GPCG solve time to tol,
reduced Hessian-vector products/s, the CG iteration's algorithmic GB/s, and the a4 kernel
microbenchmark (one reduced HVP, gpcg_hessvec, at the solution's free set: 5 warm-ups, then
50 reps each after an L2 flush, CUDA events around the launch only, median), with the
oracle timed beside it on a bounded sample on 1 host core.

C3 at full size (8000^2) does not reach tau in a bounded run: it is timed for
max_it = 3 outer iterations and labelled so.

usage: python scripts/metrics_all.py [--out profiles/metrics_r1.json] [--oracle-budget 10] [CONFIGS...]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

MAX_IT = {"C3": 3}


def cg_bytes(prob):
    """Algorithmic bytes per free point of one CG iteration of the kernel this build runs,
    and per grid point (mask): 2-D stencil k4/k6 three-vector recurrence 48 B (+16 B full face
    arrays); 3-D plane march 80 B (rho, q, s, p, w read + written) + 48 B faces / shift;
    CSR 80 B + 8 B row_ptr + 12 B per entry."""
    if prob.kind == "stencil2d":
        return 48.0 + (16.0 if (prob.wx_ld or prob.wy_ld) else 0.0), 1.0
    if prob.kind == "stencil3d":
        return 80.0 + 48.0, 1.0
    z = prob.val.size / prob.n
    return 80.0 + 8.0 + 12.0 * z, 1.0


def hvp_bytes(prob, m):
    """Algorithmic bytes of one reduced HVP (the minimum any kernel must move): p on the free
    set (8 B m), y written (8 B n), mask (1 B n), operator data of the free rows only (full
    2-D faces 16 B, 3-D faces + shift 48 B, CSR 8 B row_ptr + 12 B per entry)."""
    n = prob.n
    b = 8.0 * m + 9.0 * n
    if prob.kind == "stencil2d" and (prob.wx_ld or prob.wy_ld):
        b += 16.0 * m
    elif prob.kind == "stencil3d":
        b += 48.0 * m
    elif prob.kind == "csr":
        b += (8.0 + 12.0 * prob.val.size / n) * m
    return b


def oracle_sample(prob, budget_s):
    from oracle import oracle as O
    A = O.problem_csr(prob)
    params = O.default_params(time_budget_s=float(budget_s))
    t0 = time.perf_counter()
    rc, x, st = O.solve(A, prob.b, prob.l, prob.u, prob.c, prob.x0, prob.tol, 500, params)
    dt = time.perf_counter() - t0
    return {"hvp_per_s": st["cg_iters"] / max(st["seconds"], 1e-9), "cg_iters": st["cg_iters"],
            "seconds": st["seconds"], "wall_s": dt, "completed": bool(rc == 0 and st["seconds"] < budget_s),
            "outer_iters": st["outer_iters"], "cores": 1}


def measure(name, peak, oracle_budget):
    prob = P.get(name)
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream()
    s = gpcg.Solver.from_problem(prob, device=dev, stream=stream)
    x0 = torch.from_numpy(prob.x0).to(dev)
    x = torch.empty_like(x0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    max_it = MAX_IT.get(name, 500)
    s.solve(x0, prob.tol, max_it=max_it, x_out=x, allow_error=True)      # warm-up
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rc, _, st = s.solve(x0, prob.tol, max_it=max_it, x_out=x, allow_error=True)
    e1.record(stream)
    torch.cuda.synchronize()
    solve_s = e0.elapsed_time(e1) / 1e3
    m_free, per_pt = cg_bytes(prob)
    it = max(st["cg_iters_timed"], 1)
    cg_us = 1e3 * st["t_cg_timed_ms"] / it
    cg_gbs = None
    if st["cg_iters_timed"]:
        bpl = (m_free * st["cg_free_iters_timed"] + per_pt * prob.n * st["cg_iters_timed"]) / it
        cg_gbs = bpl / (cg_us * 1e-6) / 1e9
    # a4: reduced HVP at the solution's free set (the handle's free mask after the solve)
    s.project(x)
    v = torch.from_numpy(2.0 * P.uniform(99, 1, prob.n) - 1.0).to(dev)
    y = torch.empty_like(v)
    for _ in range(5):
        s.hessvec(v, y, reduced=True)
    ts = []
    for _ in range(50):
        flush.zero_()
        torch.cuda.synchronize()
        e0.record(stream)
        s.hessvec(v, y, reduced=True)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    hv_us = statistics.median(ts)
    m = st["n_free"]
    hv_b = hvp_bytes(prob, m)
    s.close()
    row = {"config": name, "n": prob.n, "rc": rc, "max_it": max_it, "solve_s": solve_s,
           "outer": st["outer_iters"], "gp_iters": st["gp_iters"], "cg_iters": st["cg_iters"],
           "hvp_per_s": st["cg_iters"] / solve_s, "n_free": m,
           "cg_us_per_iter": cg_us if st["cg_iters_timed"] else None, "cg_alg_gbs": cg_gbs,
           "cg_alg_frac": (cg_gbs / peak) if cg_gbs else None, "cg_bytes_per_free_point": m_free,
           "a4_hvp_us_median": hv_us, "a4_alg_bytes": hv_b, "a4_alg_gbs": hv_b / (hv_us * 1e-6) / 1e9,
           "a4_alg_frac": hv_b / (hv_us * 1e-6) / 1e9 / peak}
    if oracle_budget > 0 and name != "C3":
        row["oracle"] = oracle_sample(prob, oracle_budget)
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--oracle-budget", type=float, default=10.0)
    ap.add_argument("configs", nargs="*", default=["C0", "C1", "C2", "C3_1600", "C3", "C4", "C4s"])
    args = ap.parse_args()
    pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "MEASURED_PEAKS.json")))
    peak = float(pk["hbm_gbs"])
    rows = []
    for name in args.configs:
        r = measure(name, peak, args.oracle_budget)
        rows.append(r)
        print(json.dumps(r), flush=True)
    if args.out:
        json.dump({"what": __doc__.strip().splitlines()[0], "gpu": torch.cuda.get_device_name(0),
                   "peak_gbs": peak, "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
