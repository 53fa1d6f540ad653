"""Preconditioners on the bench workloads (C2 / C1 / C3 1600^2 member, tol of BASELINE.json):
plain CG (the hot path), point Jacobi, block-Jacobi ILU(0) / ILU(2) -- solve time and iteration counts.

usage: python scripts/precond_compare.py [--out profiles/precond_compare_r1.json] [CONFIGS...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

NAMES = {0: "none", 1: "jacobi", 2: "bj-ilu0 (32x32 tiles)", 3: "bj-ilu2 (32x32 tiles)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3_1600"])
    args = ap.parse_args()
    rows = []
    for name in args.configs:
        prob = P.get(name)
        for pc in (0, 1, 2, 3):
            s = gpcg.Solver.from_problem(prob, device="cuda")
            s.set_params(precond=pc)
            x0 = torch.from_numpy(prob.x0).cuda()
            s.solve(x0, prob.tol)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc, x, st = s.solve(x0, prob.tol)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            s.close()
            r = {"config": name, "precond": NAMES[pc], "rc": rc, "seconds": dt, "outer": st["outer_iters"],
                 "gp_iters": st["gp_iters"], "cg_iters": st["cg_iters"], "t_cg_ms": st["t_cg_ms"],
                 "us_per_cg_iter": 1e3 * st["t_cg_timed_ms"] / max(st["cg_iters_timed"], 1), "q": st["q"]}
            rows.append(r)
            print(json.dumps(r), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"what": __doc__.strip().splitlines()[0], "gpu": torch.cuda.get_device_name(0), "rows": rows},
                      f, indent=1)


if __name__ == "__main__":
    main()
