"""Paper-setting runs (SURVEY.md 8(f) NEXT-4, C2' of 8(d)): the journal-bearing problem
with the paper's algorithm settings -- tau = 1e-4 absolute, x0 = l, eta1 = 0.1, eta2 =
0.05 -- at the paper's sizes, with plain CG and with the point-Jacobi
preconditioner (the "Diagonal" column of Table 4), on one B200.  Prints
iterations, n_GP, CG iterations, t_CG % and seconds next to the paper's IBM SP numbers
(context only: FD instead of the FE discretisation, B200 instead of the SP, 32x32-tile
blocks instead of one block per processor for the paper's block-Jacobi ILU(2) of Tables 1/2).

usage: python scripts/paper_setting.py [--out profiles/paper_setting.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402

# (grid, eps) -> the paper's rows: Table 1 (n = 2,560,000, BJ-ILU(2), p = 8 .. 64),
# Table 2 (n = 640,000), Table 4 (n = 640,000, Diagonal preconditioner, p = 4 / 16)
PAPER = {
    (1600, 0.1): {"table": "T1 (BJ-ILU(2))", "iters": 46, "n_GP": 431, "t_cg_pct": 86,
                  "time_s": {"p=8": 7419, "p=64": 1279}},
    (1600, 0.9): {"table": "T1 (BJ-ILU(2))", "iters": 37, "n_GP": 105, "t_cg_pct": 70,
                  "time_s": {"p=8": 2134, "p=64": 397}},
    (800, 0.1): {"table": "T4 Diagonal", "iters": 26, "cg_iters": 37045, "time_s": {"p=4": 2928, "p=16": 851}},
    (800, 0.9): {"table": "T4 Diagonal", "iters": 21, "cg_iters": 18118, "time_s": {"p=4": 1216, "p=16": 390}},
}


PRECOND_NAMES = {0: "none", 1: "jacobi", 2: "bj-ilu0 (32x32 tiles)", 3: "bj-ilu2 (32x32 tiles)"}


def run(grid, eps, precond):
    prob = P.journal_bearing(grid, grid, eps)
    s = gpcg.Solver.from_problem(prob, device="cuda")
    s.set_params(precond=precond)
    x0 = torch.zeros(prob.n, dtype=torch.float64, device="cuda")    # x0 = l
    s.solve(x0, 1e-4)                                                  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc, x, st = s.solve(x0, 1e-4)                                      # tau = 1e-4 absolute
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    s.close()
    return {"grid": grid, "n": prob.n, "eps": eps, "precond": PRECOND_NAMES[precond], "rc": rc,
            "iters": st["outer_iters"], "n_GP": st["gp_iters"], "cg_iters": st["cg_iters"],
            "t_cg_pct": round(100.0 * st["t_cg_ms"] / max(st["t_total_ms"], 1e-9), 1), "seconds": dt,
            "free_fraction": st["n_free"] / prob.n, "q": st["q"], "pg_norm": st["pg_norm"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for grid, eps in [(800, 0.1), (800, 0.9), (1600, 0.1), (1600, 0.9)]:
        for pc in (0, 1, 2, 3):
            r = run(grid, eps, pc)
            r["paper"] = PAPER[(grid, eps)]
            rows.append(r)
            print(json.dumps(r), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"what": __doc__.strip().splitlines()[0], "gpu": torch.cuda.get_device_name(0),
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
