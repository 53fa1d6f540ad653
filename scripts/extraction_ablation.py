"""Extraction ablation (the paper's design choice P:675-700): the
same GPCG solves with A_k applied in place on masked vectors (cg_mode 0, the hot path)
and with A_k extracted as a compact CSR matrix each CG call (cg_mode 1, PETSc's
MatGetSubMatrix route).  Reports solve time, CG time, extraction time and iteration counts.

usage: python scripts/extraction_ablation.py [--out profiles/extraction_ablation_r1.json] [CONFIGS...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_cs_0101018_b200 import problems as P, gpcg  # noqa: E402


def run(name, mode):
    prob = P.get(name)
    s = gpcg.Solver.from_problem(prob, device="cuda")
    s.set_params(cg_mode=mode)
    x0 = torch.from_numpy(prob.x0).cuda()
    s.solve(x0, prob.tol)                         # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc, x, st = s.solve(x0, prob.tol)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    s.close()
    return {"config": name, "n": prob.n, "cg_mode": mode, "rc": rc, "seconds": dt, "outer": st["outer_iters"],
            "gp_iters": st["gp_iters"], "cg_iters": st["cg_iters"], "cg_calls": st["cg_calls"],
            "t_cg_ms": st["t_cg_ms"], "t_extract_ms": st["t_extract_ms"], "n_free": st["n_free"], "q": st["q"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3_1600", "C4", "C4s"])
    args = ap.parse_args()
    rows = []
    for name in args.configs:
        for mode in (0, 1):
            r = run(name, mode)
            rows.append(r)
            print(json.dumps(r), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"what": __doc__.strip().splitlines()[0], "gpu": torch.cuda.get_device_name(0), "rows": rows},
                      f, indent=1)


if __name__ == "__main__":
    main()
