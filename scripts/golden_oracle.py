"""Write tests/golden/oracle_<name>.json: the CPU oracle's solution of a full-size
(or down-scaled) config, sampled at seeded indices, for the GPU parity tests at
sizes the oracle cannot finish inside a test run (SURVEY.md 8(c) "Parity").

Calls only oracle/ (the plain-C GPCG) and the seeded input generators; no value
comes from the CUDA path.

usage: python scripts/golden_oracle.py NAME [NAME ...]
  NAME in: C2 (1600^2, configs[2]), C3_1600 (C3 family, 1600^2 member),
           C4_128 (C4 family, 128^3 member)
"""
import base64
import json
import os
import sys
import time
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_cs_0101018_b200 import problems as P  # noqa: E402

# (problem factory, relative tol): the polish tolerance of the parity protocol
# (both sides solved well below the configured tau so that the
# 1e-7 x-parity is certified by ||grad_Omega q|| / lambda_min).
CASES = {
    "C2": (lambda: P.c2(), -1e-10),
    "C3_1600": (lambda: P.c3_family(1600, 1600), -1e-10),
    "C4_128": (lambda: P.c4_family(m=128), -1e-10),
    "C4": (lambda: P.c4(), -1e-10),
}
NSAMPLE = 16384


def sample_indices(n, k=NSAMPLE):
    idx = np.unique((P.uniform(2026, 1, k) * n).astype(np.int64))
    return idx


def main():
    for name in sys.argv[1:]:
        make, tol = CASES[name]
        prob = make()
        t0 = time.time()
        rc, x, st = O.solve_problem(prob, tol=tol)
        secs = time.time() - t0
        A = O.problem_csr(prob)
        g = O.gradient(A, prob.b, x)
        act, bnd, na, nb = O.sets(x, g, prob.l, prob.u)
        idx = sample_indices(prob.n)
        # 1e-7 window around each bound, for the tie rule of the active-set comparison
        near = np.flatnonzero((~act) & ((np.abs(x - prob.l) <= 1e-7) | (np.abs(x - prob.u) <= 1e-7)))
        # the whole active set (bit-packed, zlib, base64): the GPU test compares it point by point
        act_z = base64.b64encode(zlib.compress(np.packbits(act.astype(np.uint8)).tobytes(), 9)).decode()
        # ties: the oracle's free points within 1e-7 of a bound, with x and |g| there
        gnear = np.abs(g[near])
        out = {
            "name": name, "problem": prob.name, "n": int(prob.n), "tol": tol, "rc": int(rc),
            "oracle_seconds": secs, "stats": {k: (float(v) if isinstance(v, float) else int(v))
                                               for k, v in st.items()},
            "q": float(st["q"]), "pg_norm": float(st["pg_norm"]), "n_active": int(na),
            "n_active_nonbinding": int(na - nb),
            "idx": idx.tolist(), "x": [float(v) for v in x[idx]],
            "active_sample": [int(v) for v in act[idx]],
            "n_free_near_bound": int(near.size),
            "near_idx": near.tolist(), "near_x": [float(v) for v in x[near]],
            "near_absg": [float(v) for v in gnear],
            "active_packbits_zlib_b64": act_z,
            "active_sum_index": int(np.sum(np.flatnonzero(act) % 1000003)),
            "source": "scripts/golden_oracle.py -> oracle/gpcg_oracle.c (plain C, fp64, 1 thread)",
        }
        path = os.path.join(ROOT, "tests", "golden", f"oracle_{name}.json")
        with open(path, "w") as f:
            json.dump(out, f)
        print(f"{name}: rc={rc} q={st['q']:.15g} pg={st['pg_norm']:.3e} outer={st['outer_iters']} "
              f"cg={st['cg_iters']} {secs:.0f}s -> {path}", flush=True)


if __name__ == "__main__":
    main()
