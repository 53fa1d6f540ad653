"""Freeze the obstacle constants of C1 and C3 (DESIGN.md input recipe).

Calls only oracle/ (the CPU reference) and the input generators; prints the
bisection trace.  The constants it finds are typed into problems.py
(C1_OBSTACLE_A, C3_OBSTACLE_C).  Targets: ~40% active at the solution for C1
(BASELINE.json configs[1]) and ~50% active for C3 (configs[3]), the latter on a
down-scaled member since the obstacles are mesh-independent.
"""
import math
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O                     # noqa: E402
from paper_cs_0101018_b200 import problems as P     # noqa: E402


def active_fraction(prob):
    rc, x, st = O.solve_problem(prob, tol=-1e-8)
    assert rc == 0, rc
    return st["n_active"] / prob.n


def bisect(make, lo, hi, target, increasing, iters=14):
    """Geometric bisection of a scalar so that active_fraction(make(s)) ~ target."""
    for _ in range(iters):
        mid = math.sqrt(lo * hi)
        f = active_fraction(make(mid))
        print(f"  s={mid:.6g} active={f:.4f}", flush=True)
        if (f < target) == increasing:
            lo = mid
        else:
            hi = mid
    return math.sqrt(lo * hi)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("c1", "all"):
        print("C1: a such that |A(x*)|/n = 0.40 at 400x400")
        a = bisect(lambda a: P.c1_family(a=a), 1e-5, 1e-3, 0.40, increasing=False)
        print(f"C1_OBSTACLE_A = {a:.4g}  (check: {active_fraction(P.c1_family(a=float(f'{a:.4g}'))):.4f})")
    if which in ("c3", "all"):
        nx = int(sys.argv[2]) if len(sys.argv) > 2 else 200
        lo = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3      # optional bracket
        hi = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
        its = int(sys.argv[5]) if len(sys.argv) > 5 else 14
        print(f"C3: c such that |A(x*)|/n = 0.50 at {nx}x{nx}")
        c = bisect(lambda c: P.c3_family(nx, nx, c=c), lo, hi, 0.50, increasing=False, iters=its)
        print(f"C3_OBSTACLE_C = {c:.4g}  (check: {active_fraction(P.c3_family(nx, nx, c=float(f'{c:.4g}'))):.4f})")
