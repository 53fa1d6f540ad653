"""Pin the CPU oracle to things other than itself (run with -m "not gpu").

Each test names the passage (PAPER.md / SPEC.md line) or the mathematical
fact it checks.  References are built independently in tests/_brute.py.
"""
import json
import math
import os

import numpy as np
import pytest

from paper_cs_0101018_b200 import problems as P
from tests import _brute as B

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def csr_of(O, A):
    rp, ci, va = P.dense_to_csr(A)
    return O.CSR(A.shape[0], rp, ci, va)


# ---------------------------------------------------------------- operator
def test_spmv_spec_values(oracle):
    # A=I3 x=(1,2,3) -> (1,2,3); [[2,-1],[-1,2]](1,1) = (1,1)
    A = csr_of(oracle, np.eye(3))
    assert np.array_equal(oracle.spmv(A, [1.0, 2.0, 3.0]), [1.0, 2.0, 3.0])
    A = csr_of(oracle, np.array([[2.0, -1.0], [-1.0, 2.0]]))
    assert np.array_equal(oracle.spmv(A, [1.0, 1.0]), [1.0, 1.0])


def test_spmv_dense_bruteforce(oracle):
    # random 50x50 SPD vs dense product within 1e-12
    A, b, l, u = P.random_dense_qp(50, seed=7, bounds="inf")
    x = P.gaussian(7, 40, 50)
    y = oracle.spmv(csr_of(oracle, A), x)
    assert np.max(np.abs(y - A @ x)) <= 1e-12 * np.max(np.abs(A) @ np.abs(x))


@pytest.mark.parametrize("nx,ny,full,shift", [(7, 5, True, True), (6, 9, False, False), (1, 1, False, False),
                                              (11, 1, True, False), (1, 8, False, True)])
def test_stencil_assembly_matches_grad_form(oracle, nx, ny, full, shift):
    # The oracle's 5-point assembly == G'WG assembled by a different route (BASELINE.json configs[0])
    seed = nx * 100 + ny
    if full:
        wx = 0.5 + P.uniform(seed, 1, ny * (nx + 1)); wx_ld = nx + 1
        wy = 0.5 + P.uniform(seed, 2, (ny + 1) * nx); wy_ld = nx
    else:
        wx = 0.5 + P.uniform(seed, 1, nx + 1); wx_ld = 0
        wy = 0.5 + P.uniform(seed, 2, nx); wy_ld = 0
    sh = P.uniform(seed, 3, nx * ny) if shift else None
    Ad = B.dense_stencil_grad_form(nx, ny, wx, wx_ld, wy, wy_ld, sh)
    A = oracle.stencil2d_to_csr(nx, ny, wx, wx_ld, wy, wy_ld, sh)
    assert np.allclose(A.todense(), Ad, rtol=0, atol=1e-15)
    x = P.gaussian(seed, 4, nx * ny)
    assert np.max(np.abs(oracle.spmv(A, x) - Ad @ x)) <= 1e-13 * max(1.0, np.max(np.abs(Ad) @ np.abs(x)))


def test_stencil_eps0_eigenpairs(oracle):
    # eps=0: A is the constant-coefficient anisotropic Laplacian; sin x sin modes are exact eigenvectors
    nx, ny = 13, 9
    p = P.journal_bearing(nx, ny, eps=0.0)
    A = oracle.problem_csr(p)
    hx, hy = p.meta["hx"], p.meta["hy"]
    for (pp, qq) in [(1, 1), (3, 2), (13, 9), (7, 4)]:
        v, lam = B.laplacian_eigpair(nx, ny, hx, hy, pp, qq)
        Av = oracle.spmv(A, v)
        assert np.max(np.abs(Av - lam * v)) <= 1e-13 * max(lam, 1.0) * (hy / hx + hx / hy) * 4


def test_masked_spmv_spec_and_submatrix(oracle):
    # SPEC.md:68 / S:345: tridiag(-1,2,-1), free={0,2} -> A_k = diag(2,2)
    T = np.array([[2.0, -1, 0], [-1, 2, -1], [0, -1, 2]])
    A = csr_of(oracle, T)
    fr = np.array([1, 0, 1], np.uint8)
    assert np.array_equal(oracle.spmv_masked(A, fr, [1.0, 5.0, 1.0]), [2.0, 0.0, 2.0])
    # general: equals the dense principal submatrix product (P:434-437 A_k = Z'AZ)
    Ad, b, l, u = P.random_dense_qp(30, seed=3, bounds="inf")
    A = csr_of(oracle, Ad)
    fr = (P.uniform(3, 30, 30) < 0.6).astype(np.uint8)
    x = P.gaussian(3, 31, 30)
    F = np.flatnonzero(fr)
    Z = np.eye(30)[:, F]
    ref = Z @ (Z.T @ Ad @ Z) @ (Z.T @ x)
    assert np.max(np.abs(oracle.spmv_masked(A, fr, x) - ref)) <= 1e-12 * np.max(np.abs(Ad) @ np.abs(x))
    # q_k(w) = q(x + Zw) - q(x) = 1/2 w'A_k w + r_k'w  (Eq. cg2)
    xx = P.gaussian(3, 32, 30)
    w = P.gaussian(3, 33, 30) * fr
    r = Ad @ xx - b
    qk = 0.5 * w @ oracle.spmv_masked(A, fr, w) + r[F] @ w[F]
    assert abs(qk - (B.q_dense(Ad, b, 0, xx + w) - B.q_dense(Ad, b, 0, xx))) <= 1e-10 * (1 + abs(qk))


# ---------------------------------------------------------------- projection and sets
def test_projection_spec_values(oracle):
    # SPEC.md:97-99
    assert np.array_equal(oracle.project([0, 0, 0], [1, 1, 1], [-1, 0.5, 2]), [0, 0.5, 1])
    assert oracle.project([0], [np.inf], [7.0])[0] == 7.0
    x = P.gaussian(1, 50, 100)
    l = -np.abs(P.gaussian(1, 51, 100)); u = np.abs(P.gaussian(1, 52, 100))
    px = oracle.project(l, u, x)
    assert np.all(px >= l) and np.all(px <= u)
    assert np.array_equal(oracle.project(l, u, px), px)               # idempotent


def test_projected_gradient_and_sets_spec_values(oracle):
    # SPEC.md:184-206 and Eq. proj-gradient
    l = np.array([0.0, 0.0, 0.0, 0.0, 1.0])
    u = np.array([5.0, 5.0, 5.0, 5.0, 1.0])
    x = np.array([0.0, 0.0, 5.0, 2.0, 1.0])
    g = np.array([3.0, -2.0, -2.0, 4.0, 9.0])
    assert np.array_equal(oracle.proj_grad(x, g, l, u), [0.0, -2.0, 0.0, 4.0, 0.0])
    act, bnd, na, nb = oracle.sets(x, g, l, u)
    assert list(act) == [True, True, True, False, True]
    assert list(bnd) == [True, False, True, False, True]
    # B subset of A; ||grad_Omega q|| <= ||grad q||
    rng_x = P.gaussian(2, 60, 200)
    l = -np.abs(P.gaussian(2, 61, 200)); u = np.abs(P.gaussian(2, 62, 200))
    xx = oracle.project(l, u, rng_x)
    gg = P.gaussian(2, 63, 200)
    act, bnd, na, nb = oracle.sets(xx, gg, l, u)
    assert np.all(~bnd | act)
    pg = oracle.proj_grad(xx, gg, l, u)
    assert np.linalg.norm(pg) <= np.linalg.norm(gg)
    # grad_Omega q == 0 exactly on binding variables, == g on free ones
    assert np.all(pg[bnd] == 0.0) and np.array_equal(pg[~act], gg[~act])


def test_objective_values_and_gradient_fd(oracle):
    # SPEC.md:156-158, 166-168
    A = csr_of(oracle, np.eye(2))
    assert oracle.objective(A, [0.0, 0.0], 0.0, [3.0, 4.0]) == 12.5
    assert oracle.objective(A, [1.0, 2.0], 1.25, [0.0, 0.0]) == 1.25
    Ad, b, l, u = P.random_dense_qp(10, seed=11, bounds="inf")
    A = csr_of(oracle, Ad)
    x = P.gaussian(11, 70, 10)
    g = oracle.gradient(A, b, x)
    h = 1e-6
    for i in range(10):
        e = np.zeros(10); e[i] = h
        fd = (oracle.objective(A, b, 0.0, x + e) - oracle.objective(A, b, 0.0, x - e)) / (2 * h)
        assert abs(fd - g[i]) <= 1e-5


# ---------------------------------------------------------------- Cauchy step and searches
def test_cauchy_alpha(oracle):
    # A=I -> 1; A=2I -> 1/2; random = golden-section argmin of q(y - a d)
    for s, ref in [(1.0, 1.0), (2.0, 0.5)]:
        A = csr_of(oracle, s * np.eye(4))
        y = np.zeros(4); g = np.array([1.0, -2, 3, 0.5])
        a, st = oracle.cauchy_alpha(A, y, g, np.full(4, -np.inf), np.full(4, np.inf))
        assert st == 0 and a == ref
    Ad, b, l, u = P.random_dense_qp(5, seed=5, bounds="mixed")
    A = csr_of(oracle, Ad)
    y = oracle.project(l, u, P.gaussian(5, 80, 5))
    g = Ad @ y - b
    d = oracle.proj_grad(y, g, l, u)
    a, st = oracle.cauchy_alpha(A, y, g, l, u)
    ref = B.golden_section(lambda t: B.q_dense(Ad, b, 0, y - t * d), 0.0, 10.0)
    assert st == 0 and abs(a - ref) <= 1e-6


def test_cauchy_not_spd(oracle):
    A = csr_of(oracle, -np.eye(3))
    a, st = oracle.cauchy_alpha(A, np.zeros(3), np.ones(3), np.full(3, -np.inf), np.full(3, np.inf))
    assert st == oracle.ENOTSPD


def test_projected_search_gp_1d_and_inequality(oracle):
    # q = 1/2 x^2, y=1, no bounds -> alpha0=1, y+=0 accepted at h=0
    A = csr_of(oracle, np.eye(1))
    y = np.array([1.0]); g = np.array([1.0])
    a0, _ = oracle.cauchy_alpha(A, y, g, [-np.inf], [np.inf])
    h, yn, delta, alpha = oracle.projected_search(A, y, g, -g, [-np.inf], [np.inf], a0)
    assert (a0, h, yn[0], alpha) == (1.0, 0, 0.0, 1.0) and delta == -0.5
    # clipped 2-D step: the accepted alpha satisfies Eq. gplsstop re-evaluated with q values,
    # and the previous trial (alpha*2) does not
    Ad = np.array([[4.0, 1.0], [1.0, 3.0]]); b = np.array([1.0, 8.0])
    A = csr_of(oracle, Ad)
    l = np.array([0.0, 0.0]); u = np.array([0.1, 0.3])
    y = np.array([0.05, 0.0]); g = Ad @ y - b
    for base in [1.0, 40.0]:
        h, yn, delta, alpha = oracle.projected_search(A, y, g, -g, l, u, base)
        assert h >= 0
        lhs = B.q_dense(Ad, b, 0, yn)
        rhs = B.q_dense(Ad, b, 0, y) + 0.1 * g @ (yn - y)
        assert lhs <= rhs + 1e-15 and abs(delta - (lhs - B.q_dense(Ad, b, 0, y))) <= 1e-14
        if h > 0:
            prev = np.clip(y - 2 * alpha * g, l, u)
            assert B.q_dense(Ad, b, 0, prev) > B.q_dense(Ad, b, 0, y) + 0.1 * g @ (prev - y)


def test_projected_search_zero_direction(oracle):
    # d = 0 -> x+ = x with alpha = 1
    A = csr_of(oracle, np.eye(3))
    x = np.array([0.5, 0.0, 1.0]); g = np.array([0.3, 1.0, -1.0])
    h, xn, delta, alpha = oracle.projected_search(A, x, g, np.zeros(3), np.zeros(3), np.ones(3), 1.0)
    assert h == 0 and alpha == 1.0 and np.array_equal(xn, x) and delta == 0.0


# ---------------------------------------------------------------- CG
def test_cg_identity_one_iteration(oracle):
    # A_k = I -> one iteration, w = -r_k
    A = csr_of(oracle, np.eye(5))
    r = np.array([1.0, -2, 3, 4, -5])
    it, w, decs = oracle.cg(A, np.ones(5, np.uint8), r, 0.05)
    assert it == 1 and np.allclose(w, -r, atol=1e-15)


def test_cg_dense_solve_and_finite_termination(oracle):
    # 10x10 SPD with eta2=1e-12 -> dense solve; terminates within m
    for seed, m in [(1, 10), (2, 17), (3, 30)]:
        Ad, b, l, u = P.random_dense_qp(m, seed=seed, bounds="inf")
        A = csr_of(oracle, Ad)
        r = P.gaussian(seed, 90, m)
        ref = np.linalg.solve(Ad, -r)
        it, w, decs = oracle.cg(A, np.ones(m, np.uint8), r, 1e-12)
        assert 1 <= it <= m and np.max(np.abs(w - ref)) <= 1e-6
        # progress test effectively off: finite termination within m steps
        it, w, decs = oracle.cg(A, np.ones(m, np.uint8), r, 1e-300)
        assert 1 <= it <= m
        assert np.max(np.abs(w - ref)) <= 1e-12 * np.linalg.cond(Ad) * np.max(np.abs(ref))
        # the decreases 1/2 alpha rho'rho sum to q_k(0) - q_k(w) (reading R17)
        qk = 0.5 * w @ Ad @ w + r @ w
        assert abs(decs.sum() + qk) <= 1e-10 * abs(qk)
        assert np.all(decs >= 0)


def test_cg_masked_matches_reduced_dense(oracle):
    Ad, b, l, u = P.random_dense_qp(12, seed=4, bounds="inf")
    A = csr_of(oracle, Ad)
    fr = (P.uniform(4, 91, 12) < 0.5).astype(np.uint8)
    F = np.flatnonzero(fr)
    r = P.gaussian(4, 92, 12)
    it, w, decs = oracle.cg(A, fr, r, 1e-12)
    ref = np.linalg.solve(Ad[np.ix_(F, F)], -r[F])
    assert np.all(w[fr == 0] == 0.0)
    assert np.max(np.abs(w[F] - ref)) <= 1e-9


def test_cg_progress_stop_rule(oracle):
    # Eq. cgstop1: the returned step is the first j>=2 whose decrease <= eta2 * max earlier
    m = 40
    Ad = np.diag(np.linspace(1.0, 1e3, m)) + 0.0
    A = csr_of(oracle, Ad)
    r = np.ones(m)
    it, w, decs = oracle.cg(A, np.ones(m, np.uint8), r, 0.05)
    assert it >= 2
    for j in range(2, it):
        assert decs[j - 1] > 0.05 * decs[:j - 1].max()
    assert decs[it - 1] <= 0.05 * decs[:it - 1].max() or it == m


# ---------------------------------------------------------------- point-Jacobi PCG
def test_jacobi_inverse_is_inverse_diagonal(oracle):
    Ad, b, l, u = P.random_dense_qp(9, seed=12, bounds="inf")
    d = oracle.jacobi_inverse(csr_of(oracle, Ad))
    assert np.array_equal(d, 1.0 / np.diag(Ad))


def test_pcg_exact_for_diagonal_operator(oracle):
    # M = diag(A) = A for a diagonal A: z_0 = A^-1 rho_0, one step solves (w = -A^-1 r)
    dvals = np.linspace(0.5, 40.0, 11)
    Ad = np.diag(dvals)
    A = csr_of(oracle, Ad)
    r = P.gaussian(13, 1, 11)
    it, w, decs = oracle.pcg(A, np.ones(11, np.uint8), r, oracle.jacobi_inverse(A), 0.05)
    assert it == 1
    assert np.max(np.abs(w + r / dvals)) <= 1e-15 * np.max(np.abs(r / dvals))
    # plain CG needs more than one step on the same system
    assert oracle.cg(A, np.ones(11, np.uint8), r, 1e-300)[0] > 1


def test_pcg_dense_solve_decreases_and_termination(oracle):
    for seed, m in [(21, 10), (22, 17), (23, 30)]:
        Ad, b, l, u = P.random_dense_qp(m, seed=seed, bounds="inf")
        # badly scaled rows/cols: the case a diagonal preconditioner is for
        sc = np.exp(2.0 * P.uniform(seed, 70, m))
        Ad = (Ad * sc[:, None]) * sc[None, :]
        A = csr_of(oracle, Ad)
        r = P.gaussian(seed, 71, m)
        ref = np.linalg.solve(Ad, -r)
        it, w, decs = oracle.pcg(A, np.ones(m, np.uint8), r, oracle.jacobi_inverse(A), 1e-300)
        assert 1 <= it <= m                                   # finite termination
        assert np.max(np.abs(w - ref)) <= 1e-10 * np.linalg.cond(Ad) * np.max(np.abs(ref))
        qk = 0.5 * w @ Ad @ w + r @ w
        assert abs(decs.sum() + qk) <= 1e-10 * abs(qk)        # 1/2 alpha rho'z sums to -q_k(w)
        assert np.all(decs >= 0)


def test_pcg_masked_matches_reduced_dense(oracle):
    Ad, b, l, u = P.random_dense_qp(14, seed=24, bounds="inf")
    A = csr_of(oracle, Ad)
    fr = (P.uniform(24, 91, 14) < 0.6).astype(np.uint8)
    F = np.flatnonzero(fr)
    r = P.gaussian(24, 92, 14)
    it, w, decs = oracle.pcg(A, fr, r, oracle.jacobi_inverse(A), 1e-300)     # progress test off
    assert it <= len(F) and np.all(w[fr == 0] == 0.0)
    assert np.max(np.abs(w[F] - np.linalg.solve(Ad[np.ix_(F, F)], -r[F]))) <= 1e-12


def test_gpcg_pcg_same_minimiser(oracle):
    # x* is unique: the preconditioner changes the path, not the answer
    for sd in range(40):
        n = 2 + sd % 7
        Ad, b, l, u = P.random_dense_qp(n, seed=4000 + sd, bounds="mixed")
        A = csr_of(oracle, Ad)
        rc, x, st = oracle.solve(A, b, l, u, 0.0, P.gaussian(sd, 1, n), -1e-12,
                                 params=oracle.default_params(precond=1))
        assert rc == 0 and np.max(np.abs(x - B.enum_solve(Ad, b, l, u))) <= 1e-6
    prob = P.c0()
    rc0, x0, st0 = oracle.solve_problem(prob, tol=-1e-12)
    rc1, x1, st1 = oracle.solve_problem(prob, tol=-1e-12, params=oracle.default_params(precond=1))
    assert rc0 == rc1 == 0 and np.max(np.abs(x0 - x1)) <= 1e-7
    assert abs(st0["q"] - st1["q"]) <= 1e-10 * abs(st0["q"])


# ---------------------------------------------------------------- whole GPCG
def test_gpcg_two_var(oracle):
    g = GOLD["two_var_solution"]
    A = csr_of(oracle, np.array(g["A"], float))
    b = -np.array(g["b_paper"], float)
    rc, x, st = oracle.solve(A, b, g["l"], g["u"], 0.0, [1.0, 1.0], 1e-12)
    assert rc == 0 and np.array_equal(x, g["x_star"]) and st["pg_norm"] <= 1e-10


@pytest.mark.parametrize("seed", range(50))
def test_gpcg_infinite_bounds_is_cholesky(oracle, seed):
    # no bounds -> A x* = b; dense Cholesky solve
    n = 2 + (seed * 7) % 49
    Ad, b, l, u = P.random_dense_qp(n, seed=100 + seed, bounds="inf")
    A = csr_of(oracle, Ad)
    rc, x, st = oracle.solve(A, b, l, u, 0.0, np.zeros(n), -1e-12)
    L = np.linalg.cholesky(Ad)
    ref = np.linalg.solve(L.T, np.linalg.solve(L, b))
    assert rc == 0 and np.max(np.abs(x - ref)) <= 1e-6


def test_gpcg_enumeration_200(oracle):
    # 200 seeded instances n in 2..8 vs 3^n enumeration within 1e-6
    for s in range(200):
        n = 2 + s % 7
        Ad, b, l, u = P.random_dense_qp(n, seed=1000 + s, bounds="mixed")
        A = csr_of(oracle, Ad)
        x0 = P.gaussian(1000 + s, 95, n)
        rc, x, st = oracle.solve(A, b, l, u, 0.0, x0, -1e-12)
        ref = B.enum_solve(Ad, b, l, u)
        assert rc == 0, (s, rc)
        assert np.max(np.abs(x - ref)) <= 1e-6, (s, x, ref)


def test_gpcg_enumeration_n12(oracle):
    for s in range(3):
        Ad, b, l, u = P.random_dense_qp(12, seed=5000 + s, bounds="mixed")
        rc, x, st = oracle.solve(csr_of(oracle, Ad), b, l, u, 0.0, np.zeros(12), -1e-12)
        assert rc == 0 and np.max(np.abs(x - B.enum_solve(Ad, b, l, u))) <= 1e-6


def test_gpcg_journal_bearing_c0_kkt_and_exact_face(oracle):
    # KKT, B = A at the solution, and x equals the exact
    # solution of its own face (dense solve of the free block) within the a-posteriori bound
    p = P.c0()
    A = oracle.problem_csr(p)
    rc, x, st = oracle.solve_problem(p, tol=-1e-12)
    assert rc == 0
    g = oracle.gradient(A, p.b, x)
    assert np.all(x >= p.l) and np.all(x <= p.u)
    assert B.kkt_residual(x, g, p.l, p.u) <= 1e-12 * np.linalg.norm(p.b) * 10
    act, bnd, na, nb = oracle.sets(x, g, p.l, p.u)
    assert na == nb
    Ad = A.todense()
    F = np.flatnonzero(~act)
    xf = np.linalg.solve(Ad[np.ix_(F, F)], p.b[F])       # active values are 0
    assert np.max(np.abs(xf - x[F])) <= 1e-9
    # the exact face solution is itself a KKT point (so it is x*)
    xs = np.zeros(p.n); xs[F] = xf
    gs = Ad @ xs - p.b
    assert np.all(xf > 0) and np.all(gs[act] >= -1e-14)


def test_gpcg_eps0_zero_solution(oracle):
    # eps = 0 -> w_l = 0 -> x* = 0
    p = P.journal_bearing(20, 20, eps=0.0)
    rc, x, st = oracle.solve_problem(p, tol=1e-12)
    assert rc == 0 and np.all(x == 0.0)


def test_gpcg_spec_trivial_one_point(oracle):
    # nx=ny=1, eps=0, b_dom=pi -> A=[4]
    p = P.journal_bearing(1, 1, eps=0.0, bdom=math.pi)
    A = oracle.problem_csr(p)
    assert np.allclose(A.todense(), [[4.0]], atol=1e-15)


@pytest.mark.parametrize("eps,key,rkey", [(0.1, "free_fraction_eps0.1", "free_fraction_range_200_eps0.1"),
                                          (0.9, "free_fraction_eps0.9", "free_fraction_range_200_eps0.9")])
def test_free_fraction_matches_paper(oracle, eps, key, rkey):
    # ~68% free at eps=0.1, 54% at eps=0.9; SPEC.md:654 ranges at 200x200
    p = P.journal_bearing(200, 200, eps=eps)
    rc, x, st = oracle.solve_problem(p)
    assert rc == 0
    frac = st["n_free"] / p.n
    lo, hi = GOLD[rkey]["value"]
    assert lo <= frac <= hi
    assert abs(frac - GOLD[key]["value"]) <= 0.02
    assert st["n_active_nonbinding"] == 0


def test_gpcg_error_cases(oracle):
    A = csr_of(oracle, np.eye(2))
    rc, x, st = oracle.solve(A, [1.0, 1.0], [1.0, 0.0], [0.0, 1.0], 0.0, [0.0, 0.0], 1e-8)
    assert rc == oracle.EINVAL
    A = csr_of(oracle, np.array([[1.0, 2.0], [2.0, 1.0]]))      # indefinite
    rc, x, st = oracle.solve(A, [1.0, -1.0], [-1e3, -1e3], [1e3, 1e3], 0.0, [0.0, 0.0], 1e-8)
    assert rc in (oracle.ENOTSPD,)


def test_gpcg_fixed_variables(oracle):
    # l_i = u_i allowed; fixed variables are always active, grad_Omega component 0 (R16)
    Ad, b, l, u = P.random_dense_qp(6, seed=77, bounds="mixed")
    l[2] = u[2] = 0.25
    rc, x, st = oracle.solve(csr_of(oracle, Ad), b, l, u, 0.0, np.zeros(6), -1e-12)
    assert rc == 0 and x[2] == 0.25
    assert np.max(np.abs(x - B.enum_solve(Ad, b, l, u))) <= 1e-6


# ---------------------------------------------------------------- generator facts
def test_generator_closed_forms():
    # ||b||_2 = 0.1 hx hy sqrt(ny (nx+1)/2); w_q(0; 0.1) = 1.331
    for nx in (50, 1600):
        p = P.journal_bearing(nx, 1, 0.1) if nx > 100 else P.c0()
        hx, hy = p.meta["hx"], p.meta["hy"]
        ny = p.ny
        ref = 0.1 * hx * hy * math.sqrt(ny * (nx + 1) / 2.0)
        assert abs(np.linalg.norm(p.b) - ref) <= 1e-12 * ref
    assert abs((1 + 0.1 * math.cos(0.0)) ** 3 - GOLD["wq_xi0_eps0.1"]["value"]) < 1e-15


def test_generator_mmatrix_and_nnz(oracle):
    # off-diagonals <= 0, diagonally dominant, mean nnz/row in [4.9, 5.0] at 100^2
    p = P.journal_bearing(100, 100, 0.1)
    A = oracle.problem_csr(p)
    lo, hi = GOLD["nnz_per_row_100"]["value"]
    assert lo <= A.val.size / p.n <= hi
    rows = np.repeat(np.arange(p.n), np.diff(A.rp))
    diag = rows == A.ci
    assert np.all(A.val[~diag] <= 0)
    off = np.bincount(rows[~diag], weights=np.abs(A.val[~diag]), minlength=p.n)
    assert np.all(A.val[diag] >= off * (1 - 1e-14))


def test_generator_c4_small_structure():
    p = P.c4_family(m=6)
    n = 216
    assert p.row_ptr[-1] == 7 * n - 6 * 36
    rows = np.repeat(np.arange(n), np.diff(p.row_ptr))
    A = np.zeros((n, n)); A[rows, p.col] = p.val
    assert np.allclose(A, A.T, atol=0)
    assert np.allclose(A.sum(axis=1), 1e-3, atol=1e-12)       # diag = sum of incident w + 1e-3
    assert np.all(np.diff(p.col.astype(np.int64))[np.diff(rows) == 0] > 0)   # sorted columns


def test_rng_determinism():
    a = P.uniform(1, 5, 10)
    b = P.uniform(1, 5, 5, offset=5)
    assert np.array_equal(a[5:], b)
    z = P.gaussian(4, 14, 100000)
    assert abs(z.mean()) < 0.02 and abs(z.std() - 1) < 0.02


# ---------------------------------------------------------------- 3-D 7-point stencil (NEXT-2)
def test_stencil3d_assembly_matches_edge_list_csr(oracle):
    # two independent routes to C4's matrix: face assembly (oracle) vs the generator's edge-list CSR
    for m in (4, 7, 12):
        A = oracle.problem_csr(P.c4_family(m=m))
        S = oracle.problem_csr(P.c4_stencil_family(m=m))
        assert np.array_equal(A.rp, S.rp) and np.array_equal(A.ci, S.ci)
        assert np.max(np.abs(A.val - S.val)) <= 1e-14 * np.max(np.abs(A.val))


def test_stencil3d_constant_coefficient_eigenpairs(oracle):
    # unit faces incl. Dirichlet boundary faces: A = Laplacian_x + _y + _z with the textbook
    # eigenvectors sin(p pi i/(n+1)) ... and eigenvalues sum_d 4 sin^2(p_d pi / (2(n_d+1)))
    nx, ny, nz = 5, 4, 3
    A = oracle.stencil3d_to_csr(nx, ny, nz, np.ones((nx + 1) * ny * nz), np.ones(nx * (ny + 1) * nz),
                                np.ones(nx * ny * (nz + 1)))
    i, j, k = np.meshgrid(np.arange(1, nx + 1), np.arange(1, ny + 1), np.arange(1, nz + 1), indexing="ij")
    for p, q, r in [(1, 1, 1), (2, 3, 1), (5, 4, 3)]:
        v = (np.sin(p * np.pi * i / (nx + 1)) * np.sin(q * np.pi * j / (ny + 1)) *
             np.sin(r * np.pi * k / (nz + 1))).transpose(2, 1, 0).reshape(-1)     # v = i + nx (j + ny k)
        lam = sum(4 * np.sin(a * np.pi / (2 * (m + 1))) ** 2 for a, m in [(p, nx), (q, ny), (r, nz)])
        assert np.max(np.abs(oracle.spmv(A, v) - lam * v)) <= 1e-13
    D = A.todense()
    assert np.array_equal(D, D.T)


# ---------------------------------------------------------------- block-Jacobi ILU(0) (NEXT-3)
def _grid_csr(oracle, nx, ny, seed):
    wx = 0.5 + P.uniform(seed, 1, ny * (nx + 1))
    wy = 0.5 + P.uniform(seed, 2, (ny + 1) * nx)
    return oracle.stencil2d_to_csr(nx, ny, wx, nx + 1, wy, nx, 0.01 * P.uniform(seed, 3, nx * ny))


def test_bjilu_reproduces_a_on_its_pattern(oracle):
    # ILU(0): M = (D+L) D^-1 (D+U) equals A on A's pattern inside every block (and the
    # inter-block entries are dropped); checked densely on a 7 x 6 grid with 3 x 4 tiles
    nx, ny, tx, ty = 7, 6, 3, 4
    A = _grid_csr(oracle, nx, ny, 31)
    n = nx * ny
    free = (P.uniform(31, 9, n) < 0.8).astype(np.uint8)
    d = oracle.bjilu_factor(A, free, nx, tx, ty)
    Ad = A.todense()
    F = np.flatnonzero(free)
    tile = lambda v: ((v % nx) // tx, (v // nx) // ty)   # noqa: E731
    L = np.zeros((n, n)); U = np.zeros((n, n)); D = np.diag(np.where(free == 1, d, 1.0))
    for v in F:
        for u in F:
            if u != v and Ad[v, u] != 0 and tile(u) == tile(v):
                (L if u < v else U)[v, u] = Ad[v, u]
    M = (D + L) @ np.linalg.inv(D) @ (D + U)
    for v in F:
        for u in F:
            if Ad[v, u] != 0 and tile(u) == tile(v):
                assert abs(M[v, u] - Ad[v, u]) <= 1e-12 * abs(Ad[v, v])
    # and M^-1 r through the oracle's triangular solves equals the dense solve on F
    r = P.gaussian(31, 10, n)
    z = oracle.bjilu_apply(A, free, nx, tx, ty, d, r)
    MF = M[np.ix_(F, F)]
    assert np.max(np.abs(z[F] - np.linalg.solve(MF, r[F]))) <= 1e-12 * np.max(np.abs(z[F]))
    assert np.all(z[free == 0] == 0.0)


def test_bjilu_exact_on_a_single_row(oracle):
    # one grid row inside one tile: A_F tridiagonal, ILU(0) = exact LDL' -> one PCG step solves
    nx = 24
    A = _grid_csr(oracle, nx, 1, 32)
    free = np.ones(nx, np.uint8)
    r = P.gaussian(32, 11, nx)
    it, w, decs = oracle.pcg_bjilu(A, free, r, nx, 32, 32, 1e-300)
    assert it == 1
    assert np.max(np.abs(w + np.linalg.solve(A.todense(), r))) <= 1e-12 * np.max(np.abs(w))


def test_bjilu_1x1_tiles_is_jacobi(oracle):
    nx, ny = 9, 7
    A = _grid_csr(oracle, nx, ny, 33)
    free = (P.uniform(33, 9, nx * ny) < 0.7).astype(np.uint8)
    r = P.gaussian(33, 12, nx * ny)
    it_b, w_b, dec_b = oracle.pcg_bjilu(A, free, r, nx, 1, 1, 1e-300)
    it_j, w_j, dec_j = oracle.pcg(A, free, r, oracle.jacobi_inverse(A), 1e-300)
    assert it_b == it_j
    assert np.max(np.abs(w_b - w_j)) <= 1e-12 * np.max(np.abs(w_j))


def test_gpcg_bjilu_same_minimiser_fewer_cg_iterations(oracle):
    prob = P.c0()
    base = oracle.solve_problem(prob, tol=-1e-12, params=oracle.default_params(precond=1))
    ilu = oracle.solve_problem(prob, tol=-1e-12, params=oracle.default_params(
        precond=2, grid_nx=50, grid_ny=50, tile_x=32, tile_y=32))
    assert base[0] == ilu[0] == 0
    assert np.max(np.abs(base[1] - ilu[1])) <= 1e-7
    assert ilu[2]["cg_iters"] < base[2]["cg_iters"]      # fewer CG iterations than Jacobi
