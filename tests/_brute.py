"""Independent brute-force references used to PIN the oracle (tests only).

Nothing here calls the oracle or the CUDA path; each routine is a plain
definition written out with numpy/scipy so that a mistake in the oracle (a
dropped term, a wrong sign, a transposed operand) shows up as a mismatch.
"""
import itertools
import math

import numpy as np


def dense_stencil_grad_form(nx, ny, wx, wx_ld, wy, wy_ld, shift=None):
    """A = Gx' Wx Gx + Gy' Wy Gy (+ diag(shift)), the discrete div(w grad) form.

    Gx maps grid values to x-face differences (one row per x-face, Dirichlet
    zeros outside), Wx the diagonal of face weights; same for y.  This is a
    different construction from the 5-point stencil assembly in the oracle.
    """
    n = nx * ny
    rows_x = []
    wxs = []
    for j in range(ny):
        for k in range(nx + 1):
            r = np.zeros(n)
            if k - 1 >= 0:
                r[(k - 1) + nx * j] = -1.0
            if k <= nx - 1:
                r[k + nx * j] = 1.0
            rows_x.append(r)
            wxs.append(wx[j * wx_ld + k])
    rows_y = []
    wys = []
    for f in range(ny + 1):
        for i in range(nx):
            r = np.zeros(n)
            if f - 1 >= 0:
                r[i + nx * (f - 1)] = -1.0
            if f <= ny - 1:
                r[i + nx * f] = 1.0
            rows_y.append(r)
            wys.append(wy[f * wy_ld + i])
    Gx = np.array(rows_x)
    Gy = np.array(rows_y)
    A = Gx.T @ np.diag(wxs) @ Gx + Gy.T @ np.diag(wys) @ Gy
    if shift is not None:
        A = A + np.diag(shift)
    return A


def q_dense(A, b, c, x):
    return 0.5 * x @ A @ x - b @ x + c


def enum_solve(A, b, l, u, tol=1e-9):
    """Unique KKT point of min 1/2x'Ax - b'x on [l,u] by 3^n enumeration.

    Each variable is at its lower bound, at its upper bound, or free; the free
    block solves A_FF x_F = b_F - A_F,fix x_fix; accept the assignment whose
    point is feasible and whose gradient signs satisfy the Kuhn-Tucker conditions.
    """
    n = len(b)
    choices = []
    for i in range(n):
        c = ["F"]
        if np.isfinite(l[i]):
            c.append("L")
        if np.isfinite(u[i]):
            c.append("U")
        choices.append(c)
    sols = []
    for assign in itertools.product(*choices):
        x = np.zeros(n)
        F = [i for i in range(n) if assign[i] == "F"]
        X = [i for i in range(n) if assign[i] != "F"]
        for i in X:
            x[i] = l[i] if assign[i] == "L" else u[i]
        if F:
            rhs = b[F] - A[np.ix_(F, X)] @ x[X] if X else b[F]
            x[F] = np.linalg.solve(A[np.ix_(F, F)], rhs)
        if np.any(x < l - tol) or np.any(x > u + tol):
            continue
        g = A @ x - b
        ok = True
        for i in range(n):
            if assign[i] == "L" and g[i] < -tol:
                ok = False
            elif assign[i] == "U" and g[i] > tol:
                ok = False
            elif assign[i] == "F" and (x[i] < l[i] - tol or x[i] > u[i] + tol):
                ok = False
        if ok:
            sols.append(x)
            return x
    raise AssertionError("no KKT point found")


def kkt_residual(x, g, l, u):
    """max violation of the Kuhn-Tucker conditions with x feasible."""
    viol = 0.0
    for xi, gi, li, ui in zip(x, g, l, u):
        if xi == li and xi == ui:
            continue
        if xi == li:
            viol = max(viol, max(-gi, 0.0))
        elif xi == ui:
            viol = max(viol, max(gi, 0.0))
        else:
            viol = max(viol, abs(gi))
    return viol


def golden_section(f, a, b, tol=1e-12, it=300):
    gr = (math.sqrt(5.0) - 1.0) / 2.0
    c = b - gr * (b - a)
    d = a + gr * (b - a)
    for _ in range(it):
        if f(c) < f(d):
            b = d
        else:
            a = c
        c = b - gr * (b - a)
        d = a + gr * (b - a)
        if abs(b - a) < tol:
            break
    return 0.5 * (a + b)


def laplacian_eigpair(nx, ny, hx, hy, p, q):
    """Exact eigenpair of the constant-coefficient FD operator with weights hy/hx, hx/hy."""
    i = np.arange(1, nx + 1)
    j = np.arange(1, ny + 1)
    v = np.outer(np.sin(q * math.pi * j / (ny + 1)), np.sin(p * math.pi * i / (nx + 1))).ravel()
    lam = (hy / hx) * 4.0 * math.sin(p * math.pi / (2 * (nx + 1))) ** 2 + \
          (hx / hy) * 4.0 * math.sin(q * math.pi / (2 * (ny + 1))) ** 2
    return v, lam


# ---------------------------------------------------------------------------------------------
# Algorithm GPCG written out densely (numpy), independently of oracle/gpcg_oracle.c, to pin the
# oracle's CONTROL PATH: the GP-phase stop tests (Eqs. pgstop1 / pgstop2), the
# CG progress test (Eq. cgstop1) and the eta2 refinement of Eq. cgstop3.
# The CG runs on the extracted free block A_FF (the paper's own MatExtractSubmatrix route,
# P:689-700), not on the masked full-length operator the oracle uses; every q difference uses
# the exact expansion <g,s> + 1/2 <s,As> (R17).  Readings R9-R13, R26 as in DESIGN.md.
# Emits the same record layout as the oracle's trace: (kind, k, i1, i2, v1, v2).
# ---------------------------------------------------------------------------------------------
def _active(x, l, u):
    return (x == l) | (x == u)


def _pgrad(x, g, l, u):
    d = g.copy()
    at_l, at_u = x == l, x == u
    d[at_l & (g > 0)] = 0.0
    d[at_u & (g < 0)] = 0.0
    d[at_l & at_u] = 0.0
    return d


def _search(A, y, g, direction, l, u, alpha_base, mu, max_halvings):
    """first alpha = alpha_base 2^-h with q(P[y + alpha dir]) <= q(y) + mu <g, P[..] - y>"""
    for h in range(max_halvings):
        alpha = alpha_base * 0.5 ** h
        yt = np.minimum(np.maximum(y + alpha * direction, l), u)
        s = yt - y
        gs = float(g @ s)
        dq = gs + 0.5 * float(s @ (A @ s))
        if dq <= mu * gs:
            return h, yt, dq, alpha
    return -1, y, 0.0, 0.0


def gpcg_dense_trace(A, b, l, u, x0, tau, mu=0.1, eta1=0.1, eta2_0=0.05, eta2_shrink=0.1,
                     eta2_floor=1e-12, gp_cap=100000, refine_cap=30, max_halvings=50, max_it=500):
    """-> (status, x, trace list of (kind, k, i1, i2, v1, v2)); status 0 converged, 1 max_it."""
    A = np.asarray(A, dtype=float)
    x = np.minimum(np.maximum(np.asarray(x0, float), l), u)
    tr = []
    g = A @ x - b
    if np.linalg.norm(_pgrad(x, g, l, u)) <= tau:
        return 0, x, tr
    for k in range(max_it):
        # gradient projection phase
        j, hist, a_first = 0, [], 0.0
        while True:
            d = _pgrad(x, g, l, u)
            if np.linalg.norm(d) <= tau:
                tr.append((2, k, j, 0, max(hist, default=0.0), a_first))
                return 0, x, tr
            alpha0 = float(d @ d) / float(d @ (A @ d))           # Eq. bqpls
            h, y, dq, alpha = _search(A, x, g, -g, l, u, alpha0, mu, max_halvings)
            assert h >= 0
            same = bool(np.all(_active(y, l, u) == _active(x, l, u)))   # Eq. pgstop1
            x = y
            g = A @ x - b
            j += 1
            if j == 1:
                a_first = alpha0
            dec = -dq
            tr.append((1, k, j, h, dec, alpha))
            if same:
                reason = 1
            elif j >= 2 and dec <= eta1 * max(hist):               # Eq. pgstop2
                reason = 2
            elif j >= gp_cap:
                reason = 3
            else:
                reason = 0
            hist.append(dec)
            if reason:
                tr.append((2, k, j, reason, max(hist), a_first))
                break
        if np.linalg.norm(_pgrad(x, g, l, u)) <= tau:
            return 0, x, tr
        # CG phase with eta2 refinement
        eta2 = eta2_0
        for rep in range(refine_cap):
            F = ~_active(x, l, u)
            m = int(F.sum())
            if m == 0:
                break
            AF = A[np.ix_(F, F)]
            r = g[F]
            wF = np.zeros(m)
            rho = -r
            p = rho.copy()
            rr = float(rho @ rho)
            r0 = np.sqrt(rr)
            decs = []
            it = 0
            while True:
                it += 1
                a = AF @ p
                alpha = rr / float(p @ a)
                wF = wF + alpha * p
                dec = 0.5 * alpha * rr
                rho = rho - alpha * a
                rr_new = float(rho @ rho)
                stop = (it >= 2 and dec <= eta2 * max(decs)) or np.sqrt(rr_new) <= 1e-14 * (1.0 + r0) or it >= m
                decs.append(dec)
                if stop:
                    break
                p = rho + (rr_new / rr) * p
                rr = rr_new
            tr.append((3, k, rep, it, eta2, m))
            w = np.zeros_like(x)
            w[F] = wF
            h, y, dq, alpha = _search(A, x, g, w, l, u, 1.0, mu, max_halvings)   # Eq. cglsstop2
            assert h >= 0
            x = y
            g = A @ x - b
            act = _active(x, l, u)
            binding = ((x == l) & (g >= 0)) | ((x == u) & (g <= 0))
            nonbinding = int(np.sum(act & ~binding))
            tr.append((4, k, rep, h, -dq, nonbinding))
            if np.linalg.norm(_pgrad(x, g, l, u)) <= tau:
                return 0, x, tr
            if nonbinding != 0:                                      # Eq. cgstop3 fails
                break
            eta2 = max(eta2 * eta2_shrink, eta2_floor)
    return 1, x, tr
