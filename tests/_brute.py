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
