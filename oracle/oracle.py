"""ctypes front of the plain-C GPCG oracle (oracle/gpcg_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product path
(paper_cs_0101018_b200/).  Marshalling only -- all arithmetic is in the C file,
which cites the paper passage each routine follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gpcg_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
LIB_OMP = os.path.join(HERE, "liboracle_omp.so")

OK, NOT_CONVERGED, EINVAL, ENOMEM, ENOTSPD, ESEARCH = 0, 1, -1, -2, -5, -6


def build(force: bool = False, omp: bool = False) -> str:
    """Compile liboracle.so (gcc -O2 -ffp-contract=off; single thread) or, omp=True,
    liboracle_omp.so: the same source with -fopenmp (row / elementwise loops threaded, every
    sum serial: bitwise-identical results; SURVEY.md 8(d)'s all-core baseline)."""
    out = LIB_OMP if omp else LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(SRC):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c99",
                               "-D_POSIX_C_SOURCE=199309L", "-fPIC", "-shared"] +
                              (["-fopenmp"] if omp else []) + ["-o", tmp, SRC, "-lm"])
        os.replace(tmp, out)
    return out


class Params(C.Structure):
    _fields_ = [("mu", C.c_double), ("eta1", C.c_double), ("eta2", C.c_double),
                ("eta2_shrink", C.c_double), ("eta2_floor", C.c_double),
                ("gp_cap", C.c_int64), ("refine_cap", C.c_int64),
                ("max_halvings", C.c_int64), ("cg_cap", C.c_int64),
                ("time_budget_s", C.c_double), ("precond", C.c_int64),
                ("grid_nx", C.c_int64), ("grid_ny", C.c_int64), ("tile_x", C.c_int64), ("tile_y", C.c_int64),
                ("trace", C.c_void_p), ("trace_cap", C.c_int64), ("ilu_level", C.c_int64)]


class Stats(C.Structure):
    _fields_ = [("outer_iters", C.c_int64), ("gp_iters", C.c_int64), ("cg_iters", C.c_int64),
                ("cg_calls", C.c_int64), ("refinements", C.c_int64), ("full_spmvs", C.c_int64),
                ("n_free", C.c_int64), ("n_active", C.c_int64), ("n_active_nonbinding", C.c_int64),
                ("pg_norm", C.c_double), ("q", C.c_double), ("g0_norm", C.c_double),
                ("tau", C.c_double), ("seconds", C.c_double), ("status", C.c_int64),
                ("trace_len", C.c_int64)]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


TREC = 6   # doubles per control-path trace record (ORA_TREC in gpcg_oracle.c)


_lib = None
_lib_omp = None


def lib():
    global _lib
    if _lib is None:
        # ORACLE_LIB: load another build of the same source (mutation testing of the pins,
        # scripts/oracle_mutants.py); default: the in-tree build
        _lib = _bind(C.CDLL(os.environ.get("ORACLE_LIB") or build()))
    return _lib


def lib_omp():
    """The OpenMP build (all host cores unless OMP_NUM_THREADS says otherwise)."""
    global _lib_omp
    if _lib_omp is None:
        _lib_omp = _bind(C.CDLL(build(omp=True)))
    return _lib_omp


def _bind(L):
    if True:
        P = C.c_void_p
        i64 = C.c_int64
        L.ora_stencil2d_nnz.restype = i64
        L.ora_stencil2d_nnz.argtypes = [i64, i64]
        L.ora_stencil2d_to_csr.restype = C.c_int
        L.ora_stencil2d_to_csr.argtypes = [i64, i64, P, i64, P, i64, P, P, P, P]
        L.ora_stencil3d_nnz.restype = i64
        L.ora_stencil3d_nnz.argtypes = [i64, i64, i64]
        L.ora_stencil3d_to_csr.restype = C.c_int
        L.ora_stencil3d_to_csr.argtypes = [i64, i64, i64, P, P, P, P, P, P, P]
        L.ora_spmv.restype = None
        L.ora_spmv.argtypes = [i64, P, P, P, P, P]
        L.ora_spmv_masked.restype = None
        L.ora_spmv_masked.argtypes = [i64, P, P, P, P, P, P]
        L.ora_project.restype = None
        L.ora_project.argtypes = [i64, P, P, P, P]
        L.ora_proj_grad.restype = None
        L.ora_proj_grad.argtypes = [i64, P, P, P, P, P]
        L.ora_sets.restype = None
        L.ora_sets.argtypes = [i64, P, P, P, P, P, P, P, P]
        L.ora_objective.restype = C.c_double
        L.ora_objective.argtypes = [i64, P, P, P, P, C.c_double, P]
        L.ora_cauchy_alpha.restype = C.c_double
        L.ora_cauchy_alpha.argtypes = [i64, P, P, P, P, P, P, P, P, P]
        L.ora_projected_search.restype = i64
        L.ora_projected_search.argtypes = [i64, P, P, P, P, P, P, P, P, C.c_double, C.c_double,
                                           i64, P, P, P, P]
        L.ora_cg.restype = i64
        L.ora_cg.argtypes = [i64, P, P, P, P, P, C.c_double, i64, P, P, P, C.c_double]
        L.ora_pcg.restype = i64
        L.ora_pcg.argtypes = [i64, P, P, P, P, P, P, C.c_double, i64, P, P, P, C.c_double]
        L.ora_pcg_bjilu.restype = i64
        L.ora_pcg_bjilu.argtypes = [i64, P, P, P, P, P, i64, i64, i64, C.c_double, i64, P, P, P, P]
        L.ora_pcg_bjiluk.restype = i64
        L.ora_pcg_bjiluk.argtypes = [i64, P, P, P, P, P, i64, i64, i64, i64, C.c_double, i64, P, P, P, P]
        L.ora_bjiluk_export.restype = i64
        L.ora_bjiluk_export.argtypes = [i64, P, P, P, P, i64, i64, i64, i64, P, P, P, P, i64]
        L.ora_bjilu_factor.restype = None
        L.ora_bjilu_factor.argtypes = [i64, P, P, P, P, i64, i64, i64, P]
        L.ora_bjilu_apply.restype = None
        L.ora_bjilu_apply.argtypes = [i64, P, P, P, P, i64, i64, i64, P, P, P, P]
        L.ora_jacobi_inverse.restype = None
        L.ora_jacobi_inverse.argtypes = [i64, P, P, P, P]
        L.ora_params_default.restype = None
        L.ora_params_default.argtypes = [P]
        L.ora_gpcg_solve.restype = C.c_int
        L.ora_gpcg_solve.argtypes = [i64, P, P, P, P, P, P, C.c_double, P, C.c_double, i64,
                                     P, P, P]
    return L


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class CSR:
    n: int
    rp: np.ndarray
    ci: np.ndarray
    val: np.ndarray

    def todense(self):
        A = np.zeros((self.n, self.n))
        for i in range(self.n):
            for k in range(self.rp[i], self.rp[i + 1]):
                A[i, self.ci[k]] += self.val[k]
        return A


def stencil2d_to_csr(nx, ny, wx, wx_ld, wy, wy_ld, shift=None) -> CSR:
    L = lib()
    n = nx * ny
    nnz = L.ora_stencil2d_nnz(nx, ny)
    rp = np.zeros(n + 1, dtype=np.int64)
    ci = np.zeros(nnz, dtype=np.int32)
    va = np.zeros(nnz, dtype=np.float64)
    wx = _f64(wx); wy = _f64(wy)
    sh = _f64(shift) if shift is not None else None
    rc = L.ora_stencil2d_to_csr(nx, ny, _p(wx), wx_ld, _p(wy), wy_ld, _p(sh), _p(rp), _p(ci), _p(va))
    if rc != 0:
        raise ValueError("ora_stencil2d_to_csr failed")
    return CSR(n, rp, ci, va)


def stencil3d_to_csr(nx, ny, nz, wx, wy, wz, shift=None) -> CSR:
    L = lib()
    n = nx * ny * nz
    nnz = L.ora_stencil3d_nnz(nx, ny, nz)
    rp = np.zeros(n + 1, dtype=np.int64)
    ci = np.zeros(nnz, dtype=np.int32)
    va = np.zeros(nnz, dtype=np.float64)
    wx = _f64(wx); wy = _f64(wy); wz = _f64(wz)
    sh = _f64(shift) if shift is not None else None
    rc = L.ora_stencil3d_to_csr(nx, ny, nz, _p(wx), _p(wy), _p(wz), _p(sh), _p(rp), _p(ci), _p(va))
    if rc != 0:
        raise ValueError("ora_stencil3d_to_csr failed")
    return CSR(n, rp, ci, va)


def problem_csr(prob) -> CSR:
    """The oracle's own CSR of a problems.Problem (assembled here for stencils)."""
    if prob.kind == "stencil2d":
        return stencil2d_to_csr(prob.nx, prob.ny, prob.wx, prob.wx_ld, prob.wy, prob.wy_ld, prob.shift)
    if prob.kind == "stencil3d":
        return stencil3d_to_csr(prob.nx, prob.ny, prob.nz, prob.wx, prob.wy, prob.wz, prob.shift)
    return CSR(prob.n, np.ascontiguousarray(prob.row_ptr, dtype=np.int64),
               np.ascontiguousarray(prob.col, dtype=np.int32), _f64(prob.val))


def spmv(A: CSR, x):
    x = _f64(x)
    y = np.empty(A.n)
    lib().ora_spmv(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(x), _p(y))
    return y


def spmv_masked(A: CSR, free, x):
    x = _f64(x)
    fr = np.ascontiguousarray(free, dtype=np.uint8)
    y = np.empty(A.n)
    lib().ora_spmv_masked(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(fr), _p(x), _p(y))
    return y


def project(l, u, x):
    l, u, x = _f64(l), _f64(u), _f64(x)
    px = np.empty_like(x)
    lib().ora_project(x.size, _p(l), _p(u), _p(x), _p(px))
    return px


def proj_grad(x, g, l, u):
    x, g, l, u = _f64(x), _f64(g), _f64(l), _f64(u)
    pg = np.empty_like(x)
    lib().ora_proj_grad(x.size, _p(x), _p(g), _p(l), _p(u), _p(pg))
    return pg


def sets(x, g, l, u):
    """(active mask, binding mask, |A|, |B|)"""
    x, g, l, u = _f64(x), _f64(g), _f64(l), _f64(u)
    n = x.size
    act = np.zeros(n, np.uint8)
    bnd = np.zeros(n, np.uint8)
    na = C.c_int64(); nb = C.c_int64()
    lib().ora_sets(n, _p(x), _p(g), _p(l), _p(u), _p(act), _p(bnd), C.byref(na), C.byref(nb))
    return act.astype(bool), bnd.astype(bool), na.value, nb.value


def objective(A: CSR, b, c, x):
    b, x = _f64(b), _f64(x)
    return lib().ora_objective(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(b), c, _p(x))


def gradient(A: CSR, b, x):
    return spmv(A, x) - _f64(b)


def cauchy_alpha(A: CSR, y, g, l, u):
    y, g, l, u = _f64(y), _f64(g), _f64(l), _f64(u)
    work = np.empty(2 * A.n)
    st = C.c_int()
    a = lib().ora_cauchy_alpha(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(y), _p(g), _p(l), _p(u),
                               _p(work), C.byref(st))
    return a, st.value


def projected_search(A: CSR, y, g, direction, l, u, alpha_base, mu=0.1, max_halvings=50):
    """-> (h, ynew, delta, alpha); h = -1 when no trial is accepted."""
    y, g, d, l, u = _f64(y), _f64(g), _f64(direction), _f64(l), _f64(u)
    ynew = np.empty_like(y)
    work = np.empty(2 * A.n)
    delta = C.c_double(); alpha = C.c_double()
    h = lib().ora_projected_search(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(y), _p(g), _p(d),
                                   _p(l), _p(u), alpha_base, mu, max_halvings, _p(ynew),
                                   _p(work), C.byref(delta), C.byref(alpha))
    return h, ynew, delta.value, alpha.value


def cg(A: CSR, free, r, eta2, cap=0, omp=False):
    """Textbook CG on A_F w = -r.  -> (iterations or error code, w, decreases).
    omp: run the OpenMP build (same results bitwise)."""
    fr = np.ascontiguousarray(free, dtype=np.uint8)
    r = _f64(r)
    m = int(fr.sum())
    cap = cap if cap > 0 else m
    w = np.empty(A.n)
    work = np.empty(4 * A.n)
    decs = np.zeros(max(cap, 1))
    it = (lib_omp() if omp else lib()).ora_cg(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(fr), _p(r), eta2, cap,
                      _p(w), _p(work), _p(decs), 0.0)
    return it, w, decs[:max(it, 0)]


def jacobi_inverse(A: CSR):
    """1 / diag(A) (the point-Jacobi preconditioner, oracle routine)."""
    d = np.empty(A.n)
    lib().ora_jacobi_inverse(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(d))
    return d


def bjilu_factor(A: CSR, free, nx, tx, ty):
    """Block-Jacobi ILU(0) pivots on tiles tx x ty of an nx-wide grid (oracle routine)."""
    fr = np.ascontiguousarray(free, dtype=np.uint8)
    d = np.empty(A.n)
    lib().ora_bjilu_factor(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(fr), nx, tx, ty, _p(d))
    return d


def bjilu_apply(A: CSR, free, nx, tx, ty, d, r):
    fr = np.ascontiguousarray(free, dtype=np.uint8)
    r = _f64(r)
    t = np.empty(A.n)
    z = np.empty(A.n)
    lib().ora_bjilu_apply(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(fr), nx, tx, ty, _p(d), _p(r), _p(t), _p(z))
    return z


def pcg_bjilu(A: CSR, free, r, nx, tx, ty, eta2, cap=0):
    """Block-Jacobi ILU(0) PCG on A_F w = -r. -> (iterations, w, decreases)."""
    fr = np.ascontiguousarray(free, dtype=np.uint8)
    r = _f64(r)
    m = int(fr.sum())
    cap = cap if cap > 0 else m
    w = np.empty(A.n)
    work = np.empty(4 * A.n)
    scratch = np.empty(2 * A.n)
    decs = np.zeros(max(cap, 1))
    it = lib().ora_pcg_bjilu(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(fr), _p(r), nx, tx, ty, eta2, cap,
                             _p(w), _p(work), _p(scratch), _p(decs))
    return it, w, decs[:max(it, 0)]


def bjiluk_factor(A: CSR, free, nx, tx, ty, level):
    """Block-Jacobi ILU(level) factor (oracle routine) -> (rows, cols, levels, values): the L
    (col < row, unit diagonal implied) and U (col >= row) entries of every tile."""
    fr = np.ascontiguousarray(free, dtype=np.uint8)
    L = lib()
    m = L.ora_bjiluk_export(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(fr), nx, tx, ty, level,
                            None, None, None, None, 0)
    rows = np.empty(m, np.int64); cols = np.empty(m, np.int64); levs = np.empty(m, np.int64)
    vals = np.empty(m)
    L.ora_bjiluk_export(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(fr), nx, tx, ty, level,
                        _p(rows), _p(cols), _p(levs), _p(vals), m)
    return rows, cols, levs, vals


def pcg_bjiluk(A: CSR, free, r, nx, tx, ty, level, eta2, cap=0):
    """Block-Jacobi ILU(level) PCG on A_F w = -r. -> (iterations, w, decreases)."""
    fr = np.ascontiguousarray(free, dtype=np.uint8)
    r = _f64(r)
    m = int(fr.sum())
    cap = cap if cap > 0 else m
    w = np.empty(A.n)
    work = np.empty(4 * A.n)
    scratch = np.empty(A.n)
    decs = np.zeros(max(cap, 1))
    it = lib().ora_pcg_bjiluk(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(fr), _p(r), nx, tx, ty, level, eta2, cap,
                              _p(w), _p(work), _p(scratch), _p(decs))
    return it, w, decs[:max(it, 0)]


def pcg(A: CSR, free, r, dinv, eta2, cap=0):
    """Point-Jacobi PCG on A_F w = -r (M^-1 = diag(dinv) on F). -> (iterations, w, decreases)."""
    fr = np.ascontiguousarray(free, dtype=np.uint8)
    r = _f64(r)
    dinv = _f64(dinv)
    m = int(fr.sum())
    cap = cap if cap > 0 else m
    w = np.empty(A.n)
    work = np.empty(4 * A.n)
    decs = np.zeros(max(cap, 1))
    it = lib().ora_pcg(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(fr), _p(r), _p(dinv), eta2, cap,
                       _p(w), _p(work), _p(decs), 0.0)
    return it, w, decs[:max(it, 0)]


def default_params(**kw) -> Params:
    p = Params()
    lib().ora_params_default(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def solve(A: CSR, b, l, u, c, x0, tol, max_it=500, params: Params = None):
    """Algorithm GPCG (oracle).  -> (status, x, stats dict)."""
    b, l, u, x0 = _f64(b), _f64(l), _f64(u), _f64(x0)
    params = params or default_params()
    x = np.empty(A.n)
    st = Stats()
    rc = lib().ora_gpcg_solve(A.n, _p(A.rp), _p(A.ci), _p(A.val), _p(b), _p(l), _p(u), c,
                              _p(x0), tol, max_it, C.byref(params), _p(x), C.byref(st))
    return rc, x, st.asdict()


def solve_problem(prob, tol=None, max_it=500, params: Params = None):
    A = problem_csr(prob)
    return solve(A, prob.b, prob.l, prob.u, prob.c, prob.x0,
                 prob.tol if tol is None else tol, max_it, params)


def solve_trace(A: CSR, b, l, u, c, x0, tol, max_it=500, params: Params = None, cap=200000):
    """Algorithm GPCG with the control-path trace (see gpcg_oracle.c, trace_put).
    -> (status, x, stats dict, trace as an (records, 6) array)."""
    params = params or default_params()
    buf = np.zeros(cap * TREC)
    params.trace = buf.ctypes.data
    params.trace_cap = cap
    try:
        rc, x, st = solve(A, b, l, u, c, x0, tol, max_it, params)
    finally:
        params.trace = None
        params.trace_cap = 0
    if st["trace_len"] > cap:
        raise RuntimeError("oracle trace truncated")
    return rc, x, st, buf[: st["trace_len"] * TREC].reshape(-1, TREC).copy()
