"""Seeded synthetic inputs for the GPCG hot path (configs C0-C4 of BASELINE.json).

This module is the ONE piece shared by the CUDA path and the CPU oracle.  It
only *draws problems* (face weights, CSR entries, b, l, u, x0, tol); it holds
none of the method's arithmetic (no matvec, no projection, no CG, no search).

Problem statement (Eq. def-quadratic): minimise
q(x) = 1/2 x^T A x - b^T x + c subject to l <= x <= u, with A SPD.  Note the
ABI sign convention b_abi = -b_paper (reading R1): the paper writes
+b^T x while BASELINE.json's north_star writes -b^T x.

Journal-bearing problem (Sec. 5): q(v) = int 1/2 w_q |grad v|^2
- w_l v over D=(0,2pi)x(0,2b), w_q=(1+eps cos xi1)^3, w_l = eps sin xi1, l=0,
u=+inf.  Discretised here by BASELINE.json configs[0]'s finite-difference
operator (reading R2): interior grid points xi1=i*hx (i=1..nx), xi2=j*hy
(j=1..ny), hx=2pi/(nx+1), hy=2b/(ny+1), b=10 (reading R3); x-faces weigh
(hy/hx) w_q((i-1/2)hx), y-faces weigh (hx/hy) w_q(i*hx); Dirichlet boundary.

Stencil face-array convention (identical to include/gpcg.h):
  * grid point (i, j), 0-based, linear index v = i + nx*j (i fastest);
  * wx: x-face weights, nx+1 per grid row; face k (0..nx) joins points k-1
    and k of that row (faces 0 and nx touch the Dirichlet boundary).
    wx_ld == 0 -> one row broadcast to every grid row, else row j at wx[j*wx_ld];
  * wy: y-face weights, ny+1 face rows of nx each; face row f (0..ny) joins
    grid rows f-1 and f.  wy_ld == 0 -> broadcast, else face row f at wy[f*wy_ld];
  * A v = sum over faces of weight * (difference across the face), i.e.
    (Ap)_v = (sum of the 4 incident face weights + shift_v) p_v - sum w_f p_nbr.

Counter RNG: splitmix64; key(seed, stream) = splitmix64(seed*2^32
+ stream); element i draws splitmix64(key + i); U = (u64 >> 11) * 2^-53;
Gaussian by Box-Muller with streams a and a+100.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


# --------------------------------------------------------------------------
# counter-based RNG
# --------------------------------------------------------------------------
def _splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)).astype(np.uint64)
        return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int) -> np.uint64:
    v = np.array([((seed << 32) + stream) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    return _splitmix64(v)[0]


def uniform(seed: int, stream: int, count: int, offset: int = 0) -> np.ndarray:
    """U[0,1) draws for element indices offset..offset+count-1 of (seed, stream)."""
    k = _key(seed, stream)
    idx = np.arange(offset, offset + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = _splitmix64((idx + k).astype(np.uint64))
    return (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def gaussian(seed: int, stream: int, count: int, offset: int = 0) -> np.ndarray:
    """N(0,1) via Box-Muller from streams `stream` and `stream+100`."""
    ua = uniform(seed, stream, count, offset)
    ub = uniform(seed, stream + 100, count, offset)
    return np.sqrt(-2.0 * np.log1p(-ua)) * np.cos(2.0 * math.pi * ub)


# --------------------------------------------------------------------------
# problem container
# --------------------------------------------------------------------------
@dataclass
class Problem:
    """One bound-constrained QP instance as handed to gpcg_create_* and the oracle."""
    name: str
    kind: str                      # "stencil2d" | "csr"
    n: int
    b: np.ndarray
    l: np.ndarray
    u: np.ndarray
    x0: np.ndarray
    tol: float                     # <0: relative to ||g(P[x0])||_2 (BASELINE.json convention)
    c: float = 0.0
    # stencil2d
    nx: int = 0
    ny: int = 0
    nz: int = 0
    wz: Optional[np.ndarray] = None          # stencil3d z-face weights
    wx: Optional[np.ndarray] = None
    wx_ld: int = 0
    wy: Optional[np.ndarray] = None
    wy_ld: int = 0
    shift: Optional[np.ndarray] = None
    # csr (int64 row_ptr, int32 col, fp64 val; both triangles stored)
    row_ptr: Optional[np.ndarray] = None
    col: Optional[np.ndarray] = None
    val: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)

    def input_bytes(self) -> int:
        """Bytes of all host arrays a create+solve call uploads (operator, b, l, u, x0)."""
        arrs = [self.b, self.l, self.u, self.x0, self.wx, self.wy, self.wz, self.shift,
                self.row_ptr, self.col, self.val]
        return int(sum(a.nbytes for a in arrs if a is not None))


# --------------------------------------------------------------------------
# journal bearing (C0 / C2 / C3 family)
# --------------------------------------------------------------------------
def journal_bearing_faces(nx: int, ny: int, eps: float, bdom: float = 10.0):
    """Row-broadcast face weights and b of the FD journal-bearing operator.

    x-face k (0..nx) sits at xi1=(k+1/2)hx  (1-based "(i-1/2)hx", i=k+1);
    y-faces of point column i sit at xi1=(i+1)hx (0-based i).
    b_{ij} = eps*sin(xi1)*hx*hy in the ABI sign (= -b_paper, reading R1).
    """
    hx = 2.0 * math.pi / (nx + 1)
    hy = 2.0 * bdom / (ny + 1)
    k = np.arange(nx + 1, dtype=np.float64)
    wq_x = (1.0 + eps * np.cos((k + 0.5) * hx)) ** 3
    wx = (hy / hx) * wq_x
    i = np.arange(nx, dtype=np.float64)
    xi1 = (i + 1.0) * hx
    wy = (hx / hy) * (1.0 + eps * np.cos(xi1)) ** 3
    brow = eps * np.sin(xi1) * hx * hy
    return wx, wy, brow, hx, hy


def journal_bearing(nx: int, ny: int, eps: float = 0.1, bdom: float = 10.0,
                    name: str = "jb", tol: float = -1e-8) -> Problem:
    """The paper's benchmark under readings R1-R3: l=0, u=+inf, x0=l=0."""
    wx, wy, brow, hx, hy = journal_bearing_faces(nx, ny, eps, bdom)
    n = nx * ny
    b = np.tile(brow, ny)
    l = np.zeros(n)
    u = np.full(n, np.inf)
    x0 = np.zeros(n)
    return Problem(name=name, kind="stencil2d", n=n, b=b, l=l, u=u, x0=x0, tol=tol,
                   nx=nx, ny=ny, wx=wx, wx_ld=0, wy=wy, wy_ld=0,
                   meta=dict(eps=eps, bdom=bdom, hx=hx, hy=hy, family="journal_bearing"))


def c0() -> Problem:
    """BASELINE.json configs[0]: 50x50, eps=0.1, l=0, u=inf, x0=0, tol 1e-8*||g(x0)||."""
    return journal_bearing(50, 50, 0.1, name="C0")


def c2() -> Problem:
    """BASELINE.json configs[2]: 1600x1600 (n=2.56M, the paper's largest size PAPER.md:784-786)."""
    return journal_bearing(1600, 1600, 0.1, name="C2")


# --------------------------------------------------------------------------
# C1: noisy faces, Gaussian b, two-sided piecewise-constant obstacles
# --------------------------------------------------------------------------
# obstacle amplitude `a`, frozen by scripts/calibrate.py (oracle solves only)
C1_OBSTACLE_A = 0.0001926


def c1_family(nx: int = 400, ny: int = 400, a: float = None, seed: int = 1,
              tiles: int = 16, name: str = "C1") -> Problem:
    """BASELINE.json configs[1] (recipe SURVEY.md 8(d), reading R7)."""
    a = C1_OBSTACLE_A if a is None else a
    wxr, wyr, _, hx, hy = journal_bearing_faces(nx, ny, 0.1)
    n = nx * ny
    eta_x = 0.9 + 0.2 * uniform(seed, 1, ny * (nx + 1))
    eta_y = 0.9 + 0.2 * uniform(seed, 2, (ny + 1) * nx)
    wx = (np.tile(wxr, ny) * eta_x).astype(np.float64)
    wy = (np.tile(wyr, ny + 1) * eta_y).astype(np.float64)
    b = hx * hy * gaussian(seed, 3, n)
    # piecewise-constant obstacles on tiles x tiles blocks
    ti = (np.arange(nx) * tiles) // nx
    tj = (np.arange(ny) * tiles) // ny
    tid = (tj[:, None] * tiles + ti[None, :]).ravel()
    lt = -a * (0.5 + uniform(seed, 5, tiles * tiles))
    ut = +a * (0.5 + uniform(seed, 6, tiles * tiles))
    l = lt[tid].copy()
    u = ut[tid].copy()
    x0 = l + uniform(seed, 7, n) * (u - l)
    return Problem(name=name, kind="stencil2d", n=n, b=b, l=l, u=u, x0=x0, tol=-1e-8,
                   nx=nx, ny=ny, wx=wx, wx_ld=nx + 1, wy=wy, wy_ld=nx,
                   meta=dict(a=a, seed=seed, family="c1"))


def c1() -> Problem:
    return c1_family()


# --------------------------------------------------------------------------
# C3: journal bearing with mesh-independent two-sided obstacles
# --------------------------------------------------------------------------
C3_X = 0.133            # max of the l=0 solution
C3_OBSTACLE_C = 0.01045  # frozen by scripts/calibrate.py c3 1600 (oracle solves only): 0.500 active at 1600^2
                         # (round 1 froze 0.01514 at 400^2, which leaves only 43 % active at 8000^2)


def c3_family(nx: int = 8000, ny: int = 8000, c: float = None, seed: int = 3,
              tiles: int = 32, name: str = "C3") -> Problem:
    """BASELINE.json configs[3]: obstacles on a tiles x tiles tiling of the continuous domain."""
    c = C3_OBSTACLE_C if c is None else c
    p = journal_bearing(nx, ny, 0.1, name=name)
    hx, hy = p.meta["hx"], p.meta["hy"]
    xi1 = (np.arange(nx) + 1.0) * hx
    xi2 = (np.arange(ny) + 1.0) * hy
    ti = np.minimum((tiles * xi1 / (2.0 * math.pi)).astype(np.int64), tiles - 1)
    tj = np.minimum((tiles * xi2 / 20.0).astype(np.int64), tiles - 1)
    lt = -0.25 * c * C3_X * uniform(seed, 5, tiles * tiles)
    ut = c * C3_X * (0.5 + uniform(seed, 6, tiles * tiles))
    l = np.empty(p.n)
    u = np.empty(p.n)
    for j in range(ny):                      # row by row keeps peak memory at 64M x 8B per array
        tid = tj[j] * tiles + ti
        l[j * nx:(j + 1) * nx] = lt[tid]
        u[j * nx:(j + 1) * nx] = ut[tid]
    p.l, p.u = l, u
    p.x0 = np.zeros(p.n)                    # = mid(l,u,0) since l<=0<=u
    p.meta.update(c=c, seed=seed, family="c3")
    return p


def c3() -> Problem:
    return c3_family()


# --------------------------------------------------------------------------
# C4: 3D 7-point lognormal-weight CSR
# --------------------------------------------------------------------------
def c4_family(m: int = 256, seed: int = 4, box: float = 0.01, name: str = "C4") -> Problem:
    """BASELINE.json configs[4]: m^3 grid, natural order v=i+m(j+m k), general CSR.

    Edge (v, v+stride) for in-grid neighbours only; w_e = exp(0.5 Z_e);
    A_uv = -w_e; A_vv = sum incident w_e + 1e-3.  Edge ids: x-edge at the
    lower endpoint v (valid when i<m-1) drawn at element v of streams 11/111,
    y-edges streams 12/112, z-edges streams 13/113.
    """
    n = m ** 3
    v = np.arange(n, dtype=np.int64)
    i = v % m
    j = (v // m) % m
    k = v // (m * m)
    wx = np.exp(0.5 * gaussian(seed, 11, n)); wx[i == m - 1] = 0.0
    wy = np.exp(0.5 * gaussian(seed, 12, n)); wy[j == m - 1] = 0.0
    wz = np.exp(0.5 * gaussian(seed, 13, n)); wz[k == m - 1] = 0.0
    del i, j, k
    # incident weights: upper edge at v, lower edge at v - stride
    diag = wx + wy + wz + 1e-3
    diag[1:] += wx[:-1]
    diag[m:] += wy[:-m]
    diag[m * m:] += wz[:-m * m]
    # slots in ascending column order: -z, -y, -x, diag, +x, +y, +z
    strides = [-m * m, -m, -1, 0, 1, m, m * m]
    vals = np.zeros((n, 7))
    vals[m * m:, 0] = -wz[:-m * m]
    vals[m:, 1] = -wy[:-m]
    vals[1:, 2] = -wx[:-1]
    vals[:, 3] = diag
    vals[:, 4] = -wx
    vals[:, 5] = -wy
    vals[:, 6] = -wz
    del wx, wy, wz, diag
    present = vals != 0.0
    present[:, 3] = True
    cnt = present.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=row_ptr[1:])
    cols = (v[:, None] + np.array(strides, dtype=np.int64)[None, :])
    col = cols[present].astype(np.int32)
    val = vals[present]
    del cols, vals, present
    b = gaussian(seed, 14, n)
    l = np.full(n, -box)
    u = np.full(n, box)
    x0 = np.zeros(n)
    return Problem(name=name, kind="csr", n=n, b=b, l=l, u=u, x0=x0, tol=-1e-8,
                   row_ptr=row_ptr, col=col, val=val,
                   meta=dict(m=m, seed=seed, family="c4"))


def c4_stencil_family(m: int = 256, seed: int = 4, box: float = 0.01, name: str = "C4s") -> Problem:
    """The C4 problem as a 3-D 7-point face-weight stencil (kind "stencil3d", SURVEY.md
    8(f) NEXT-2): the same edge weights (streams 11/12/13), b (14) and bounds as
    c4_family, laid out as face arrays (include/gpcg.h, gpcg_create_stencil3d); there
    are no boundary faces and the 1e-3 of the diagonal is the shift."""
    n = m ** 3
    ex = np.exp(0.5 * gaussian(seed, 11, n)).reshape(m, m, m)     # [k, j, i]: edge (i,j,k)-(i+1,j,k)
    ey = np.exp(0.5 * gaussian(seed, 12, n)).reshape(m, m, m)
    ez = np.exp(0.5 * gaussian(seed, 13, n)).reshape(m, m, m)
    wx = np.zeros((m, m, m + 1)); wx[:, :, 1:m] = ex[:, :, :m - 1]   # face i' joins i'-1, i'
    wy = np.zeros((m, m + 1, m)); wy[:, 1:m, :] = ey[:, :m - 1, :]
    wz = np.zeros((m + 1, m, m)); wz[1:m, :, :] = ez[:m - 1, :, :]
    del ex, ey, ez
    b = gaussian(seed, 14, n)
    return Problem(name=name, kind="stencil3d", n=n, b=b, l=np.full(n, -box), u=np.full(n, box),
                   x0=np.zeros(n), tol=-1e-8, nx=m, ny=m, nz=m, wx=wx.reshape(-1), wy=wy.reshape(-1),
                   wz=wz.reshape(-1), shift=np.full(n, 1e-3), meta=dict(m=m, seed=seed, family="c4"))


def c4() -> Problem:
    return c4_family()


# --------------------------------------------------------------------------
# small random instances for enumeration / direct-solve pins
# --------------------------------------------------------------------------
def random_dense_qp(n: int, seed: int, bounds: str = "mixed"):
    """Small dense SPD instance (A, b, l, u) for n<=12 brute-force pins.

    A = M M^T + n I (M uniform in [-1,1]); b ~ N(0,1)*2; bounds per element:
    'inf' -> (-inf, inf); 'mixed' -> each side finite with prob 1/2.
    """
    M = 2.0 * uniform(seed, 21, n * n).reshape(n, n) - 1.0
    A = M @ M.T + n * np.eye(n)
    b = 2.0 * gaussian(seed, 22, n)
    if bounds == "inf":
        l = np.full(n, -np.inf)
        u = np.full(n, np.inf)
    else:
        lo = -uniform(seed, 23, n)
        hi = uniform(seed, 24, n)
        fl = uniform(seed, 25, n) < 0.5
        fu = uniform(seed, 26, n) < 0.5
        l = np.where(fl, lo, -np.inf)
        u = np.where(fu, hi, np.inf)
    return A, b, l, u


def dense_to_csr(A: np.ndarray):
    """CSR (int64 row_ptr, int32 col, fp64 val) of a dense matrix, both triangles, zeros dropped."""
    n = A.shape[0]
    nz = A != 0.0
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(nz.sum(axis=1), out=row_ptr[1:])
    rows, cols = np.nonzero(nz)
    return row_ptr, cols.astype(np.int32), A[rows, cols].astype(np.float64)


def csr_problem(A: np.ndarray, b, l, u, x0=None, tol=-1e-10, name="dense") -> Problem:
    rp, ci, va = dense_to_csr(A)
    n = A.shape[0]
    x0 = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64)
    return Problem(name=name, kind="csr", n=n, b=np.asarray(b, float), l=np.asarray(l, float),
                   u=np.asarray(u, float), x0=x0, tol=tol, row_ptr=rp, col=ci, val=va)


CONFIGS = {"C0": c0, "C1": c1, "C2": c2, "C3": c3, "C4": c4}


def get(name: str) -> Problem:
    """A config by name; family members as e.g. C3_1600 (1600^2 member of C3's family),
    C4_128 (128^3 member of C4's)."""
    if name in CONFIGS:
        return CONFIGS[name]()
    fam, _, size = name.partition("_")
    if fam == "C3" and size:
        return c3_family(int(size), int(size))
    if fam == "C4" and size:
        return c4_family(m=int(size))
    if fam == "C4s":
        return c4_stencil_family(m=int(size) if size else 256)
    raise KeyError(name)
