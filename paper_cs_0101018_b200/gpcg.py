"""Thin ctypes binding of libgpcg.so (include/gpcg.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this
module only converts numpy arrays / torch tensors into pointers.  There is no
CPU fallback: if libgpcg.so is missing or no CUDA device is present, the calls
raise.  Arrays may live on the host (numpy, CPU tensors) or on the handle's
device (CUDA tensors); the library detects which.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GPCG_LIB") or os.path.join(_HERE, "libgpcg.so")   # GPCG_LIB: A/B builds

OK, NOT_CONVERGED, EINVAL, ENOMEM, ECUDA, ENCCL, ENOTSPD, ESEARCH, ESTATE = 0, 1, -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "OK", 1: "NOT_CONVERGED", -1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENCCL",
                -5: "ENOTSPD", -6: "ESEARCH", -7: "ESTATE"}

# every symbol include/gpcg.h declares (checked by tests/test_abi.py)
SYMBOLS = ["gpcg_params_default", "gpcg_create_stencil2d", "gpcg_create_stencil2d_dist",
           "gpcg_create_stencil3d", "gpcg_create_stencil3d_dist", "gpcg_create_csr",
           "gpcg_create_csr_dist", "gpcg_set_params", "gpcg_solve", "gpcg_hessvec", "gpcg_free_count",
           "gpcg_hessvec_free", "gpcg_project",
           "gpcg_objective", "gpcg_size", "gpcg_destroy", "gpcg_last_error", "gpcg_partition_rows",
           "gpcg_nccl_unique_id"]


class Params(C.Structure):
    _fields_ = [("mu", C.c_double), ("eta1", C.c_double), ("eta2", C.c_double),
                ("eta2_shrink", C.c_double), ("eta2_floor", C.c_double),
                ("gp_cap", C.c_int64), ("refine_cap", C.c_int64), ("max_halvings", C.c_int64),
                ("cg_cap", C.c_int64), ("search_k", C.c_int32), ("cg_chunk", C.c_int32),
                ("gp_chunk", C.c_int32), ("precond", C.c_int32), ("cg_mode", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("outer_iters", C.c_int64), ("gp_iters", C.c_int64), ("cg_iters", C.c_int64),
                ("cg_calls", C.c_int64), ("refinements", C.c_int64), ("full_spmvs", C.c_int64),
                ("n_free", C.c_int64), ("n_active", C.c_int64), ("n_active_nonbinding", C.c_int64),
                ("pg_norm", C.c_double), ("q", C.c_double), ("g0_norm", C.c_double), ("tau", C.c_double),
                ("t_total_ms", C.c_double), ("t_cg_ms", C.c_double), ("t_gp_ms", C.c_double),
                ("status", C.c_int32), ("kernel_launches", C.c_int32),
                ("cg_iters_timed", C.c_int64), ("cg_free_iters_timed", C.c_int64),
                ("t_cg_timed_ms", C.c_double), ("t_extract_ms", C.c_double),
                ("gp_spec_rejected", C.c_int64)]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Dist(C.Structure):
    """gpcg_dist: the rank's row slab (include/gpcg.h)."""
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("nccl_id", C.c_void_p),
                ("row_begin", C.c_int64), ("row_end", C.c_int64), ("local_slabs", C.c_int32)]


class GpcgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def load():
    """Load libgpcg.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_cs_0101018_b200._build` "
                          "or __graft_entry__.build() (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int, C.c_double
    L.gpcg_params_default.restype = Params
    L.gpcg_params_default.argtypes = []
    L.gpcg_create_stencil2d.restype = i32
    L.gpcg_create_stencil2d.argtypes = [C.POINTER(P), P, i64, i64, P, i64, P, i64, P, P, P, P, dbl]
    L.gpcg_create_csr.restype = i32
    L.gpcg_create_csr.argtypes = [C.POINTER(P), P, i64, P, P, P, P, P, P, dbl]
    L.gpcg_create_stencil2d_dist.restype = i32
    L.gpcg_create_stencil2d_dist.argtypes = [C.POINTER(P), C.POINTER(Dist), P, i64, i64, P, i64, P, i64, P, P, P,
                                             P, dbl]
    L.gpcg_create_stencil3d.restype = i32
    L.gpcg_create_stencil3d.argtypes = [C.POINTER(P), P, i64, i64, i64, P, P, P, P, P, P, P, dbl]
    L.gpcg_create_stencil3d_dist.restype = i32
    L.gpcg_create_stencil3d_dist.argtypes = [C.POINTER(P), C.POINTER(Dist), P, i64, i64, i64, P, P, P, P, P, P, P,
                                             dbl]
    L.gpcg_create_csr_dist.restype = i32
    L.gpcg_create_csr_dist.argtypes = [C.POINTER(P), C.POINTER(Dist), P, i64, P, P, P, P, P, P, dbl]
    L.gpcg_partition_rows.restype = None
    L.gpcg_partition_rows.argtypes = [i64, C.c_int32, C.c_int32, C.POINTER(i64), C.POINTER(i64)]
    L.gpcg_nccl_unique_id.restype = i32
    L.gpcg_nccl_unique_id.argtypes = [P]
    L.gpcg_set_params.restype = i32
    L.gpcg_set_params.argtypes = [P, C.POINTER(Params)]
    L.gpcg_solve.restype = i32
    L.gpcg_solve.argtypes = [P, P, dbl, i64, P, C.POINTER(Stats)]
    L.gpcg_hessvec.restype = i32
    L.gpcg_hessvec.argtypes = [P, P, P, i32]
    L.gpcg_free_count.restype = i64
    L.gpcg_free_count.argtypes = [P]
    L.gpcg_hessvec_free.restype = i32
    L.gpcg_hessvec_free.argtypes = [P, P, P]
    L.gpcg_project.restype = i32
    L.gpcg_project.argtypes = [P, P, P, C.POINTER(dbl), C.POINTER(i64), C.POINTER(i64)]
    L.gpcg_objective.restype = i32
    L.gpcg_objective.argtypes = [P, P, C.POINTER(dbl)]
    L.gpcg_size.restype = i64
    L.gpcg_size.argtypes = [P]
    L.gpcg_destroy.restype = None
    L.gpcg_destroy.argtypes = [P]
    L.gpcg_last_error.restype = C.c_char_p
    L.gpcg_last_error.argtypes = []
    _lib = L
    return L


def last_error() -> str:
    return load().gpcg_last_error().decode()


def _check(rc, allow=(OK,)):
    if rc not in allow:
        raise GpcgError(rc, last_error())
    return rc


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a, dtype):
    """(pointer, keepalive) for a numpy array or torch tensor of the given numpy dtype."""
    if a is None:
        return None, None
    if _is_torch(a):
        import torch
        tdt = {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[dtype]
        if a.dtype != tdt or not a.is_contiguous():
            a = a.to(tdt).contiguous()
        return C.c_void_p(a.data_ptr()), a
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data_as(C.c_void_p), arr


def _like(x, n):
    """Output buffer on the same side (host numpy / device tensor) as x."""
    if _is_torch(x):
        import torch
        return torch.empty(n, dtype=torch.float64, device=x.device)
    return np.empty(n, dtype=np.float64)


def _stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def default_params() -> Params:
    return load().gpcg_params_default()


# ---------------------------------------------------------------- row slabs (gpcg_dist)
def partition_rows(total, parts, part):
    """[begin, end) of part `part` of a balanced contiguous split of [0, total) (the C helper)."""
    b, e = C.c_int64(), C.c_int64()
    load().gpcg_partition_rows(int(total), int(parts), int(part), C.byref(b), C.byref(e))
    return b.value, e.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load().gpcg_nccl_unique_id(buf))
    return buf.raw


def problem_rows(prob):
    """Rows the slab split runs over: grid rows (stencil2d), z-planes (stencil3d), matrix rows (CSR)."""
    return {"stencil2d": prob.ny, "stencil3d": prob.nz}.get(prob.kind, prob.n)


def local_part(prob, row_begin, row_end):
    """The arrays a rank owning global rows [row_begin, row_end) passes to the *_dist
    creators (include/gpcg.h): its rows of b, l, u, x0, shift; its grid rows of
    full x-face arrays and face rows row_begin..row_end of full y-face arrays; for
    CSR its rows of row_ptr (rebased) / col (global ids) / val.  Host-side slicing
    only."""
    out = {}
    if prob.kind == "stencil2d":
        nx = prob.nx
        sl = slice(row_begin * nx, row_end * nx)
        for k in ("b", "l", "u", "x0"):
            out[k] = np.ascontiguousarray(np.asarray(getattr(prob, k))[sl])
        out["shift"] = None if prob.shift is None else np.ascontiguousarray(np.asarray(prob.shift)[sl])
        wx = np.asarray(prob.wx)
        wy = np.asarray(prob.wy)
        out["wx"] = wx if not prob.wx_ld else np.ascontiguousarray(
            wx[row_begin * prob.wx_ld:(row_end - 1) * prob.wx_ld + nx + 1])
        out["wy"] = wy if not prob.wy_ld else np.ascontiguousarray(
            wy[row_begin * prob.wy_ld:row_end * prob.wy_ld + nx])
        out["n"] = (row_end - row_begin) * nx
    elif prob.kind == "stencil3d":
        nx, ny = prob.nx, prob.ny
        pl = nx * ny
        sl = slice(row_begin * pl, row_end * pl)
        for k in ("b", "l", "u", "x0"):
            out[k] = np.ascontiguousarray(np.asarray(getattr(prob, k))[sl])
        out["shift"] = None if prob.shift is None else np.ascontiguousarray(np.asarray(prob.shift)[sl])
        out["wx"] = np.ascontiguousarray(np.asarray(prob.wx)[row_begin * (nx + 1) * ny:row_end * (nx + 1) * ny])
        out["wy"] = np.ascontiguousarray(np.asarray(prob.wy)[row_begin * nx * (ny + 1):row_end * nx * (ny + 1)])
        out["wz"] = np.ascontiguousarray(np.asarray(prob.wz)[row_begin * pl:(row_end + 1) * pl])   # face planes rb..re
        out["n"] = (row_end - row_begin) * pl
    else:
        rp = np.asarray(prob.row_ptr, dtype=np.int64)
        k0, k1 = int(rp[row_begin]), int(rp[row_end])
        out["row_ptr"] = rp[row_begin:row_end + 1] - k0
        out["col"] = np.ascontiguousarray(np.asarray(prob.col, dtype=np.int32)[k0:k1])
        out["val"] = np.ascontiguousarray(np.asarray(prob.val, dtype=np.float64)[k0:k1])
        for k in ("b", "l", "u", "x0"):
            out[k] = np.ascontiguousarray(np.asarray(getattr(prob, k))[row_begin:row_end])
        out["n"] = row_end - row_begin
    return out


class Solver:
    """One GPCG problem instance on the current CUDA device (wraps gpcg_problem*)."""

    def __init__(self, handle, n):
        self._h = handle
        self.n = n

    # ------------------------------------------------------------ creation
    @classmethod
    def stencil2d(cls, nx, ny, wx, wx_ld, wy, wy_ld, b, l, u, c=0.0, shift=None, stream=None):
        L = load()
        h = C.c_void_p()
        keep = []
        args = []
        for a in (wx, wy, shift, b, l, u):
            p, k = _ptr(a, np.float64)
            args.append(p)
            keep.append(k)
        rc = L.gpcg_create_stencil2d(C.byref(h), _stream_ptr(stream), nx, ny, args[0], wx_ld, args[1],
                                     wy_ld, args[2], args[3], args[4], args[5], float(c))
        _check(rc)
        return cls(h, nx * ny)

    @classmethod
    def stencil3d(cls, nx, ny, nz, wx, wy, wz, b, l, u, c=0.0, shift=None, stream=None):
        L = load()
        h = C.c_void_p()
        keep = []
        args = []
        for a in (wx, wy, wz, shift, b, l, u):
            p, k = _ptr(a, np.float64)
            args.append(p)
            keep.append(k)
        rc = L.gpcg_create_stencil3d(C.byref(h), _stream_ptr(stream), nx, ny, nz, *args, float(c))
        _check(rc)
        return cls(h, nx * ny * nz)

    @classmethod
    def csr(cls, n, row_ptr, col, val, b, l, u, c=0.0, stream=None):
        L = load()
        h = C.c_void_p()
        prp, k1 = _ptr(row_ptr, np.int64)
        pci, k2 = _ptr(col, np.int32)
        pva, k3 = _ptr(val, np.float64)
        pb, k4 = _ptr(b, np.float64)
        pl, k5 = _ptr(l, np.float64)
        pu, k6 = _ptr(u, np.float64)
        rc = L.gpcg_create_csr(C.byref(h), _stream_ptr(stream), n, prp, pci, pva, pb, pl, pu, float(c))
        _check(rc)
        return cls(h, n)

    @classmethod
    def dist(cls, prob, rank=0, nranks=1, nccl_id=None, local_slabs=1, stream=None, device=None, local=None):
        """The rank's slab of a problems.Problem (rows split by partition_rows) through
        gpcg_create_*_dist.  Returns (solver, row_begin, row_end, local arrays).
        local: precomputed local_part arrays (e.g. pinned copies) to pass instead."""
        rb, re = partition_rows(problem_rows(prob), nranks, rank)
        loc = local_part(prob, rb, re) if local is None else local
        conv = (lambda a: a) if device is None else _to_device(device)
        idbuf = None
        if nranks > 1:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        d = Dist(rank, nranks, C.cast(idbuf, C.c_void_p) if idbuf is not None else None, rb, re, local_slabs)
        L = load()
        h = C.c_void_p()
        keep = []

        def P(a, dt=np.float64):
            p, k = _ptr(None if a is None else conv(a), dt)
            keep.append(k)
            return p
        if prob.kind == "stencil2d":
            rc = L.gpcg_create_stencil2d_dist(C.byref(h), C.byref(d), _stream_ptr(stream), prob.nx, prob.ny,
                                              P(loc["wx"]), prob.wx_ld, P(loc["wy"]), prob.wy_ld, P(loc["shift"]),
                                              P(loc["b"]), P(loc["l"]), P(loc["u"]), float(prob.c))
        elif prob.kind == "stencil3d":
            rc = L.gpcg_create_stencil3d_dist(C.byref(h), C.byref(d), _stream_ptr(stream), prob.nx, prob.ny,
                                              prob.nz, P(loc["wx"]), P(loc["wy"]), P(loc["wz"]), P(loc["shift"]),
                                              P(loc["b"]), P(loc["l"]), P(loc["u"]), float(prob.c))
        else:
            rc = L.gpcg_create_csr_dist(C.byref(h), C.byref(d), _stream_ptr(stream), prob.n,
                                        P(loc["row_ptr"], np.int64), P(loc["col"], np.int32), P(loc["val"]),
                                        P(loc["b"]), P(loc["l"]), P(loc["u"]), float(prob.c))
        _check(rc)
        return cls(h, loc["n"]), rb, re, loc

    @classmethod
    def from_problem(cls, prob, stream=None, device=None, slabs=1):
        """Create from a problems.Problem; device='cuda' uploads inputs as CUDA tensors first.
        slabs > 1: the same problem split into that many row slabs on this device (gpcg_dist
        local_slabs; the multi-rank code path with device-copy halos)."""
        if slabs > 1:
            return cls.dist(prob, local_slabs=slabs, stream=stream, device=device)[0]
        conv = (lambda a: a) if device is None else _to_device(device)
        if prob.kind == "stencil3d":
            return cls.stencil3d(prob.nx, prob.ny, prob.nz, conv(prob.wx), conv(prob.wy), conv(prob.wz),
                                 conv(prob.b), conv(prob.l), conv(prob.u), prob.c,
                                 shift=None if prob.shift is None else conv(prob.shift), stream=stream)
        if prob.kind == "stencil2d":
            return cls.stencil2d(prob.nx, prob.ny, conv(prob.wx), prob.wx_ld, conv(prob.wy), prob.wy_ld,
                                 conv(prob.b), conv(prob.l), conv(prob.u), prob.c,
                                 shift=None if prob.shift is None else conv(prob.shift), stream=stream)
        return cls.csr(prob.n, conv(prob.row_ptr), conv(prob.col), conv(prob.val), conv(prob.b),
                       conv(prob.l), conv(prob.u), prob.c, stream=stream)

    # ------------------------------------------------------------ calls
    def set_params(self, **kw):
        p = default_params()
        for k, v in kw.items():
            if not hasattr(p, k):
                raise AttributeError(k)
            setattr(p, k, v)
        _check(load().gpcg_set_params(self._h, C.byref(p)))

    def solve(self, x0, tol, max_it=500, x_out=None, allow_error=False):
        """-> (status, x, stats dict).  Raises on errors unless allow_error."""
        px0, k0 = _ptr(x0, np.float64)
        if x_out is None:
            x_out = _like(x0, self.n)
        pxo, ko = _ptr(x_out, np.float64)
        st = Stats()
        rc = load().gpcg_solve(self._h, px0, float(tol), int(max_it), pxo, C.byref(st))
        if not allow_error:
            _check(rc, (OK, NOT_CONVERGED))
        if ko is not x_out and not _is_torch(x_out):
            x_out[...] = ko
        return rc, x_out, st.asdict()

    def hessvec(self, v, y=None, reduced=False):
        pv, kv = _ptr(v, np.float64)
        if y is None:
            y = _like(v, self.n)
        py, ky = _ptr(y, np.float64)
        _check(load().gpcg_hessvec(self._h, pv, py, 1 if reduced else 0))
        return y

    def free_count(self):
        """|F| of the recorded free set (-1: none, or no compacted free-row list for this handle)"""
        return int(load().gpcg_free_count(self._h))

    def hessvec_free(self, v, y_free=None):
        """y_free[k] = (A_F v) at the k-th free index (compact output, gpcg_hessvec_free)"""
        pv, kv = _ptr(v, np.float64)
        if y_free is None:
            y_free = _like(v, max(self.free_count(), 0))
        py, ky = _ptr(y_free, np.float64)
        _check(load().gpcg_hessvec_free(self._h, pv, py))
        if ky is not y_free and not _is_torch(y_free):
            y_free[...] = ky
        return y_free

    def project(self, x, px=None):
        """-> (px, ||grad_Omega q(px)||^2, |A(px)|, |A(px) minus B(px)|)"""
        pxx, kx = _ptr(x, np.float64)
        if px is None:
            px = _like(x, self.n)
        ppx, kp = _ptr(px, np.float64)
        pg2 = C.c_double()
        na = C.c_int64()
        nnb = C.c_int64()
        _check(load().gpcg_project(self._h, pxx, ppx, C.byref(pg2), C.byref(na), C.byref(nnb)))
        return px, pg2.value, na.value, nnb.value

    def objective(self, x):
        pxx, kx = _ptr(x, np.float64)
        q = C.c_double()
        _check(load().gpcg_objective(self._h, pxx, C.byref(q)))
        return q.value

    def close(self):
        if self._h:
            load().gpcg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _to_device(device):
    import torch

    def conv(a):
        if a is None:
            return None
        return torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return conv
