"""CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Tolerances are those of BASELINE.json's north_star:
  * single SpMV: ||y - y_ora||_inf <= 1e-13 ||(|A||p|)||_inf and
                 ||y - y_ora||_2  <= 1e-13 ||y_ora||_2;
  * projection, active/free sets, counts: bit-exact;
  * solve: |q - q_ora| <= 1e-10 |q_ora|, ||x - x_ora||_inf <= 1e-7 (both solved to
    a tolerance whose a-posteriori bound certifies it), identical active sets
    away from degenerate ties (free copy within 1e-7 of the bound).
"""
import numpy as np
import pytest

from paper_cs_0101018_b200 import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_cs_0101018_b200 import _build, gpcg
    _build.build()
    return gpcg


def abs_op(A, p):
    """|A| |p| rowwise (oracle CSR), the cancellation-free SpMV scale."""
    rows = np.repeat(np.arange(A.n), np.diff(A.rp))
    return np.bincount(rows, weights=np.abs(A.val) * np.abs(p[A.ci]), minlength=A.n)


def abs_op_rows(A, p, idx):
    """|A| |p| on the rows idx only (sampled checks at full size)."""
    out = np.zeros(len(idx))
    for t, i in enumerate(idx):
        k0, k1 = A.rp[i], A.rp[i + 1]
        out[t] = np.sum(np.abs(A.val[k0:k1]) * np.abs(p[A.ci[k0:k1]]))
    return out


def spmv_close(y, yref, scale):
    d = np.abs(np.asarray(y) - yref)
    assert d.max() <= 1e-13 * max(scale.max(), 1e-300), (d.max(), scale.max())
    assert np.linalg.norm(d) <= 1e-13 * max(np.linalg.norm(yref), 1e-300) + 1e-13 * scale.max()


def ragged_stencil(nx, ny, seed, full=True, shift=True, bounds="two"):
    if full:
        wx = 0.5 + P.uniform(seed, 1, ny * (nx + 1)); wx_ld = nx + 1
        wy = 0.5 + P.uniform(seed, 2, (ny + 1) * nx); wy_ld = nx
    else:
        wx = 0.5 + P.uniform(seed, 1, nx + 1); wx_ld = 0
        wy = 0.5 + P.uniform(seed, 2, nx); wy_ld = 0
    n = nx * ny
    sh = 0.01 * P.uniform(seed, 3, n) if shift else None
    b = P.gaussian(seed, 4, n)
    if bounds == "two":
        l = -0.3 * P.uniform(seed, 5, n)
        u = 0.3 * P.uniform(seed, 6, n)
    elif bounds == "inf":
        l = np.full(n, -np.inf); u = np.full(n, np.inf)
    else:
        l = np.zeros(n); u = np.full(n, np.inf)
    return P.Problem(name=f"ragged{nx}x{ny}", kind="stencil2d", n=n, b=b, l=l, u=u,
                     x0=P.gaussian(seed, 7, n), tol=-1e-10, nx=nx, ny=ny, wx=wx, wx_ld=wx_ld,
                     wy=wy, wy_ld=wy_ld, shift=sh)


def dense_problem(n, seed, bounds="mixed"):
    A, b, l, u = P.random_dense_qp(n, seed, bounds)
    return P.csr_problem(A, b, l, u, x0=P.gaussian(seed, 9, n), tol=-1e-12, name=f"dense{n}")


SPMV_CASES = {
    "C0": lambda: P.c0(),
    "C1": lambda: P.c1(),
    "ragged37x23": lambda: ragged_stencil(37, 23, 5),
    "ragged1x9": lambda: ragged_stencil(1, 9, 6, full=False),
    "ragged33x1": lambda: ragged_stencil(33, 1, 7),
    "c4_m12": lambda: P.c4_family(m=12),
    "dense40": lambda: dense_problem(40, 3),
}


@pytest.mark.parametrize("case", list(SPMV_CASES))
def test_spmv_full_and_reduced(G, oracle, case):
    prob = SPMV_CASES[case]()
    A = oracle.problem_csr(prob)
    p = 2.0 * P.uniform(99, 1, prob.n) - 1.0
    with G.Solver.from_problem(prob) as s:
        y = s.hessvec(p)
        spmv_close(y, oracle.spmv(A, p), abs_op(A, p))
        # reduced: free set of P[x] for a point with ~half the bounds active
        x = prob.x0 if np.isfinite(prob.l).any() or np.isfinite(prob.u).any() else p
        px, pg2, na, nnb = s.project(x)
        pref = oracle.project(prob.l, prob.u, x)
        assert np.array_equal(px, pref)
        free = ~oracle.sets(pref, np.zeros(prob.n), prob.l, prob.u)[0]
        yr = s.hessvec(p, reduced=True)
        yref = oracle.spmv_masked(A, free, p)
        spmv_close(yr, yref, abs_op(A, p * free))
        assert np.all(np.asarray(yr)[~free] == 0.0)


@pytest.mark.parametrize("case", ["C0", "C1", "ragged37x23", "c4_m12", "dense40"])
def test_project_counts_exact(G, oracle, case):
    prob = SPMV_CASES[case]()
    A = oracle.problem_csr(prob)
    x = prob.x0 + 0.05 * P.gaussian(5, 5, prob.n)
    with G.Solver.from_problem(prob) as s:
        px, pg2, na, nnb = s.project(x)
    pref = oracle.project(prob.l, prob.u, x)
    assert np.array_equal(px, pref)
    g = oracle.gradient(A, prob.b, pref)
    act, bnd, na_ref, nb_ref = oracle.sets(pref, g, prob.l, prob.u)
    assert na == na_ref
    assert nnb == na_ref - nb_ref
    pg_ref = np.sum(oracle.proj_grad(pref, g, prob.l, prob.u) ** 2)
    assert abs(pg2 - pg_ref) <= 1e-12 * pg_ref


def test_objective(G, oracle):
    prob = P.c1()
    A = oracle.problem_csr(prob)
    x = P.gaussian(3, 3, prob.n) * 1e-3
    with G.Solver.from_problem(prob) as s:
        q = s.objective(x)
    qref = oracle.objective(A, prob.b, prob.c, x)
    assert abs(q - qref) <= 1e-12 * abs(qref)


def _tie_mismatches(x, xr, l, u):
    act = (x == l) | (x == u)
    actr = (xr == l) | (xr == u)
    mism = np.flatnonzero(act != actr)
    nontie = []
    for i in mism:
        free_val = x[i] if not act[i] else xr[i]
        bound = l[i] if (xr[i] == l[i] or x[i] == l[i]) else u[i]
        if abs(free_val - bound) > 1e-7:
            nontie.append(i)
    return len(mism), nontie


SOLVE_CASES = {
    "C0": (lambda: P.c0(), -1e-12),
    "C1": (lambda: P.c1(), -1e-11),
    "jb80_eps0.9": (lambda: P.journal_bearing(80, 60, eps=0.9), -1e-11),
    "c3_family_160": (lambda: P.c3_family(160, 160), -1e-11),
    "c4_family_m16": (lambda: P.c4_family(m=16), -1e-11),
    "ragged37x23": (lambda: ragged_stencil(37, 23, 5), -1e-12),
    "ragged_inf": (lambda: ragged_stencil(19, 13, 8, bounds="inf"), -1e-12),
    "dense8": (lambda: dense_problem(8, 21), -1e-12),
}


@pytest.mark.parametrize("case", list(SOLVE_CASES))
def test_solve_parity(G, oracle, case):
    make, tol = SOLVE_CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    assert rc_o == 0
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0, (rc, st)
    assert np.all(x >= prob.l) and np.all(x <= prob.u)
    assert st["pg_norm"] <= st["tau"]
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7
    nm, nontie = _tie_mismatches(x, x_o, prob.l, prob.u)
    assert not nontie, (nm, nontie[:10])
    # oracle's own certificate of the GPU point: KKT via one CPU SpMV
    A = oracle.problem_csr(prob)
    g = oracle.gradient(A, prob.b, x)
    pg = np.linalg.norm(oracle.proj_grad(x, g, prob.l, prob.u))
    assert pg <= 1.01 * st["tau"] + 1e-15


def test_solve_unconstrained_is_direct_solve(G):
    prob = dense_problem(30, 77, bounds="inf")
    A = np.zeros((30, 30))
    rows = np.repeat(np.arange(30), np.diff(prob.row_ptr))
    A[rows, prob.col] = prob.val
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(np.zeros(30), -1e-13)
    assert rc == 0 and np.max(np.abs(x - np.linalg.solve(A, prob.b))) <= 1e-9


def test_solve_enumeration_small(G):
    from tests import _brute as B
    for sd in range(20):
        n = 2 + sd % 7
        A, b, l, u = P.random_dense_qp(n, seed=3000 + sd, bounds="mixed")
        prob = P.csr_problem(A, b, l, u, x0=P.gaussian(sd, 1, n))
        with G.Solver.from_problem(prob) as s:
            rc, x, st = s.solve(prob.x0, -1e-12)
        assert rc == 0
        assert np.max(np.abs(x - B.enum_solve(A, b, l, u))) <= 1e-6


def test_c_example_matches_oracle(G, oracle, tmp_path):
    """examples/solve_bearing.c -- the ABI from plain C, host arrays -- solves C0 to the oracle's q*."""
    import subprocess
    from tests.test_abi import example_binary
    exe = example_binary(str(tmp_path))
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    fields = dict(kv.split("=") for kv in out.stdout.split())
    rc_o, x_o, st_o = oracle.solve_problem(P.c0(), tol=-1e-8)
    assert fields["status"] == "0" and rc_o == 0
    assert abs(float(fields["q"]) - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert abs(int(fields["free"]) - int(np.sum(x_o > 0.0))) <= 2      # degenerate ties aside


def test_device_pointers_and_determinism(G):
    import torch
    prob = P.c1()
    with G.Solver.from_problem(prob, device="cuda") as s:
        x0 = torch.from_numpy(prob.x0).cuda()
        rc1, x1, st1 = s.solve(x0, -1e-8)
        rc2, x2, st2 = s.solve(x0, -1e-8)
    assert x1.is_cuda and rc1 == 0
    assert torch.equal(x1, x2)                     # bitwise reproducible
    assert st1["cg_iters"] == st2["cg_iters"]


@pytest.mark.parametrize("pool", ["1", "0"])
def test_create_destroy_cycles_reuse_memory(G, monkeypatch, pool):
    """Handles allocate from a retained stream-ordered pool (GPCG_POOL=0: cudaMalloc): repeated
    create / solve / destroy cycles, with a live handle in between, give bitwise the same result."""
    import torch
    monkeypatch.setenv("GPCG_POOL", pool)
    prob = P.c1()
    x0 = torch.from_numpy(prob.x0).cuda()
    ref = None
    keep = G.Solver.from_problem(P.c0(), device="cuda")
    for _ in range(3):
        with G.Solver.from_problem(prob, device="cuda") as s:
            rc, x, st = s.solve(x0, -1e-8)
        assert rc == 0
        if ref is None:
            ref = x.clone()
        assert torch.equal(x, ref)
    rc0, _, _ = keep.solve(torch.zeros(P.c0().n, dtype=torch.float64, device="cuda"), -1e-8)
    keep.close()
    assert rc0 == 0


# ------------------------------------------------------------------ edge cases
def test_edge_tiny_grids(G, oracle):
    for nx, ny in [(1, 1), (1, 2), (3, 1)]:
        prob = ragged_stencil(nx, ny, 40 + nx + ny)
        rc_o, x_o, st_o = oracle.solve_problem(prob, tol=-1e-12)
        with G.Solver.from_problem(prob) as s:
            rc, x, st = s.solve(prob.x0, -1e-12)
        assert rc == 0 and np.max(np.abs(x - x_o)) <= 1e-9


def test_edge_all_fixed_and_converged_start(G):
    prob = ragged_stencil(9, 7, 3)
    prob.l = prob.u = np.full(prob.n, 0.125)
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(np.zeros(prob.n), 1e-10)
    assert rc == 0 and np.all(x == 0.125) and st["outer_iters"] == 0 and st["n_free"] == 0
    prob = P.journal_bearing(10, 10, eps=0.0)                # x* = 0 = x0
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(np.zeros(prob.n), 1e-12)
    assert rc == 0 and np.all(x == 0.0) and st["outer_iters"] == 0


def test_edge_errors(G):
    prob = ragged_stencil(5, 4, 1)
    with G.Solver.from_problem(prob) as s:
        with pytest.raises(G.GpcgError) as e:
            s.hessvec(np.ones(prob.n), reduced=True)
        assert e.value.code == G.ESTATE
    bad = ragged_stencil(5, 4, 1)
    bad.l = bad.l.copy(); bad.l[3] = 1.0; bad.u = bad.u.copy(); bad.u[3] = 0.0
    with pytest.raises(G.GpcgError) as e:
        G.Solver.from_problem(bad)
    assert e.value.code == G.EINVAL
    nanb = ragged_stencil(5, 4, 1)
    nanb.b = nanb.b.copy(); nanb.b[0] = np.nan
    with pytest.raises(G.GpcgError):
        G.Solver.from_problem(nanb)
    indef = P.csr_problem(np.array([[1.0, 2.0], [2.0, 1.0]]), [1.0, -1.0], [-1e3, -1e3], [1e3, 1e3])
    with G.Solver.from_problem(indef) as s:
        rc, x, st = s.solve(np.zeros(2), 1e-8, allow_error=True)
    assert rc == G.ENOTSPD


def test_not_converged_returns_feasible(G):
    prob = P.c1()
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(prob.x0, -1e-12, max_it=1)
    assert rc == G.NOT_CONVERGED and st["outer_iters"] == 1
    assert np.all(x >= prob.l) and np.all(x <= prob.u)


# ------------------------------------------------------------------ full size (bench config)
def test_c2_full_size_certificate(G, oracle):
    """C2 (1600^2, the bench workload): GPU solve certified by the oracle's own
    SpMV (KKT / ||grad_Omega q|| / B = A), sampled SpMV rows, free fraction."""
    prob = P.c2()
    A = oracle.problem_csr(prob)
    with G.Solver.from_problem(prob) as s:
        p = 2.0 * P.uniform(5, 1, prob.n) - 1.0
        y = s.hessvec(p)
        idx = (P.uniform(5, 2, 2000) * prob.n).astype(np.int64)
        sub = oracle.spmv(A, p)
        spmv_close(y[idx], sub[idx], abs_op(A, p)[idx])
        rc, x, st = s.solve(prob.x0, prob.tol)
    assert rc == 0
    g = oracle.gradient(A, prob.b, x)
    pg = np.linalg.norm(oracle.proj_grad(x, g, prob.l, prob.u))
    assert pg <= 1.01 * st["tau"]
    act, bnd, na, nb = oracle.sets(x, g, prob.l, prob.u)
    assert na == st["n_active"] and na - nb == 0
    assert 0.60 <= 1 - na / prob.n <= 0.76           # PAPER.md:876-878 (~68% free)


# ------------------------------------------------------------------ oracle goldens (sizes the oracle
# cannot solve inside a test run; written by scripts/golden_oracle.py, which calls only oracle/)
GOLDEN = {
    "C2": lambda: P.c2(),
    "C3_1600": lambda: P.c3_family(1600, 1600),
    "C4_128": lambda: P.c4_family(m=128),
    "C4": lambda: P.c4(),
}


@pytest.mark.parametrize("name", list(GOLDEN))
def test_solve_parity_vs_oracle_golden(G, name):
    import base64
    import json
    import os
    import zlib
    path = os.path.join(os.path.dirname(__file__), "golden", f"oracle_{name}.json")
    gold = json.load(open(path))
    prob = GOLDEN[name]()
    assert prob.n == gold["n"] and gold["rc"] == 0
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(prob.x0, gold["tol"])
    assert rc == 0, (rc, st)
    assert abs(st["q"] - gold["q"]) <= 1e-10 * abs(gold["q"]), (st["q"], gold["q"])
    idx = np.asarray(gold["idx"])
    xo = np.asarray(gold["x"])
    assert np.max(np.abs(x[idx] - xo)) <= 1e-7, np.max(np.abs(x[idx] - xo))
    # active sets over ALL n points (the oracle's set is stored bit-packed): identical away from
    # degenerate ties: a point active on one side only must be free on the other
    # side within 1e-7 of the bound -- the GPU's x is at hand; the oracle's free points near a
    # bound are stored with their x (near_idx / near_x)
    acto = np.unpackbits(np.frombuffer(zlib.decompress(base64.b64decode(gold["active_packbits_zlib_b64"])),
                                       dtype=np.uint8))[: prob.n].astype(bool)
    assert int(acto.sum()) == gold["n_active"]
    act = (x == prob.l) | (x == prob.u)
    mism = np.flatnonzero(act != acto)
    near = dict(zip(gold["near_idx"], gold["near_x"]))
    nontie = []
    for i in mism:
        if acto[i]:      # oracle active, GPU free: the GPU's value must sit within 1e-7 of a bound
            ok = min(abs(x[i] - prob.l[i]), abs(x[i] - prob.u[i])) <= 1e-7
        else:            # GPU active, oracle free: the oracle's point must be a stored near-bound tie
            ok = int(i) in near
        if not ok:
            nontie.append(int(i))
    assert not nontie, (len(mism), nontie[:10])
    ties = [int(i) for i in mism]
    print(f"[parity] {name}: active-set mismatches {len(mism)} (all ties within 1e-7 of the bound); "
          f"oracle near-bound free points {gold['n_free_near_bound']}; "
          f"min |g_i| over the oracle's ties {min(gold['near_absg'], default=float('nan')):.3e}; "
          f"tie indices {ties[:8]}")
    assert st["n_active"] == int(act.sum())


# ------------------------------------------------------------------ C3 at full size (BASELINE.json configs[3],
# 8000^2 = 64M variables): no oracle solve fits a test run, so the GPU solution is certified by the
# oracle's own code (SURVEY 8(c) "at full C3 size"): one CPU SpMV gives g, then the KKT conditions,
# ||grad_Omega q|| <= tau (to 1 %) and B = A; plus the reduced HVP at 1e-13 on sampled rows.
def test_c3_full_size_solve_certified_by_oracle(G, oracle):
    import time
    prob = P.c3()
    assert prob.n == 64_000_000
    t0 = time.perf_counter()
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(prob.x0, prob.tol)          # default parameters, tau = 1e-8 ||g(x0)||
        t_solve = time.perf_counter() - t0
        p = 2.0 * P.uniform(33, 1, prob.n) - 1.0
        yr = s.hessvec(p, reduced=True)                 # on the solution's free set
    assert rc == 0, (rc, st)
    A = oracle.problem_csr(prob)
    g = oracle.gradient(A, prob.b, x)
    assert np.all(x >= prob.l) and np.all(x <= prob.u)
    pg = np.linalg.norm(oracle.proj_grad(x, g, prob.l, prob.u))
    assert pg <= 1.01 * st["tau"], (pg, st["tau"])
    act, bnd, na, nb = oracle.sets(x, g, prob.l, prob.u)
    assert na == nb, (na, nb)                            # B = A
    assert na == st["n_active"]
    assert 0.47 <= na / prob.n <= 0.53                   # calibrated ~50 % active (configs[3])
    free = ~act
    idx = np.unique((P.uniform(33, 2, 20000) * prob.n).astype(np.int64))
    ysub = oracle.spmv_masked(A, free, p)
    spmv_close(yr[idx], ysub[idx], abs_op_rows(A, p * free, idx))
    # a-posteriori bound E = ||grad_Omega q|| / lambda_lb (SURVEY 8(c) parity protocol)
    hx, hy = prob.meta["hx"], prob.meta["hy"]
    lam = (0.9 ** 3) * ((hy / hx) * 4 * np.sin(np.pi / (2 * (prob.nx + 1))) ** 2 +
                        (hx / hy) * 4 * np.sin(np.pi / (2 * (prob.ny + 1))) ** 2)
    print(f"[C3] solve {t_solve:.1f} s outer={st['outer_iters']} gp={st['gp_iters']} cg={st['cg_iters']} "
          f"|A|/n={na / prob.n:.4f} pg={pg:.3e} tau={st['tau']:.3e} E=pg/lambda_lb={pg / lam:.3e}")


# ------------------------------------------------------------------ point-Jacobi PCG
PCG_CASES = ["C0", "C1", "jb80_eps0.9", "c4_family_m16", "ragged37x23", "dense8"]


@pytest.mark.parametrize("case", PCG_CASES)
def test_solve_parity_pcg(G, oracle, case):
    make, tol = SOLVE_CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol, params=oracle.default_params(precond=1))
    assert rc_o == 0
    with G.Solver.from_problem(prob) as s:
        s.set_params(precond=1)
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0, (rc, st)
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7
    nm, nontie = _tie_mismatches(x, x_o, prob.l, prob.u)
    assert not nontie


def test_pcg_fewer_cg_iterations_on_scaled_operator(G):
    """Badly scaled rows (full faces with a wide spread): the diagonal preconditioner
    must cut CG iterations (the point Jacobi method is the baseline of Table 4)."""
    prob = ragged_stencil(60, 50, 9, bounds="inf")
    sc = np.exp(3.0 * P.uniform(9, 50, prob.n))
    prob.shift = prob.shift * 0 + sc            # diagonal shift spanning 3 decades
    its = {}
    for pc in (0, 1):
        with G.Solver.from_problem(prob) as s:
            s.set_params(precond=pc)
            rc, x, st = s.solve(np.zeros(prob.n), -1e-10)
        assert rc == 0
        its[pc] = st["cg_iters"]
    assert its[1] < its[0], its


# ------------------------------------------------------------------ every stencil kernel family
# GPCG_TILE selects the sweep implementations (gpcg.cu): 0 column march (k2),
# 63 TMA-fed march with stored g (k4), 127 g-free TMA-fed march (k5, the default).  Each must
# reach the oracle's solution on its own.
@pytest.mark.parametrize("tile", ["0", "63", "127"])
@pytest.mark.parametrize("case", ["C0", "c3_family_160", "jb80_eps0.9"])
def test_kernel_families_parity(G, oracle, monkeypatch, tile, case):
    monkeypatch.setenv("GPCG_TILE", tile)
    make, tol = SOLVE_CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    for pc in (0, 1):
        with G.Solver.from_problem(prob) as s:
            s.set_params(precond=pc)
            rc, x, st = s.solve(prob.x0, tol)
        assert rc == 0, (tile, pc, st)
        assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
        assert np.max(np.abs(x - x_o)) <= 1e-7
    # the GP phase on the host (GPCG_GP_GRAPH=0) reaches the same point
    monkeypatch.setenv("GPCG_GP_GRAPH", "0")
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0 and np.max(np.abs(x - x_o)) <= 1e-7


# ------------------------------------------------------------------ the GP-phase cap (reading R13)
@pytest.mark.parametrize("cap", [2, 5])
@pytest.mark.parametrize("case", ["C0", "c3_family_160", "jb80_eps0.9"])
def test_gp_cap_parity(G, oracle, monkeypatch, case, cap):
    """GP phases that stop at gpcg_params.gp_cap (persistent GP loop and host-driven path)
    follow the oracle with the same cap: same first-outer-iteration counts, same x*."""
    make, tol = SOLVE_CASES[case]
    prob = make()
    prm = oracle.default_params(gp_cap=cap, refine_cap=1)
    rc_o1, x_o1, st_o1 = oracle.solve_problem(prob, tol=tol, max_it=1, params=prm)
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol, params=oracle.default_params(gp_cap=cap))
    for graph in ("1", "0"):
        monkeypatch.setenv("GPCG_GP_GRAPH", graph)
        with G.Solver.from_problem(prob) as s:
            s.set_params(gp_cap=cap, refine_cap=1)
            rc1, x1, st1 = s.solve(prob.x0, tol, max_it=1, allow_error=True)
            s.set_params(gp_cap=cap, refine_cap=30)
            rc, x, st = s.solve(prob.x0, tol)
        assert st1["gp_iters"] == st_o1["gp_iters"], (graph, st1["gp_iters"], st_o1["gp_iters"])
        # after a capped GP phase the CG call starts far from the face minimiser and runs long
        # on a flat decrease profile, so the C-G vs textbook rounding can move the cgstop1
        # iteration by a few (C0: 1e-7 relative in x; jb80: 213 vs 210 iterations)
        assert abs(st1["cg_iters"] - st_o1["cg_iters"]) <= 1 + 0.03 * st_o1["cg_iters"], \
            (st1["cg_iters"], st_o1["cg_iters"])
        assert rc == 0 and rc_o == 0
        assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
        assert np.max(np.abs(x - x_o)) <= 1e-7


# ------------------------------------------------------------------ A/B switches of the single-slab path
@pytest.mark.parametrize("switch", ["GPCG_CG_PERSIST", "GPCG_GP_PERSIST", "GPCG_CG_SKIP", "GPCG_GP_SPEC"])
@pytest.mark.parametrize("case", ["C0", "jb80_eps0.9", "c3_family_160"])
def test_path_switches_parity(G, oracle, monkeypatch, switch, case):
    """Each switch turns one device-side optimisation off (graph-chunk CG / GP instead of the
    persistent loops, no all-active block skipping, no speculative GP step): the same x*."""
    monkeypatch.setenv(switch, "0")
    make, tol = SOLVE_CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    for pc in (0, 1):
        with G.Solver.from_problem(prob) as s:
            s.set_params(precond=pc)
            rc, x, st = s.solve(prob.x0, tol)
        assert rc == 0 and rc_o == 0
        assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
        assert np.max(np.abs(x - x_o)) <= 1e-7


# ------------------------------------------------------------------ 3-D 7-point stencil (NEXT-2)
@pytest.mark.parametrize("m", [5, 12, 16])
def test_stencil3d_spmv_and_solve_parity(G, oracle, m):
    prob = P.c4_stencil_family(m=m)
    A = oracle.problem_csr(prob)
    p = 2.0 * P.uniform(97, 1, prob.n) - 1.0
    with G.Solver.from_problem(prob) as s:
        spmv_close(s.hessvec(p), oracle.spmv(A, p), abs_op(A, p))
        rc, x, st = s.solve(prob.x0, -1e-11)
        yr = s.hessvec(p, reduced=True)
    free = (x > prob.l) & (x < prob.u)
    spmv_close(yr, oracle.spmv_masked(A, free, p), abs_op(A, p * free))
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=-1e-11)
    assert rc == 0 and rc_o == 0
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7
    nm, nontie = _tie_mismatches(x, x_o, prob.l, prob.u)
    assert not nontie


def ragged_stencil3d(nx, ny, nz, seed, shift=True, bounds="two"):
    """3-D 7-point face-weight stencil with every face (boundary faces too) positive, so the
    diagonal carries the Dirichlet boundary faces; sizes chosen off the plane-march tiles."""
    wx = 0.5 + P.uniform(seed, 1, nz * ny * (nx + 1))
    wy = 0.5 + P.uniform(seed, 2, nz * (ny + 1) * nx)
    wz = 0.5 + P.uniform(seed, 3, (nz + 1) * ny * nx)
    n = nx * ny * nz
    sh = 0.01 * P.uniform(seed, 4, n) if shift else None
    b = P.gaussian(seed, 5, n)
    if bounds == "two":
        l = -0.2 * P.uniform(seed, 6, n)
        u = 0.2 * P.uniform(seed, 7, n)
    else:
        l = np.full(n, -0.05); u = np.full(n, 0.05)      # scalar bounds (the SB kernels)
    return P.Problem(name=f"r3d_{nx}x{ny}x{nz}", kind="stencil3d", n=n, b=b, l=l, u=u,
                     x0=P.gaussian(seed, 8, n) * 0.1, tol=-1e-10, nx=nx, ny=ny, nz=nz, wx=wx, wy=wy, wz=wz,
                     shift=sh)


R3D_CASES = {
    "31x7x33": lambda: ragged_stencil3d(31, 7, 33, 11),
    "45x13x65_sb": lambda: ragged_stencil3d(45, 13, 65, 12, shift=False, bounds="scalar"),
    "1x1x9": lambda: ragged_stencil3d(1, 1, 9, 13),
    "2x3x1": lambda: ragged_stencil3d(2, 3, 1, 14),
    "61x6x5_sb": lambda: ragged_stencil3d(61, 6, 5, 15, bounds="scalar"),
}


@pytest.mark.parametrize("generic", ["0", "1"])   # plane-march kernels (march3.cuh) / generic kernels
@pytest.mark.parametrize("case", list(R3D_CASES))
def test_stencil3d_ragged_parity(G, oracle, monkeypatch, case, generic):
    monkeypatch.setenv("GPCG_GENERIC", generic)
    prob = R3D_CASES[case]()
    A = oracle.problem_csr(prob)
    p = 2.0 * P.uniform(98, 1, prob.n) - 1.0
    with G.Solver.from_problem(prob) as s:
        spmv_close(s.hessvec(p), oracle.spmv(A, p), abs_op(A, p))
        rc, x, st = s.solve(prob.x0, prob.tol)
        yr = s.hessvec(p, reduced=True)
        for pc in (1,):
            s.set_params(precond=pc)
            rc1, x1, st1 = s.solve(prob.x0, prob.tol)
    free = (x > prob.l) & (x < prob.u)
    spmv_close(yr, oracle.spmv_masked(A, free, p), abs_op(A, p * free))
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=prob.tol)
    assert rc == 0 and rc_o == 0 and rc1 == 0
    for xx, stt in ((x, st), (x1, st1)):
        assert abs(stt["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
        assert np.max(np.abs(xx - x_o)) <= 1e-7
    nm, nontie = _tie_mismatches(x, x_o, prob.l, prob.u)
    assert not nontie


def test_stencil3d_march_first_outer_iteration_matches_generic(G, monkeypatch):
    """One outer iteration through the plane-march kernels and through the generic kernels:
    the same per-point arithmetic, so the same GP / CG iteration counts and x to rounding."""
    prob = ragged_stencil3d(47, 19, 41, 16)
    out = {}
    for generic in ("0", "1"):
        monkeypatch.setenv("GPCG_GENERIC", generic)
        with G.Solver.from_problem(prob) as s:
            s.set_params(refine_cap=1)
            rc, x, st = s.solve(prob.x0, prob.tol, max_it=1)
        out[generic] = (x, st)
    (x0, st0), (x1, st1) = out["0"], out["1"]
    assert st0["gp_iters"] == st1["gp_iters"] and st0["cg_iters"] == st1["cg_iters"]
    assert np.max(np.abs(x0 - x1)) <= 1e-12 * np.max(np.abs(x1))


def test_stencil3d_full_c4_matches_csr_golden(G):
    """Full-size C4 (256^3) through gpcg_create_stencil3d against the oracle's CSR golden:
    the same matrix (face assembly == the edge-list CSR, pinned in test_oracle_pins)."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "oracle_C4.json")
    gold = json.load(open(path))
    prob = P.c4_stencil_family(m=256)
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(prob.x0, gold["tol"])
    assert rc == 0
    assert abs(st["q"] - gold["q"]) <= 1e-10 * abs(gold["q"])
    idx = np.asarray(gold["idx"])
    assert np.max(np.abs(x[idx] - np.asarray(gold["x"]))) <= 1e-7


# ------------------------------------------------------------------ edge grids for the band kernels
# (bands of 112 / 104 columns, row segments, persistent cooperative loops): widths that leave a
# partial band, a single column / row, fewer rows than a pipeline block.
@pytest.mark.parametrize("nx,ny", [(1, 37), (37, 1), (2, 2), (113, 9), (105, 41), (230, 3), (224, 17)])
def test_band_kernels_edge_grids(G, oracle, nx, ny):
    prob = P.journal_bearing(nx, ny, eps=0.5)
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=-1e-12)
    for pc in (0, 1):
        with G.Solver.from_problem(prob) as s:
            s.set_params(precond=pc)
            rc, x, st = s.solve(prob.x0, -1e-12)
            p = 2.0 * P.uniform(95, 1, prob.n) - 1.0
            y = s.hessvec(p)
            yr = s.hessvec(p, reduced=True)
            if prob.nx % 32 == 0:                         # device pointers: the map is built on the input
                import torch
                pd = torch.from_numpy(p).cuda()
                yd = s.hessvec(pd, reduced=True).cpu().numpy()
                assert np.array_equal(yd, yr)
        assert rc == 0 and rc_o == 0, (rc, st)
        A = oracle.problem_csr(prob)
        spmv_close(y, oracle.spmv(A, p), abs_op(A, p))
        free = (x > prob.l) & (x < prob.u)
        spmv_close(yr, oracle.spmv_masked(A, free, p), abs_op(A, p * free))
        assert abs(st["q"] - st_o["q"]) <= 1e-10 * max(abs(st_o["q"]), 1e-300)
        assert np.max(np.abs(x - x_o)) <= 1e-7


# ------------------------------------------------------------------ extraction ablation (NEXT-4)
@pytest.mark.parametrize("case", ["C0", "C1", "c4_family_m16", "ragged37x23", "dense8", "jb80_eps0.9"])
def test_solve_parity_explicit_extraction(G, oracle, case):
    """cg_mode = 1: A_k extracted as a compact CSR matrix each CG call (the paper's PETSc
    route) reaches the oracle's solution too, with and without the Jacobi preconditioner."""
    make, tol = SOLVE_CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    for pc in (0, 1):
        with G.Solver.from_problem(prob) as s:
            s.set_params(cg_mode=1, precond=pc)
            rc, x, st = s.solve(prob.x0, tol)
        assert rc == 0, (rc, st)
        assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
        assert np.max(np.abs(x - x_o)) <= 1e-7
        assert st["cg_iters"] == 0 or st["t_extract_ms"] > 0.0


def test_explicit_extraction_same_cg_iterates(G):
    """The compact CG runs the same recurrences on the same numbers (A_F's rows in the
    operator's neighbour order): one CG call from the same point gives w to rounding."""
    prob = P.c1()
    out = {}
    for mode in (0, 1):
        with G.Solver.from_problem(prob) as s:
            s.set_params(cg_mode=mode, cg_cap=40, eta2=1e-10, refine_cap=1)
            rc, x, st = s.solve(prob.x0, -1e-12, max_it=1)
        out[mode] = (x, st)
    x0, st0 = out[0]
    x1, st1 = out[1]
    assert st0["cg_iters"] == st1["cg_iters"] and st0["gp_iters"] == st1["gp_iters"]
    assert np.max(np.abs(x0 - x1)) <= 1e-10 * np.max(np.abs(x0))


# ------------------------------------------------------------------ block-Jacobi ILU(0) PCG (NEXT-3)
BJ_CASES = ["C0", "C1", "jb80_eps0.9", "c3_family_160", "ragged37x23"]


def _bj_params(oracle, prob):
    return oracle.default_params(precond=2, grid_nx=prob.nx, grid_ny=prob.ny, tile_x=32, tile_y=32)


@pytest.mark.parametrize("generic", ["0", "1"])   # PCG matvec: column march (k2) / generic kernel
@pytest.mark.parametrize("case", BJ_CASES)
def test_solve_parity_bjilu(G, oracle, monkeypatch, case, generic):
    monkeypatch.setenv("GPCG_GENERIC", generic)
    make, tol = SOLVE_CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol, params=_bj_params(oracle, prob))
    assert rc_o == 0
    with G.Solver.from_problem(prob) as s:
        s.set_params(precond=2)
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0, (rc, st)
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7
    nm, nontie = _tie_mismatches(x, x_o, prob.l, prob.u)
    assert not nontie


@pytest.mark.parametrize("case", ["C0", "ragged37x23"])
def test_bjilu_first_outer_iteration_matches_oracle(G, oracle, case):
    """One outer iteration (GP phase + one block-Jacobi ILU(0) PCG call + search) on the GPU
    and in the oracle: the same algorithm on the same numbers, equal to rounding; and fewer
    CG iterations than the point-Jacobi PCG from the same point."""
    make, tol = SOLVE_CASES[case]
    prob = make()
    prm = _bj_params(oracle, prob)
    prm.refine_cap = 1
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol, max_it=1, params=prm)
    with G.Solver.from_problem(prob) as s:
        s.set_params(precond=2, refine_cap=1)
        rc, x, st = s.solve(prob.x0, tol, max_it=1)
    assert st["gp_iters"] == st_o["gp_iters"] and st["cg_iters"] == st_o["cg_iters"]
    assert np.max(np.abs(x - x_o)) <= 1e-9 * max(np.max(np.abs(x_o)), 1e-300)
    with G.Solver.from_problem(prob) as s:
        s.set_params(precond=1, refine_cap=1)
        rc1, x1, st1 = s.solve(prob.x0, tol, max_it=1)
    assert st["cg_iters"] <= st1["cg_iters"]


# ------------------------------------------------------------------ block-Jacobi ILU(2) PCG (NEXT-3, the paper's
# subdomain solver)
def _bj2_params(oracle, prob, **kw):
    return oracle.default_params(precond=3, ilu_level=2, grid_nx=prob.nx, grid_ny=prob.ny, tile_x=32, tile_y=32,
                                 **kw)


@pytest.mark.parametrize("case", BJ_CASES)
def test_solve_parity_bjilu2(G, oracle, case):
    make, tol = SOLVE_CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol, params=_bj2_params(oracle, prob))
    assert rc_o == 0
    with G.Solver.from_problem(prob) as s:
        s.set_params(precond=3)
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0, (rc, st)
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7
    nm, nontie = _tie_mismatches(x, x_o, prob.l, prob.u)
    assert not nontie


@pytest.mark.parametrize("case", ["C0", "ragged37x23", "jb80_eps0.9"])
def test_bjilu2_first_outer_iteration_matches_oracle(G, oracle, case):
    """One outer iteration (GP phase + one block-Jacobi ILU(2) PCG call + search): the same
    algorithm on the same numbers as the oracle's generic ILU(k), equal to rounding; and no
    more CG iterations than ILU(0) from the same point (Table 4)."""
    make, tol = SOLVE_CASES[case]
    prob = make()
    prm = _bj2_params(oracle, prob, refine_cap=1)
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol, max_it=1, params=prm)
    with G.Solver.from_problem(prob) as s:
        s.set_params(precond=3, refine_cap=1)
        rc, x, st = s.solve(prob.x0, tol, max_it=1)
    assert st["gp_iters"] == st_o["gp_iters"] and st["cg_iters"] == st_o["cg_iters"], (st, st_o)
    assert np.max(np.abs(x - x_o)) <= 1e-9 * max(np.max(np.abs(x_o)), 1e-300)
    with G.Solver.from_problem(prob) as s:
        s.set_params(precond=2, refine_cap=1)
        rc0, x0, st0 = s.solve(prob.x0, tol, max_it=1)
    assert st["cg_iters"] <= st0["cg_iters"]


def test_bjilu_rejected_for_csr(G):
    prob = dense_problem(8, 21)
    with G.Solver.from_problem(prob) as s:
        s.set_params(precond=2)
        rc, x, st = s.solve(prob.x0, -1e-10, allow_error=True)
    assert rc == G.EINVAL


# ------------------------------------------------------------------ compacted free-row list
COMPACT_CASES = {"c4_family_m16": lambda: P.c4_family(m=16), "c4_family_m24": lambda: P.c4_family(m=24),
                 "c4s_family_16": lambda: P.c4_stencil_family(m=16), "dense8": lambda: dense_problem(8, 21)}


@pytest.mark.parametrize("case", list(COMPACT_CASES))
def test_compact_free_rows_solve_and_hessvec(G, oracle, case):
    """cg_mode 3 (CG applied in place over the compacted free-row list) and the default (2)
    reach the oracle's solution; the reduced HVP over the list equals ora_spmv_masked on the
    recorded free set (the masked full-length kernel, cg_mode 0, beside it)."""
    prob = COMPACT_CASES[case]()
    tol = -1e-11
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    A = oracle.problem_csr(prob)
    p = 2.0 * P.uniform(77, 1, prob.n) - 1.0
    for mode in (3, 2, 0):
        with G.Solver.from_problem(prob) as s:
            s.set_params(cg_mode=mode)
            rc, x, st = s.solve(prob.x0, tol)
            yr = s.hessvec(p, reduced=True)
        assert rc == 0 and rc_o == 0, (mode, rc, st)
        assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
        assert np.max(np.abs(x - x_o)) <= 1e-7
        free = (x > prob.l) & (x < prob.u)
        spmv_close(yr, oracle.spmv_masked(A, free, p), abs_op(A, p * free))


def test_compact_free_rows_same_cg_iterates(G):
    """One CG call from the same point over the free-row list and over the masked full-length
    vectors: the same recurrences on the same numbers -> the same w to rounding."""
    prob = P.c4_family(m=24)
    out = {}
    for mode in (0, 3):
        with G.Solver.from_problem(prob) as s:
            s.set_params(cg_mode=mode, cg_cap=30, eta2=1e-10, refine_cap=1)
            rc, x, st = s.solve(prob.x0, -1e-12, max_it=1)
        out[mode] = (x, st)
    (x0, st0), (x3, st3) = out[0], out[3]
    assert st0["cg_iters"] == st3["cg_iters"] and st0["gp_iters"] == st3["gp_iters"]
    assert np.max(np.abs(x0 - x3)) <= 1e-12 * np.max(np.abs(x0))


HVFREE_CASES = {**COMPACT_CASES, "dense40": lambda: dense_problem(40, 3), "c4_family_m7": lambda: P.c4_family(m=7),
                "c4s_family_9": lambda: P.c4_stencil_family(m=9)}


def check_hessvec_free(G, oracle, s, prob, A, x, p):
    """gpcg_hessvec_free at the free set of P[x] vs ora_spmv_masked on that set (1e-13), and vs
    the full-length reduced product at the free rows (bitwise where that product also runs over
    the free-row list: |F| < 0.3 n)."""
    import torch
    px, pg2, na, nnb = s.project(x)
    free = (px > prob.l) & (px < prob.u)
    m = int(free.sum())
    assert s.free_count() == m
    yf = s.hessvec_free(p)
    assert yf.shape == (m,)
    yr = s.hessvec(p, reduced=True)
    if m == 0:
        assert not np.any(yr)
        return m
    yref = oracle.spmv_masked(A, free, p)
    spmv_close(yf, yref[free], abs_op(A, p * free)[free])
    if 10 * m < 3 * prob.n:
        assert np.array_equal(yf, yr[free])
    else:
        spmv_close(yf, yr[free], abs_op(A, p * free)[free])
    yd = s.hessvec_free(torch.from_numpy(p).cuda())       # device in / out: same kernel, same bits
    assert np.array_equal(yd.cpu().numpy(), yf)
    return m


@pytest.mark.parametrize("case", list(HVFREE_CASES))
def test_hessvec_free_compact_output(G, oracle, case):
    """the reduced product written in the reduced space (|F| entries, the
    CSR-vector row groups for CSR, one thread per free row for the 3-D stencil) at a small, a
    mid-size, an empty and the full free set; ESTATE before any free set is recorded."""
    prob = HVFREE_CASES[case]()
    A = oracle.problem_csr(prob)
    p = 2.0 * P.uniform(78, 1, prob.n) - 1.0
    fl, fu = np.isfinite(prob.l), np.isfinite(prob.u)
    span = np.where(fl & fu, prob.u - prob.l, 1.0)
    mid = np.where(fl & fu, 0.5 * (prob.l + prob.u),
                   np.where(fl, prob.l + 0.5, np.where(fu, prob.u - 0.5, 0.0)))
    with G.Solver.from_problem(prob) as s:
        assert s.free_count() == -1
        with pytest.raises(G.GpcgError) as e:
            s.hessvec_free(p)
        assert e.value.code == G.ESTATE
        ms = []
        for scale in (4.0, 0.9):          # x = mid + scale * (span / 2) * N(0, 1): most / few active
            x = mid + scale * 0.5 * span * P.gaussian(79, 2, prob.n)
            ms.append(check_hessvec_free(G, oracle, s, prob, A, x, p))
        assert ms[0] < ms[1]
        # every point at a bound -> |F| = 0 (when every point has one); every point free
        if np.all(fl | fu):
            out = np.where(fu, prob.u + 1.0, prob.l - 1.0)
            assert check_hessvec_free(G, oracle, s, prob, A, out, p) == 0
        assert check_hessvec_free(G, oracle, s, prob, A, mid, p) == prob.n


def test_hessvec_free_c4_full_size(G, oracle):
    """C4 (256^3 CSR, BASELINE.json configs[4]) at full size: the compact reduced product at a
    ~5 %-free set, every one of its |F| outputs vs ora_spmv_masked."""
    prob = P.c4()
    A = oracle.problem_csr(prob)
    p = 2.0 * P.uniform(80, 1, prob.n) - 1.0
    x = 0.0125 * P.gaussian(81, 2, prob.n)             # |x| < 0.01 (free) for ~58 %; 1/20 of that
    x[P.uniform(82, 3, prob.n) > 0.09] = 1.0            # ~5 % free, scattered like C4's solution
    with G.Solver.from_problem(prob) as s:
        m = check_hessvec_free(G, oracle, s, prob, A, x, p)
    assert 0.02 * prob.n < m < 0.08 * prob.n


# ------------------------------------------------------------------ CG sweep stage layouts (band / per-warp boxes)
@pytest.mark.parametrize("pw", ["0", "1"])
@pytest.mark.parametrize("case", ["C0", "jb80_eps0.9", "c3_family_160"])
def test_cg_sweep_box_layouts(G, oracle, monkeypatch, case, pw):
    """The persistent CG sweep with band boxes and with per-warp boxes (+ per-warp skip flags;
    the default for grids whose CG vectors exceed L2): same solution as the oracle, and the
    same CG iterates as each other from the same point."""
    monkeypatch.setenv("GPCG_CG_PW", pw)
    make, tol = SOLVE_CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    with G.Solver.from_problem(prob) as s:
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0 and rc_o == 0, (rc, st)
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7
    for slabs in (1, 2):
        with G.Solver.from_problem(prob, slabs=slabs) as s:
            s.set_params(cg_cap=25, eta2=1e-10, refine_cap=1)
            rc1, x1, st1 = s.solve(prob.x0, tol, max_it=1)
        monkeypatch.setenv("GPCG_CG_PW", "1" if pw == "0" else "0")
        with G.Solver.from_problem(prob, slabs=slabs) as s:
            s.set_params(cg_cap=25, eta2=1e-10, refine_cap=1)
            rc2, x2, st2 = s.solve(prob.x0, tol, max_it=1)
        monkeypatch.setenv("GPCG_CG_PW", pw)
        assert st1["cg_iters"] == st2["cg_iters"]
        assert np.array_equal(x1, x2)


# ------------------------------------------------------------------ speculative GP step of the generic operators
SPEC_CASES = {"c4_family_m16": (lambda: P.c4_family(m=16), -1e-11),
              "c4s_family_16": (lambda: P.c4_stencil_family(m=16), -1e-11),
              "dense40": (lambda: dense_problem(40, 3), -1e-12),
              "c4_family_m24_jacobi": (lambda: P.c4_family(m=24), -1e-11)}


@pytest.mark.parametrize("case", list(SPEC_CASES))
def test_generic_speculative_gp_step(G, oracle, monkeypatch, case):
    """k_spec (CSR / 3-D: the h = 0 step of each GP step and of the CG phase -- search sums and
    accepted point in one sweep, each with the arithmetic of k_search / k_accept) against the
    search + accept sweeps (GPCG_GP_SPEC=0): the oracle's solution, and bit for bit the same
    iterate and iteration counts, with one and with two slabs."""
    make, tol = SPEC_CASES[case]
    prob = make()
    pc = 1 if case.endswith("jacobi") else 0
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    out = {}
    for spec in ("0", "1"):
        monkeypatch.setenv("GPCG_GP_SPEC", spec)
        for slabs in (1, 2):
            if slabs > 1 and case == "dense40":
                continue
            with G.Solver.from_problem(prob, slabs=slabs) as s:
                s.set_params(precond=pc)
                rc, x, st = s.solve(prob.x0, tol)
            assert rc == 0 and rc_o == 0, (spec, slabs, st)
            assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
            assert np.max(np.abs(x - x_o)) <= 1e-7
            nm, nontie = _tie_mismatches(x, x_o, prob.l, prob.u)
            assert not nontie
            out[(spec, slabs)] = (x, st)
    for slabs in (1, 2):
        if ("1", slabs) not in out:
            continue
        (x1, st1), (x0, st0) = out[("1", slabs)], out[("0", slabs)]
        assert np.array_equal(x1, x0)
        for k in ("outer_iters", "gp_iters", "cg_iters", "q"):
            assert st1[k] == st0[k], k


@pytest.mark.parametrize("device", [False, True])
@pytest.mark.parametrize("slabs", [1, 2])
def test_csr_create_validation(G, device, slabs):
    """gpcg_create_csr rejects a non-monotone row_ptr, a column outside [0, n) and a non-finite
    value (EINVAL) -- on the one-slab path (arrays uploaded as given, checked by k_check_csr /
    k_count_nonfinite) and the slab path (host checks) -- from host and from device arrays; the
    valid matrix creates and solves."""
    import torch
    prob = dense_problem(12, 5)
    bad = {"rp": lambda: (np.concatenate([prob.row_ptr[:3], [prob.row_ptr[2] - 1], prob.row_ptr[4:]]),
                          prob.col, prob.val),
           "col": lambda: (prob.row_ptr, np.where(np.arange(prob.col.size) == 7, 12, prob.col).astype(np.int32),
                           prob.val),
           "val": lambda: (prob.row_ptr, prob.col, np.where(np.arange(prob.val.size) == 9, np.nan, prob.val))}

    def make(rp, ci, va):
        if device:
            rp, ci, va = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (rp, ci, va))
        if slabs == 1:
            return G.Solver.csr(prob.n, rp, ci, va, prob.b, prob.l, prob.u)
        p2 = P.Problem(**{**prob.__dict__})
        p2.row_ptr, p2.col, p2.val = (np.asarray(a.cpu() if hasattr(a, "cpu") else a) for a in (rp, ci, va))
        return G.Solver.from_problem(p2, slabs=slabs)
    for what, f in bad.items():
        with pytest.raises(G.GpcgError) as e:
            make(*f())
        assert e.value.code == G.EINVAL, what
    with make(prob.row_ptr, prob.col, prob.val) as s:
        rc, x, st = s.solve(prob.x0, -1e-10)
    assert rc == 0
