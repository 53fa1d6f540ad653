"""The multi-rank code path (row slabs, ghost-row halo exchange,
per-slab partial sums combined in a fixed order, k_finalize on the global
totals) on ONE GPU: gpcg_dist.local_slabs splits the problem into slabs whose
halos are device copies -- the same kernels, exchange schedule and deferred
reductions a multi-GPU run issues, with NCCL replaced by copies (the profiling
guide forbids emulating ranks that wait on one another on one GPU; nothing here
waits).  Compared with the CPU oracle on the same seeded inputs and with the
single-slab solve."""
import numpy as np
import pytest

from paper_cs_0101018_b200 import problems as P
from tests.test_gpu_parity import G, abs_op, dense_problem, ragged_stencil, spmv_close, _tie_mismatches  # noqa: F401

pytestmark = pytest.mark.gpu

CASES = {
    "C0": (lambda: P.c0(), -1e-12),
    "C1": (lambda: P.c1(), -1e-11),
    "ragged37x23_full_shift": (lambda: ragged_stencil(37, 23, 5), -1e-12),
    "ragged29x17_bcast": (lambda: ragged_stencil(29, 17, 6, full=False, shift=False), -1e-12),
    "c3_family_160": (lambda: P.c3_family(160, 160), -1e-11),
    "c4_family_m12": (lambda: P.c4_family(m=12), -1e-11),
    "dense12": (lambda: dense_problem(12, 31), -1e-12),
}


@pytest.mark.parametrize("slabs", [2, 3, 5])
@pytest.mark.parametrize("case", list(CASES))
def test_slab_solve_parity(G, oracle, case, slabs):
    make, tol = CASES[case]
    prob = make()
    rows = prob.ny if prob.kind == "stencil2d" else prob.n
    if rows < 2 * slabs:
        pytest.skip("too few rows for this many slabs")
    if case == "dense12" and slabs > 2:
        # a dense row reaches every row: beyond the neighbouring slab -> documented EINVAL
        with pytest.raises(G.GpcgError) as e:
            G.Solver.from_problem(prob, slabs=slabs)
        assert e.value.code == G.EINVAL
        return
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    with G.Solver.from_problem(prob, slabs=slabs) as s:
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0 and rc_o == 0, (rc, st)
    assert np.all(x >= prob.l) and np.all(x <= prob.u)
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7
    nm, nontie = _tie_mismatches(x, x_o, prob.l, prob.u)
    assert not nontie
    A = oracle.problem_csr(prob)
    pg = np.linalg.norm(oracle.proj_grad(x, oracle.gradient(A, prob.b, x), prob.l, prob.u))
    assert pg <= 1.01 * st["tau"] + 1e-15


@pytest.mark.parametrize("case", ["C1", "ragged37x23_full_shift", "ragged29x17_bcast", "c4_family_m12"])
def test_slab_spmv_project(G, oracle, case):
    prob = CASES[case][0]()
    A = oracle.problem_csr(prob)
    p = 2.0 * P.uniform(98, 1, prob.n) - 1.0
    with G.Solver.from_problem(prob, slabs=3) as s:
        y = s.hessvec(p)
        spmv_close(y, oracle.spmv(A, p), abs_op(A, p))
        px, pg2, na, nnb = s.project(prob.x0)
        pref = oracle.project(prob.l, prob.u, prob.x0)
        assert np.array_equal(px, pref)
        g = oracle.gradient(A, prob.b, pref)
        act, bnd, na_ref, nb_ref = oracle.sets(pref, g, prob.l, prob.u)
        assert na == na_ref and nnb == na_ref - nb_ref
        free = ~act
        yr = s.hessvec(p, reduced=True)
        spmv_close(yr, oracle.spmv_masked(A, free, p), abs_op(A, p * free))
        q = s.objective(prob.x0)
        qref = oracle.objective(A, prob.b, prob.c, prob.x0)
        assert abs(q - qref) <= 1e-12 * max(abs(qref), 1e-300)


def test_slab_matches_single_slab_iterates(G):
    """Same iterates up to reduction order: identical outer/GP counts on C0, q to 1e-12."""
    prob = P.c0()
    with G.Solver.from_problem(prob) as s1:
        rc1, x1, st1 = s1.solve(prob.x0, -1e-10)
    with G.Solver.from_problem(prob, slabs=4) as s4:
        rc4, x4, st4 = s4.solve(prob.x0, -1e-10)
    assert rc1 == rc4 == 0
    assert abs(st1["q"] - st4["q"]) <= 1e-12 * abs(st1["q"])
    assert np.max(np.abs(x1 - x4)) <= 1e-9


def test_slab_errors(G):
    prob = ragged_stencil(9, 3, 2)
    with pytest.raises(G.GpcgError) as e:
        G.Solver.from_problem(prob, slabs=2)          # a slab of < 2 stencil rows
    assert e.value.code == G.EINVAL


@pytest.mark.parametrize("case", ["C1", "c4_family_m12", "ragged37x23_full_shift"])
def test_slab_pcg_parity(G, oracle, case):
    make, tol = CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol, params=oracle.default_params(precond=1))
    with G.Solver.from_problem(prob, slabs=3) as s:
        s.set_params(precond=1)
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0 and rc_o == 0
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7


@pytest.mark.parametrize("slabs", [2, 3])
def test_slab_stencil3d_parity(G, oracle, slabs):
    prob = P.c4_stencil_family(m=10)
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=-1e-11)
    with G.Solver.from_problem(prob, slabs=slabs) as s:
        rc, x, st = s.solve(prob.x0, -1e-11)
        p = 2.0 * P.uniform(96, 1, prob.n) - 1.0
        y = s.hessvec(p)
    A = oracle.problem_csr(prob)
    spmv_close(y, oracle.spmv(A, p), abs_op(A, p))
    assert rc == 0 and rc_o == 0
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7


@pytest.mark.parametrize("case", ["C0", "c3_family_160", "ragged29x17_bcast", "ragged37x23_full_shift", "c4_family_m12"])
def test_slab_first_outer_iteration_matches_single_slab(G, case):
    """One outer iteration (GP phase, CG, projected search) on 1 slab and on 3 slabs must agree
    to rounding: every sweep must see the true neighbour values across slab edges (ghost rows
    deep enough for the operator applications a sweep chains -- a missing ghost row shows up
    as a wrong Cauchy step alpha_0 at the slab boundary and a visibly different iterate)."""
    prob = CASES[case][0]()
    # one CG iteration per CG call: the iterate is then dominated by the GP phase, whose
    # steps differ between slab counts only by the reduction order (~1e-16 relative) -- a
    # Krylov run would amplify those rounding differences and hide a real discrepancy
    with G.Solver.from_problem(prob) as s1:
        s1.set_params(cg_cap=1)
        rc1, x1, st1 = s1.solve(prob.x0, -1e-12, max_it=1)
    with G.Solver.from_problem(prob, slabs=3) as s3:
        s3.set_params(cg_cap=1)
        rc3, x3, st3 = s3.solve(prob.x0, -1e-12, max_it=1)
    assert (st1["gp_iters"], st1["cg_iters"]) == (st3["gp_iters"], st3["cg_iters"])
    scale = max(np.max(np.abs(x1)), 1e-300)
    assert np.max(np.abs(x1 - x3)) <= 1e-12 * scale, np.max(np.abs(x1 - x3)) / scale


@pytest.mark.parametrize("slabs", [1, 2])
@pytest.mark.parametrize("case", ["C0", "C1", "c4_family_m12"])
def test_nccl_collectives_one_rank(G, oracle, monkeypatch, case, slabs):
    """The NCCL path on one GPU: GPCG_FORCE_NCCL=1 gives the handle a 1-rank communicator, so
    every global sum is an ncclAllReduce (inside the captured CG / GP graphs) and the create-time
    broadcasts go through ncclBroadcast, with the deferred k_finalize decisions -- the collective
    sequence of a multi-rank run, minus the send/recv halos (no neighbouring rank)."""
    monkeypatch.setenv("GPCG_FORCE_NCCL", "1")
    make, tol = CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    with G.Solver.from_problem(prob, slabs=slabs) as s:
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0 and rc_o == 0, (rc, st)
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7


@pytest.mark.parametrize("precond", [2, 3])
@pytest.mark.parametrize("case", ["C0", "ragged37x23_full_shift"])
def test_slab_bjilu_reaches_the_minimiser(G, oracle, case, precond):
    """Block-Jacobi ILU with blocks inside each slab (the paper's one block per processor,
    here tiles per slab): a different preconditioner per slab layout, the same x*."""
    make, tol = CASES[case]
    prob = make()
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    with G.Solver.from_problem(prob, slabs=2) as s:
        s.set_params(precond=precond)
        rc, x, st = s.solve(prob.x0, tol)
    assert rc == 0 and rc_o == 0
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7


@pytest.mark.parametrize("slabs", [2, 4])
def test_multi_slab_persistent_loops_match_single_slab_per_step(G, slabs):
    """The multi-slab persistent CG / GP loops (one launch over every slab, fused halo writes):
    one outer iteration with a short GP phase and a fixed-length CG call gives the single-slab
    iterate to rounding (only the order of the partial sums differs)."""
    prob = P.c3_family(160, 160)
    out = {}
    for ns in (1, slabs):
        with G.Solver.from_problem(prob, slabs=ns) as s:
            s.set_params(gp_cap=6, cg_cap=12, eta2=1e-12, refine_cap=1)
            rc, x, st = s.solve(prob.x0, -1e-14, max_it=1)
        out[ns] = (x, st)
    (x1, st1), (xs, sts) = out[1], out[slabs]
    assert (st1["gp_iters"], st1["cg_iters"]) == (sts["gp_iters"], sts["cg_iters"])
    assert st1["cg_iters"] == 12 and st1["gp_iters"] >= 2
    assert np.max(np.abs(x1 - xs)) <= 1e-11 * max(np.max(np.abs(x1)), 1e-300)


@pytest.mark.parametrize("sys_scope", ["0", "1"])
@pytest.mark.parametrize("slabs", [2, 3, 5, 8])
@pytest.mark.parametrize("case", ["C0", "ragged29x17_bcast", "c3_family_160"])
def test_cross_rank_protocol_emulated(G, oracle, monkeypatch, case, slabs, sys_scope):
    """The cross-rank protocol of the persistent loops (march_tma.cuh XRank: per-rank arrival
    counters never reset, partials stored into every rank's mailbox, each rank summing its own
    copy in global CTA order, the mailbox slot from the global barrier count) run inside one
    cooperative launch with every slab a virtual rank (GPCG_XRANK_EMU=1): bit for bit the
    one-device multi-slab loops, over every launch of a solve and of a second solve on the same
    handle (counters and bases carried across launches), and the oracle's solution.  sys_scope = 1
    (GPCG_XRANK_SYS): the leaders' operations at system scope and the entry barrier of every
    launch, as ranks on several devices run them."""
    if sys_scope == "1" and slabs in (3, 5):
        pytest.skip("system scope: 2 and 8 virtual ranks")
    monkeypatch.setenv("GPCG_XRANK_SYS", sys_scope)
    make, tol = CASES[case]
    prob = make()
    if prob.ny < 3 * slabs:
        pytest.skip("too few rows for this many slabs (3 ghost rows)")
    res = {}
    for emu in ("0", "1"):
        monkeypatch.setenv("GPCG_XRANK_EMU", emu)
        with G.Solver.from_problem(prob, slabs=slabs) as s:
            r1 = s.solve(prob.x0, tol)
            r2 = s.solve(prob.x0, tol)
        res[emu] = (r1, r2)
    (a1, a2), (b1, b2) = res["0"], res["1"]
    for (rc, x, st), (rcb, xb, stb) in ((a1, b1), (a2, b2), (b1, b2)):
        assert rc == 0 and rcb == 0, (st, stb)
        assert np.array_equal(x, xb)
        for k in ("outer_iters", "gp_iters", "cg_iters"):
            assert st[k] == stb[k], k
    assert b1[2]["cg_iters"] > 0 and b1[2]["gp_iters"] > 1
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    rc, x, st = b1
    assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
    assert np.max(np.abs(x - x_o)) <= 1e-7


def test_xrank_switch_single_rank(G, oracle, monkeypatch):
    """GPCG_XRANK=1 on one rank: nothing spans ranks, but the handle's arenas come from cudaMalloc
    (IPC-exportable) instead of the memory pool -- the same solution, bit for bit."""
    prob = P.c0()
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("GPCG_XRANK", v)
        with G.Solver.from_problem(prob, slabs=2) as s:
            out.append(s.solve(prob.x0, -1e-12))
    (rc0, x0, st0), (rc1, x1, st1) = out
    assert rc0 == rc1 == 0 and np.array_equal(x0, x1) and st0["cg_iters"] == st1["cg_iters"]


@pytest.mark.parametrize("mode", ["1slab", "2slabs", "2slabs_nccl"])
@pytest.mark.parametrize("case", ["C0", "ragged29x17_bcast", "c3_family_160"])
def test_gp_graph_speculative_step(G, oracle, monkeypatch, case, mode):
    """The 2-D GP graph chunks (the ranks' path: GPCG_GP_PERSIST=0 here) take each step with
    k5_spec (the persistent loop's speculative sweep as one node; search / accept only when it is
    rejected): the oracle's solution with and without it (GPCG_GP_SPEC=0), one slab, two slabs
    with deferred reductions, and two slabs with every sum through a 1-rank NCCL communicator."""
    make, tol = CASES[case]
    prob = make()
    monkeypatch.setenv("GPCG_GP_PERSIST", "0")
    if mode == "2slabs_nccl":
        monkeypatch.setenv("GPCG_FORCE_NCCL", "1")
    slabs = 1 if mode == "1slab" else 2
    rc_o, x_o, st_o = oracle.solve_problem(prob, tol=tol)
    for spec in ("1", "0"):
        monkeypatch.setenv("GPCG_GP_SPEC", spec)
        with G.Solver.from_problem(prob, slabs=slabs) as s:
            rc, x, st = s.solve(prob.x0, tol)
        assert rc == 0 and rc_o == 0, (spec, st)
        assert abs(st["q"] - st_o["q"]) <= 1e-10 * abs(st_o["q"])
        assert np.max(np.abs(x - x_o)) <= 1e-7
        nm, nontie = _tie_mismatches(x, x_o, prob.l, prob.u)
        assert not nontie
