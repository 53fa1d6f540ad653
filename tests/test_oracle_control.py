"""Pin the oracle's CONTROL PATH: the GP-phase stop rules and the eta2 refinement.

The solution x* is unique, so the pins on x alone (enumeration, Cholesky,
KKT) do not see the rules that only change the path: Eq. pgstop1, Eq. pgstop2
(P:386-388), the GP-phase safety net (reading R13) and the "reduce eta2 and continue" of
Eq. cgstop3 (reading R12).  These tests check them against
  * SPEC.md's GP-phase examples: an unchanged active set stops the phase after
    one iterate; with no bounds the first step is steepest descent with
    alpha = g'g / g'Ag, always accepted at h = 0 (mu <= 1/2), decreasing q by (g'g)^2/(2 g'Ag);
  * an independent dense numpy transcription of Algorithm GPCG (tests/_brute.py,
    gpcg_dense_trace: CG on the extracted free block, dense products), compared record by
    record on the oracle's control-path trace (oracle/gpcg_oracle.c, trace_put): every GP
    step (j, h, decrease, alpha), every phase end (steps, stop reason), every CG call
    (rep, iterations, eta2, |F|) and every CG search (h, decrease, |A \\ B|);
  * the closed form of the eta2 sequence within an outer iteration (R12):
    eta2 at repetition r = max(0.05 * 0.1^r, 1e-12).
scripts/oracle_mutants.py checks that each plausible mistake in these rules (pgstop1
dropped / always true, pgstop2 with eta2, eta2 never reduced, cgstop3 inverted) fails here.
"""
import numpy as np
import pytest

from tests import _brute as B

# trace record kinds (gpcg_oracle.c)
GP_STEP, GP_END, CG_CALL, CG_SEARCH = 1, 2, 3, 4
R_CONV, R_PGSTOP1, R_PGSTOP2, R_CAP = 0, 1, 2, 3


def csr_of(O, A):
    n = A.shape[0]
    rp, ci, va = [0], [], []
    for i in range(n):
        for j in range(n):
            if A[i, j] != 0.0:
                ci.append(j)
                va.append(A[i, j])
        rp.append(len(ci))
    return O.CSR(n, np.array(rp, np.int64), np.array(ci, np.int32), np.array(va))


def instance(seed):
    """Seeded small QPs of three shapes: 2-D grid M-matrices with obstacle-like bounds (the
    paper's problem class), sparse random SPD with mixed finite / infinite bounds,
    and ill-conditioned tridiagonal M-matrices with l = 0, u = inf."""
    r = np.random.default_rng(seed)
    kind = seed % 3
    if kind == 0:
        nx, ny = int(r.integers(3, 9)), int(r.integers(3, 9))
        n = nx * ny
        A = np.zeros((n, n))
        for j in range(ny):
            for i in range(nx):
                v = i + nx * j
                for di, dj in ((1, 0), (0, 1)):
                    ii, jj = i + di, j + dj
                    w = r.uniform(0.5, 2.0)
                    if ii < nx and jj < ny:
                        o = ii + nx * jj
                        A[v, v] += w; A[o, o] += w; A[v, o] -= w; A[o, v] -= w
                    else:
                        A[v, v] += w
                A[v, v] += r.uniform(0.0, 0.1)
        b = r.normal(size=n)
        l = np.where(r.random(n) < 0.7, 0.0, -np.inf) if r.random() < 0.5 else np.full(n, -r.uniform(0.05, 0.5))
        u = np.where(r.random(n) < 0.5, r.uniform(0.1, 1.0, n), np.inf)
    elif kind == 1:
        n = int(r.integers(5, 40))
        M = r.normal(size=(n, n)) * (r.random((n, n)) < 0.3)
        A = M @ M.T + np.diag(r.uniform(0.1, 2.0, n))
        b = r.normal(size=n) * 3.0
        l = np.where(r.random(n) < 0.6, -r.uniform(0.0, 1.0, n), -np.inf)
        u = np.where(r.random(n) < 0.6, r.uniform(0.0, 1.0, n), np.inf)
    else:
        n = int(r.integers(8, 60))
        A = np.diag(r.uniform(1.0, 100.0, n))
        for i in range(n - 1):
            w = r.uniform(0.0, 1.0) * min(A[i, i], A[i + 1, i + 1]) * 0.45
            A[i, i + 1] = A[i + 1, i] = -w
        b = r.normal(size=n) * 10.0
        l = np.zeros(n)
        u = np.full(n, np.inf)
    x0 = np.minimum(np.maximum(r.normal(size=len(b)) * 0.3, l), u)
    x0 = np.where(np.isfinite(x0), x0, 0.0)
    return A, b, l, u, x0


def _rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


@pytest.mark.parametrize("block", range(5))
def test_control_path_matches_dense_transcription(oracle, block):
    """Record-by-record equality of the control path with tests/_brute.gpcg_dense_trace."""
    seen = dict(multi_step=0, pgstop2=0, pgstop1_after_2=0, refined=0)
    for seed in range(30 * block, 30 * block + 30):
        A, b, l, u, x0 = instance(seed)
        tau = 1e-10 * np.linalg.norm(A @ x0 - b)
        rc, x, st, tr = oracle.solve_trace(csr_of(oracle, A), b, l, u, 0.0, x0, tau)
        rb, xb, trb = B.gpcg_dense_trace(A, b, l, u, x0, tau)
        trb = np.array(trb, float).reshape(-1, 6)
        assert rc == rb == 0, (seed, rc, rb)
        assert tr.shape == trb.shape, (seed, tr.shape, trb.shape)
        # kinds, outer index, j / rep, h / reason / iterations: exact
        assert np.array_equal(tr[:, :4], trb[:, :4]), seed
        # decreases, alphas, eta2, |F|, |A\B|: to rounding
        for ro, rb_ in zip(tr, trb):
            for c in (4, 5):
                assert _rel(ro[c], rb_[c]) <= 1e-7 or abs(ro[c] - rb_[c]) <= 1e-14, (seed, ro, rb_)
        assert np.max(np.abs(x - xb)) <= 1e-8 * max(1.0, np.max(np.abs(xb)))
        ends = tr[tr[:, 0] == GP_END]
        seen["multi_step"] += bool((ends[:, 2] >= 2).any())
        seen["pgstop2"] += bool((ends[:, 3] == R_PGSTOP2).any())
        seen["pgstop1_after_2"] += bool(((ends[:, 3] == R_PGSTOP1) & (ends[:, 2] >= 2)).any())
        seen["refined"] += bool(((tr[:, 0] == CG_CALL) & (tr[:, 2] >= 1)).any())
    # the block exercises every rule it pins
    assert min(seen.values()) >= 5, seen


def test_trace_internal_consistency(oracle):
    """Properties of the trace that follow from the rules themselves (no second implementation):
    a phase ends at the first step meeting a stop rule and at no earlier one; pgstop2 applies
    from j >= 2 only (R10); decreases are positive (sufficient decrease, Eq. gplsstop)."""
    for seed in range(60):
        A, b, l, u, x0 = instance(seed)
        tau = 1e-10 * np.linalg.norm(A @ x0 - b)
        rc, x, st, tr = oracle.solve_trace(csr_of(oracle, A), b, l, u, 0.0, x0, tau)
        for k in np.unique(tr[:, 1]):
            steps = tr[(tr[:, 0] == GP_STEP) & (tr[:, 1] == k)]
            end = tr[(tr[:, 0] == GP_END) & (tr[:, 1] == k)]
            assert len(end) == 1
            j_end, reason = int(end[0, 2]), int(end[0, 3])
            assert len(steps) == j_end and np.array_equal(steps[:, 2], np.arange(1, j_end + 1))
            decs = steps[:, 4]
            assert np.all(decs > 0.0)
            for jj in range(1, j_end):          # no pgstop2 before the end
                if jj >= 2:
                    assert decs[jj - 1] > 0.1 * decs[: jj - 1].max(), (seed, k, jj)
            if reason == R_PGSTOP2:
                assert j_end >= 2 and decs[-1] <= 0.1 * decs[:-1].max()
            if j_end >= 1:
                assert end[0, 4] == decs.max()


def test_gp_phase_unchanged_active_set_stops_after_one_iterate(oracle):
    """SPEC.md:280 (Eq. pgstop1): with infinite bounds the active set is always empty, so
    every GP phase stops after exactly one iterate, by pgstop1."""
    for seed in range(20):
        r = np.random.default_rng(900 + seed)
        n = int(r.integers(4, 30))
        M = r.normal(size=(n, n))
        A = M @ M.T + 0.05 * np.eye(n)         # ill-conditioned: steepest descent is slow
        b = r.normal(size=n)
        l, u = np.full(n, -np.inf), np.full(n, np.inf)
        x0 = r.normal(size=n)
        tau = 1e-10 * np.linalg.norm(A @ x0 - b)
        rc, x, st, tr = oracle.solve_trace(csr_of(oracle, A), b, l, u, 0.0, x0, tau)
        assert rc == 0
        ends = tr[tr[:, 0] == GP_END]
        done = ends[ends[:, 3] != R_CONV]
        assert len(done) >= 1
        assert np.all(done[:, 2] == 1) and np.all(done[:, 3] == R_PGSTOP1), (seed, ends)
        assert st["gp_iters"] == len(done)


def test_gp_unconstrained_first_step_is_steepest_descent(oracle):
    """SPEC.md:281, 270 (Eqs. bqpls, gplsstop): with no bounds the first step size is
    alpha = g'g / g'Ag, accepted at h = 0, and the decrease is (g'g)^2 / (2 g'Ag)."""
    for seed in range(20):
        r = np.random.default_rng(700 + seed)
        n = int(r.integers(3, 25))
        M = r.normal(size=(n, n))
        A = M @ M.T + np.eye(n)
        b = r.normal(size=n)
        x0 = r.normal(size=n)
        inf = np.full(n, np.inf)
        rc, x, st, tr = oracle.solve_trace(csr_of(oracle, A), b, -inf, inf, 0.0, x0, 1e-9)
        g = A @ x0 - b
        gg, gAg = g @ g, g @ A @ g
        step = tr[0]
        assert step[0] == GP_STEP and step[2] == 1 and step[3] == 0
        assert _rel(step[5], gg / gAg) <= 1e-12
        assert _rel(step[4], gg * gg / (2.0 * gAg)) <= 1e-10
        end = tr[1]
        assert end[0] == GP_END and _rel(end[5], gg / gAg) <= 1e-12


def test_eta2_sequence_closed_form(oracle):
    """R12: within one outer iteration the r-th CG call runs with
    eta2 = max(0.05 * 0.1^r, 1e-12); a CG call follows a refinement only if the previous
    search ended with B = A (|A \\ B| = 0, Eq. cgstop3)."""
    n_refined = 0
    for seed in range(90):
        A, b, l, u, x0 = instance(seed)
        tau = 1e-10 * np.linalg.norm(A @ x0 - b)
        rc, x, st, tr = oracle.solve_trace(csr_of(oracle, A), b, l, u, 0.0, x0, tau)
        calls = tr[tr[:, 0] == CG_CALL]
        for c in calls:
            rep = int(c[2])
            assert c[4] == max(0.05 * 0.1 ** rep, 1e-12) or _rel(c[4], max(0.05 * 0.1 ** rep, 1e-12)) <= 1e-15
        for i in range(len(tr) - 1):
            if tr[i + 1, 0] == CG_CALL and tr[i + 1, 2] >= 1:
                n_refined += 1
                assert tr[i, 0] == CG_SEARCH and tr[i, 5] == 0.0 and tr[i, 1] == tr[i + 1, 1]
            if tr[i, 0] == CG_SEARCH and tr[i, 5] != 0.0:
                assert tr[i + 1, 0] == GP_STEP and tr[i + 1, 1] == tr[i, 1] + 1
        assert st["refinements"] >= int(np.sum(calls[:, 2] >= 1))
    assert n_refined >= 20


def test_gp_cap_is_a_safety_net_only(oracle):
    """R13: the paper's GP phase has no iteration cap; the default cap is a
    safety net that the paper's problem class never reaches, and a small cap ends phases by
    reason 3 exactly at the cap."""
    p = oracle.default_params()
    assert p.gp_cap >= 100000
    A, b, l, u, x0 = instance(0)
    tau = 1e-10 * np.linalg.norm(A @ x0 - b)
    rc, x, st, tr = oracle.solve_trace(csr_of(oracle, A), b, l, u, 0.0, x0, tau,
                                       params=oracle.default_params(gp_cap=2))
    ends = tr[tr[:, 0] == GP_END]
    assert np.all(ends[:, 2] <= 2)
    assert np.all((ends[:, 3] != R_CAP) | (ends[:, 2] == 2))
    rb, xb, trb = B.gpcg_dense_trace(A, b, l, u, x0, tau, gp_cap=2)
    assert np.array_equal(tr[:, :4], np.array(trb, float).reshape(-1, 6)[:, :4])


def test_openmp_build_is_bitwise_identical(oracle):
    """The OpenMP build of the same source (SURVEY 8(d)'s all-core baseline) threads only the
    row and elementwise loops; every sum stays serial, so its CG iterates are bitwise equal."""
    import os
    from paper_cs_0101018_b200 import problems as P
    if os.environ.get("ORACLE_LIB"):
        pytest.skip("mutant build under test")
    prob = P.journal_bearing(64, 48, 0.1)
    A = oracle.problem_csr(prob)
    fr = (P.uniform(3, 1, prob.n) < 0.7).astype(np.uint8)
    r = oracle.gradient(A, prob.b, prob.x0)
    it1, w1, d1 = oracle.cg(A, fr, r, 1e-3)
    it2, w2, d2 = oracle.cg(A, fr, r, 1e-3, omp=True)
    assert it1 == it2 > 5 and np.array_equal(w1, w2) and np.array_equal(d1, d2)
