"""Pin the oracle's block-Jacobi ILU(k) (block Jacobi, one block per
subdomain, subdomain solver "ILU(2), which allowed two levels of fill"; Table 4).

The oracle builds ILU(k) by the textbook levels-of-fill rule, row by row.  Independent checks:
  * the PATTERN and the LEVELS against the fill-path theorem: entry (i, j) of ILU(k) has
    level = (length of the shortest path i -> j in the graph of the block whose interior
    nodes are all numbered below min(i, j)) - 1, and exists iff that is <= k -- computed
    here by breadth-first search on the grid graph, a different route from elimination;
  * the defining property of an incomplete factorisation: (L U)_ij = a_ij on the pattern;
  * k large: the complete LU of every block, so M^-1 r = the dense block-diagonal solve;
  * k = 0: the same preconditioner as the oracle's ILU(0) routine (pinned separately);
  * the paper's observation (Table 4): ILU(2) needs fewer CG iterations than
    ILU(0) on the journal-bearing problem.
"""
from collections import deque

import numpy as np
import pytest

from paper_cs_0101018_b200 import problems as P


def grid_problem(nx, ny, seed, eps=0.3):
    p = P.journal_bearing(nx, ny, eps)
    return p


def tile_of(v, nx, tx, ty):
    return ((v % nx) // tx, (v // nx) // ty)


def fill_levels(A, free, nx, tx, ty, k):
    """{(i, j): level} of ILU(k) by the fill-path theorem: for every pair of free nodes of one
    block, a breadth-first search from i to j whose interior nodes are < min(i, j)."""
    n = A.n
    nbrs = [[] for _ in range(n)]
    for i in range(n):
        if not free[i]:
            continue
        for e in range(A.rp[i], A.rp[i + 1]):
            j = int(A.ci[e])
            if j != i and free[j] and tile_of(i, nx, tx, ty) == tile_of(j, nx, tx, ty):
                nbrs[i].append(j)
    lev = {}
    for i in range(n):
        if not free[i]:
            continue
        lev[(i, i)] = 0
        for j in range(n):
            if j == i or not free[j] or tile_of(i, nx, tx, ty) != tile_of(j, nx, tx, ty):
                continue
            lim = min(i, j)
            dist = {i: 0}
            dq = deque([i])
            found = None
            while dq and found is None:
                x = dq.popleft()
                for y in nbrs[x]:
                    if y == j:
                        found = dist[x] + 1
                        break
                    if y < lim and y not in dist:
                        dist[y] = dist[x] + 1
                        dq.append(y)
            if found is not None and found - 1 <= k:
                lev[(i, j)] = found - 1
    return lev


@pytest.mark.parametrize("nx,ny,tx,ty,k,seed", [(9, 7, 5, 4, 2, 1), (12, 10, 12, 10, 2, 2), (8, 8, 8, 8, 1, 3),
                                                (10, 6, 4, 3, 3, 4), (7, 9, 7, 9, 2, 5)])
def test_iluk_pattern_and_levels_are_the_fill_path_ones(oracle, nx, ny, tx, ty, k, seed):
    prob = grid_problem(nx, ny, seed)
    A = oracle.problem_csr(prob)
    free = (P.uniform(seed, 1, prob.n) < 0.8).astype(np.uint8)
    rows, cols, levs, vals = oracle.bjiluk_factor(A, free, nx, tx, ty, k)
    got = {(int(r), int(c)): int(l) for r, c, l in zip(rows, cols, levs)}
    ref = fill_levels(A, free, nx, tx, ty, k)
    assert got == ref


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_iluk_reproduces_a_on_its_pattern(oracle, k):
    nx, ny, tx, ty = 10, 9, 6, 5
    prob = grid_problem(nx, ny, 7)
    A = oracle.problem_csr(prob)
    free = (P.uniform(7, 1, prob.n) < 0.85).astype(np.uint8)
    rows, cols, levs, vals = oracle.bjiluk_factor(A, free, nx, tx, ty, k)
    n = prob.n
    Lm = np.eye(n)
    Um = np.zeros((n, n))
    for r, c, v in zip(rows, cols, vals):
        if c < r:
            Lm[r, c] = v
        else:
            Um[r, c] = v
    LU = Lm @ Um
    Ad = A.todense()
    for r, c in zip(rows, cols):
        assert abs(LU[r, c] - Ad[r, c]) <= 1e-12 * np.abs(Ad).max(), (k, r, c, LU[r, c], Ad[r, c])
    if k == 0:                                   # ILU(0) keeps exactly A's (free, same-tile) pattern
        for r, c in zip(rows, cols):
            assert Ad[r, c] != 0.0


def test_iluk_large_level_is_the_block_solve(oracle):
    """With enough levels the factorisation is complete: one PCG step solves a block-diagonal
    system exactly, and M^-1 equals the inverse of the block-diagonal part of A_F."""
    nx, ny, tx, ty = 12, 8, 4, 4
    prob = grid_problem(nx, ny, 9)
    A = oracle.problem_csr(prob)
    free = (P.uniform(9, 1, prob.n) < 0.75).astype(np.uint8)
    rows, cols, levs, vals = oracle.bjiluk_factor(A, free, nx, tx, ty, 1000)
    n = prob.n
    Lm = np.eye(n)
    Um = np.zeros((n, n))
    for r, c, v in zip(rows, cols, vals):
        if c < r:
            Lm[r, c] = v
        else:
            Um[r, c] = v
    Ad = A.todense()
    B = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if free[i] and free[j] and tile_of(i, nx, tx, ty) == tile_of(j, nx, tx, ty):
                B[i, j] = Ad[i, j]
    F = np.flatnonzero(free)
    M = (Lm @ Um)[np.ix_(F, F)]
    assert np.max(np.abs(M - B[np.ix_(F, F)])) <= 1e-12 * np.abs(Ad).max()


def test_iluk_level0_is_ilu0(oracle):
    nx, ny = 40, 30
    prob = grid_problem(nx, ny, 11)
    A = oracle.problem_csr(prob)
    free = (P.uniform(11, 1, prob.n) < 0.7).astype(np.uint8)
    r = oracle.gradient(A, prob.b, prob.x0)
    it0, w0, d0 = oracle.pcg_bjilu(A, free, r, nx, 8, 8, 1e-3)
    itk, wk, dk = oracle.pcg_bjiluk(A, free, r, nx, 8, 8, 0, 1e-3)
    assert it0 == itk
    assert np.max(np.abs(w0 - wk)) <= 1e-12 * np.max(np.abs(w0))


def test_iluk_pcg_dense_solve(oracle):
    """PCG with ILU(2) solves the reduced system (finite termination, dense solve)."""
    nx, ny = 20, 16
    prob = grid_problem(nx, ny, 13)
    A = oracle.problem_csr(prob)
    free = (P.uniform(13, 1, prob.n) < 0.8).astype(np.uint8)
    r = P.gaussian(13, 2, prob.n)
    it, w, d = oracle.pcg_bjiluk(A, free, r, nx, 8, 8, 2, 1e-30)
    F = np.flatnonzero(free)
    Ad = A.todense()
    ref = np.linalg.solve(Ad[np.ix_(F, F)], -r[F])
    assert np.max(np.abs(w[F] - ref)) <= 1e-9 * np.max(np.abs(ref))
    assert np.all(w[free == 0] == 0.0)


@pytest.mark.parametrize("eps", [0.1, 0.9])
def test_ilu2_fewer_cg_iterations_than_ilu0(oracle, eps):
    """Table 4: 'the block Jacobi preconditioner with subdomain solver ILU(2)
    required fewer conjugate gradient iterations than subdomain solver ILU(0)' -- on the
    journal-bearing problem at the paper's settings (x0 = l, eta1 = 0.1, eta2 = 0.05), and
    both reach the same minimiser."""
    prob = P.journal_bearing(96, 96, eps)
    base = dict(grid_nx=96, grid_ny=96, tile_x=32, tile_y=32)
    rc0, x0, st0 = oracle.solve_problem(prob, tol=-1e-10, params=oracle.default_params(precond=2, **base))
    rc2, x2, st2 = oracle.solve_problem(prob, tol=-1e-10, params=oracle.default_params(precond=3, **base))
    assert rc0 == rc2 == 0
    assert st2["cg_iters"] < st0["cg_iters"], (st2["cg_iters"], st0["cg_iters"])
    assert np.max(np.abs(x0 - x2)) <= 1e-7
