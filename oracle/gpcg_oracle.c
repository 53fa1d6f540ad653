/*
 * gpcg_oracle.c -- plain, slow, obviously-correct CPU reference of GPCG (fp64).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (libgpcg.so, the
 * Python binding paper_cs_0101018_b200/gpcg.py) may include, link, import or
 * execute this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg call it.  It shares no code with the
 * CUDA path: it has its own operator assembly, loops, reductions and control.
 *
 * Paper: Benson, McInnes, More, "GPCG: A case study in the performance and
 * scalability of optimization algorithms" (reference PAPER.md).  Every routine
 * cites the passage it follows as "P:a-b (section, equation)".  Readings of
 * silent/ambiguous passages are numbered R1.. in DESIGN.md ("Readings").
 *
 * Problem (Eq. def-quadratic, sign per reading R1):
 *     minimise q(x) = 1/2 x'Ax - b'x + c   subject to  l <= x <= u.
 * Gradient g = Ax - b.  A is held as CSR with both triangles stored.
 *
 * Style: straight loops in index order, left-to-right sums, no blocking, no
 * fusion, no reordering.  Build with -O2 -ffp-contract=off so that every
 * a*b+c rounds twice, as written.
 *
 * OpenMP build ("the OpenMP build of the same source, all host cores"):
 * compiled with -fopenmp, the row loops of the SpMVs and the elementwise vector loops
 * (no reductions) are split over threads; every sum (dot products, norms, counts) stays a
 * single left-to-right loop, so both builds return bitwise-identical results.  Without
 * -fopenmp the pragmas are ignored and the file is the plain single-threaded oracle.
 *
 * Pins (tests/test_oracle_*.py): dense brute-force products, the eps=0
 * Laplacian eigenpairs, 3^n active-set enumeration, Cholesky solves with
 * infinite bounds, KKT certificates, SPEC.md hand values, the paper's free
 * fractions.  Parity unpinned: iteration counts vs the paper's
 * tables (different discretisation and preconditioner).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* status codes (same meaning as the product ABI, defined independently) */
#define ORA_OK 0
#define ORA_NOT_CONVERGED 1
#define ORA_EINVAL (-1)
#define ORA_ENOMEM (-2)
#define ORA_ENOTSPD (-5)
#define ORA_ESEARCH (-6)

typedef struct {
    double mu;            /* sufficient-decrease constant, "mu in (0,1/2)"; 0.1 (R6)      */
    double eta1;          /* Eq. pgstop2, P:789 eta1 = 0.1                                        */
    double eta2;          /* Eq. cgstop1, P:790 eta2 = 0.05                                       */
    double eta2_shrink;   /* Eq. cgstop3 "reduce eta2" P:491: x0.1 (R12)                          */
    double eta2_floor;    /* 1e-12 (R12)                                                          */
    int64_t gp_cap;       /* GP iterates per phase: safety net only, 100000 (R13; the paper has none) */
    int64_t refine_cap;   /* cgstop3 repetitions per outer iterate, 30 (R12)                      */
    int64_t max_halvings; /* projected-search trials, 50 (R13)                                    */
    int64_t cg_cap;       /* 0 => m_k, the finite-termination bound P:444-447                     */
    double time_budget_s; /* 0 => none; else stop (NOT_CONVERGED) once exceeded (bounded samples) */
    int64_t precond;      /* 0: plain CG (the hot path); 1: point-Jacobi PCG, M = diag(A_k)
                             (the "diagonal Jacobi preconditioner" of P:1096-1098, Table 4);
                             2: block-Jacobi ILU(0) on tiles of a 2-D grid;
                             3: block-Jacobi ILU(ilu_level) on the same tiles       */
    int64_t grid_nx, grid_ny;   /* precond 2: the 2-D grid (v = i + nx j)                          */
    int64_t tile_x, tile_y;     /* precond 2: block = tile_x x tile_y tile of the grid              */
    double *trace;              /* nullable: per-step record of the control path (test pins only),  */
    int64_t trace_cap;          /* trace_cap records of ORA_TREC doubles, see trace_put()           */
    int64_t ilu_level;          /* precond 3: block-Jacobi ILU(ilu_level), 2 = the paper's ILU(2)   */
} ora_params;

typedef struct {
    int64_t outer_iters, gp_iters, cg_iters, cg_calls, refinements, full_spmvs;
    int64_t n_free, n_active, n_active_nonbinding;
    double pg_norm, q, g0_norm, tau, seconds;
    int64_t status;
    int64_t trace_len;    /* records written to prm->trace (may exceed trace_cap: then truncated) */
} ora_stats;

/* Control-path trace (test infrastructure: lets the pins check the GP-phase stop rules and
 * the eta2 refinement step by step).  One record = ORA_TREC doubles
 *   {kind, k, i1, i2, v1, v2}
 *   kind 1  GP step        i1 = j (1-based),   i2 = h (accepted halving), v1 = q(y_{j-1}) - q(y_j), v2 = alpha
 *   kind 2  GP phase end   i1 = j_k (steps),   i2 = reason: 0 converged, 1 Eq. pgstop1, 2 Eq. pgstop2,
 *                                                           3 gp_cap,   v1 = max decrease, v2 = alpha_0 of step 1
 *   kind 3  CG call        i1 = rep,           i2 = iterations,          v1 = eta2 used, v2 = m_k = |F|
 *   kind 4  CG search      i1 = rep,           i2 = h,                   v1 = q(x_k) - q(x_{k+1}),
 *                                                                        v2 = |A(x_{k+1}) \ B(x_{k+1})|     */
#define ORA_TREC 6
static void trace_put(const ora_params *prm, ora_stats *st, int kind, int64_t k, int64_t i1, int64_t i2,
                      double v1, double v2)
{
    if (prm->trace && st->trace_len < prm->trace_cap) {
        double *r = prm->trace + ORA_TREC * st->trace_len;
        r[0] = kind; r[1] = (double)k; r[2] = (double)i1; r[3] = (double)i2; r[4] = v1; r[5] = v2;
    }
    st->trace_len++;
}

/* ------------------------------------------------------------------------ */
/* operator                                                                  */
/* ------------------------------------------------------------------------ */

/* Number of stored entries of the 5-point stencil matrix on an nx x ny grid. */
int64_t ora_stencil2d_nnz(int64_t nx, int64_t ny)
{
    return 5 * nx * ny - 2 * nx - 2 * ny;
}

/* Assemble the 5-point face-weight operator as CSR.
 * Definition (BASELINE.json configs[0], reading R2): A = sum over faces f of
 * w_f (e_a - e_b)(e_a - e_b)' for interior faces joining points a, b, plus
 * w_f e_a e_a' for faces on the Dirichlet boundary, plus diag(shift).
 * Face conventions as in include/gpcg.h: wx[j*wx_ld + k] joins (k-1, j)-(k, j),
 * k = 0..nx; wy[f*wy_ld + i] joins (i, f-1)-(i, f), f = 0..ny; ld 0 = broadcast.
 * Columns come out in increasing order: (i,j-1), (i-1,j), (i,j), (i+1,j), (i,j+1). */
int ora_stencil2d_to_csr(int64_t nx, int64_t ny, const double *wx, int64_t wx_ld,
                         const double *wy, int64_t wy_ld, const double *shift,
                         int64_t *rp, int32_t *ci, double *val)
{
    if (nx <= 0 || ny <= 0) return ORA_EINVAL;
    int64_t p = 0;
    rp[0] = 0;
    for (int64_t j = 0; j < ny; j++) {
        for (int64_t i = 0; i < nx; i++) {
            int64_t v = i + nx * j;
            double w_west = wx[j * wx_ld + i];
            double w_east = wx[j * wx_ld + i + 1];
            double w_south = wy[j * wy_ld + i];
            double w_north = wy[(j + 1) * wy_ld + i];
            double d = w_west + w_east + w_south + w_north;
            if (shift) d = d + shift[v];
            if (j > 0)      { ci[p] = (int32_t)(v - nx); val[p] = -w_south; p++; }
            if (i > 0)      { ci[p] = (int32_t)(v - 1);  val[p] = -w_west;  p++; }
            ci[p] = (int32_t)v; val[p] = d; p++;
            if (i < nx - 1) { ci[p] = (int32_t)(v + 1);  val[p] = -w_east;  p++; }
            if (j < ny - 1) { ci[p] = (int32_t)(v + nx); val[p] = -w_north; p++; }
            rp[v + 1] = p;
        }
    }
    return ORA_OK;
}

/* 3-D 7-point face-weight operator (the 3-D analogue of
 * the definition above: A = sum over faces of w_f (e_a - e_b)(e_a - e_b)', boundary
 * faces w_f e_a e_a', plus diag(shift)).  Point (i, j, k) <-> v = i + nx (j + ny k).
 * wx[(k ny + j)(nx+1) + i'] joins (i'-1, j, k)-(i', j, k), i' = 0..nx;
 * wy[(k (ny+1) + j') nx + i] joins (i, j'-1, k)-(i, j', k), j' = 0..ny;
 * wz[k' nx ny + j nx + i] joins (i, j, k'-1)-(i, j, k'), k' = 0..nz.
 * Columns in increasing order: -z, -y, -x, diag, +x, +y, +z. */
int64_t ora_stencil3d_nnz(int64_t nx, int64_t ny, int64_t nz)
{
    return 7 * nx * ny * nz - 2 * (ny * nz + nx * nz + nx * ny);
}

int ora_stencil3d_to_csr(int64_t nx, int64_t ny, int64_t nz, const double *wx, const double *wy,
                         const double *wz, const double *shift, int64_t *rp, int32_t *ci, double *val)
{
    if (nx <= 0 || ny <= 0 || nz <= 0) return ORA_EINVAL;
    int64_t p = 0;
    rp[0] = 0;
    for (int64_t k = 0; k < nz; k++) {
        for (int64_t j = 0; j < ny; j++) {
            for (int64_t i = 0; i < nx; i++) {
                int64_t v = i + nx * (j + ny * k);
                double w_w = wx[(k * ny + j) * (nx + 1) + i];
                double w_e = wx[(k * ny + j) * (nx + 1) + i + 1];
                double w_s = wy[(k * (ny + 1) + j) * nx + i];
                double w_n = wy[(k * (ny + 1) + j + 1) * nx + i];
                double w_d = wz[k * nx * ny + j * nx + i];
                double w_u = wz[(k + 1) * nx * ny + j * nx + i];
                double d = w_w + w_e + w_s + w_n + w_d + w_u;
                if (shift) d = d + shift[v];
                if (k > 0)      { ci[p] = (int32_t)(v - nx * ny); val[p] = -w_d; p++; }
                if (j > 0)      { ci[p] = (int32_t)(v - nx);      val[p] = -w_s; p++; }
                if (i > 0)      { ci[p] = (int32_t)(v - 1);       val[p] = -w_w; p++; }
                ci[p] = (int32_t)v; val[p] = d; p++;
                if (i < nx - 1) { ci[p] = (int32_t)(v + 1);       val[p] = -w_e; p++; }
                if (j < ny - 1) { ci[p] = (int32_t)(v + nx);      val[p] = -w_n; p++; }
                if (k < nz - 1) { ci[p] = (int32_t)(v + nx * ny); val[p] = -w_u; p++; }
                rp[v + 1] = p;
            }
        }
    }
    return ORA_OK;
}

/* y = A x  (row-wise left-to-right sums) -- "Mat-Vec Multiply", T3 P:999-1005 */
void ora_spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
              const double *x, double *y)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) s += val[k] * x[ci[k]];
        y[i] = s;
    }
}

/* y = Z Z' A Z Z' x : the reduced Hessian A_k = Z_k' A Z_k (Eq. cg2)
 * embedded in R^n.  free[i] != 0 marks a free variable; x is read only on the
 * free set and y is zero off it. */
void ora_spmv_masked(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                     const unsigned char *free_, const double *x, double *y)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        if (free_[i]) {
            for (int64_t k = rp[i]; k < rp[i + 1]; k++)
                if (free_[ci[k]]) s += val[k] * x[ci[k]];
        }
        y[i] = s;
    }
}

static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* vectors                                                                   */
/* ------------------------------------------------------------------------ */
static double dot(int64_t n, const double *a, const double *b)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
    return s;
}

/* median of {l, u, x}: P[x] = mid(l, u, x) */
static double mid(double l, double u, double x)
{
    if (x < l) return l;
    if (x > u) return u;
    return x;
}

void ora_project(int64_t n, const double *l, const double *u, const double *x, double *px)
{
    for (int64_t i = 0; i < n; i++) px[i] = mid(l[i], u[i], x[i]);
}

/* Projected gradient, Eq. proj-gradient.  Fixed variables l=u
 * are active at both bounds; the two cases give min(g,0) and max(g,0), whose
 * only common value is 0 (reading R16). */
static double pgrad_i(double x, double g, double l, double u)
{
    int at_l = (x == l), at_u = (x == u);
    if (at_l && at_u) return 0.0;
    if (at_l) return g < 0.0 ? g : 0.0;
    if (at_u) return g > 0.0 ? g : 0.0;
    return g;
}

void ora_proj_grad(int64_t n, const double *x, const double *g, const double *l,
                   const double *u, double *pg)
{
    for (int64_t i = 0; i < n; i++) pg[i] = pgrad_i(x[i], g[i], l[i], u[i]);
}

static double pgnorm(int64_t n, const double *x, const double *g, const double *l, const double *u)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) { double d = pgrad_i(x[i], g[i], l[i], u[i]); s += d * d; }
    return sqrt(s);
}

/* A(x) = {i : x_i = l_i or x_i = u_i}; B(x) binding set. */
static int is_active(double x, double l, double u) { return x == l || x == u; }
static int is_binding(double x, double g, double l, double u)
{
    return (x == l && g >= 0.0) || (x == u && g <= 0.0);
}

void ora_sets(int64_t n, const double *x, const double *g, const double *l, const double *u,
              unsigned char *active, unsigned char *binding, int64_t *n_active, int64_t *n_binding)
{
    int64_t na = 0, nb = 0;
    for (int64_t i = 0; i < n; i++) {
        int a = is_active(x[i], l[i], u[i]);
        int b = is_binding(x[i], g[i], l[i], u[i]);
        if (active) active[i] = (unsigned char)a;
        if (binding) binding[i] = (unsigned char)b;
        na += a; nb += b;
    }
    if (n_active) *n_active = na;
    if (n_binding) *n_binding = nb;
}

/* q(x) = 1/2 x'Ax - b'x + c, computed as 1/2 x'(Ax) - b'x + c in index order */
double ora_objective(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                     const double *b, double c, const double *x)
{
    double *Ax = (double *)malloc((size_t)n * sizeof(double));
    if (!Ax) return NAN;
    ora_spmv(n, rp, ci, val, x, Ax);
    double q = 0.5 * dot(n, x, Ax) - dot(n, b, x) + c;
    free(Ax);
    return q;
}

/* g = A x - b */
static void gradient(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                     const double *b, const double *x, double *g)
{
    ora_spmv(n, rp, ci, val, x, g);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) g[i] = g[i] - b[i];
}

/* ------------------------------------------------------------------------ */
/* gradient projection pieces                                                */
/* ------------------------------------------------------------------------ */

/* alpha_0 = argmin_{alpha>0} q(y - alpha d), d = grad_Omega q(y): Eq. bqpls
 * (P:362-374).  The map is the quadratic q(y) - alpha <g,d> + alpha^2/2 <d,Ad>
 * and <g,d> = <d,d> because d_i is g_i or 0.  Returns 0 and sets *status to
 * ENOTSPD when <d,Ad> <= 0 (reading R7).  work: 2n doubles. */
double ora_cauchy_alpha(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                        const double *y, const double *g, const double *l, const double *u,
                        double *work, int *status)
{
    double *d = work, *Ad = work + n;
    ora_proj_grad(n, y, g, l, u, d);
    ora_spmv(n, rp, ci, val, d, Ad);
    double dd = dot(n, d, d), dAd = dot(n, d, Ad);
    *status = ORA_OK;
    if (!(dAd > 0.0)) { *status = ORA_ENOTSPD; return 0.0; }
    return dd / dAd;
}

/* Projected search along dir from y (Eqs. next-y/gplsstop P:341-361 with
 * dir = -g, alpha_base = alpha_0; Eq. cglsstop2 P:475-481 with dir = d_k,
 * alpha_base = 1): the first alpha = alpha_base * 2^-h, h = 0,1,.., with
 *     q(P[y + alpha dir]) <= q(y) + mu <g, P[y + alpha dir] - y>.
 * q(ytrial) - q(y) is evaluated by the exact expansion <g,s> + 1/2 <s,As>,
 * s = ytrial - y (reading R17).  Writes the accepted point (the mid() result
 * itself) to ynew.  Returns h >= 0, or -1 if no trial is accepted.
 * work: 2n doubles.  *delta = q(ynew) - q(y). */
int64_t ora_projected_search(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                             const double *y, const double *g, const double *dir,
                             const double *l, const double *u, double alpha_base, double mu,
                             int64_t max_halvings, double *ynew, double *work,
                             double *delta, double *alpha_out)
{
    double *s = work, *As = work + n;
    for (int64_t h = 0; h < max_halvings; h++) {
        double alpha = ldexp(alpha_base, (int)-h);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            ynew[i] = mid(l[i], u[i], y[i] + alpha * dir[i]);
            s[i] = ynew[i] - y[i];
        }
        ora_spmv(n, rp, ci, val, s, As);
        double gs = dot(n, g, s);
        double sAs = dot(n, s, As);
        double dq = gs + 0.5 * sAs;
        if (dq <= mu * gs) {
            *delta = dq;
            *alpha_out = alpha;
            return h;
        }
    }
    return -1;
}

/* ------------------------------------------------------------------------ */
/* conjugate gradients on the reduced system (Eqs. cg, cg2, cgstop1) */
/* ------------------------------------------------------------------------ */

/* Textbook CG (Hestenes-Stiefel) on A_k w = -r_k, w_0 = 0 (Alg. GPCG),
 * vectors embedded in R^n and zero off the free set; with dinv != NULL the
 * preconditioned (PCG) form with M^{-1} = diag(dinv) on the free set (point
 * Jacobi: dinv_i = 1 / A_ii), z_j = M^{-1} rho_j.  Stops at the
 * first j with
 *   (a) j >= 2 and q_k(w_{j-1}) - q_k(w_j) <= eta2 max_{l<j} (q_k(w_{l-1}) - q_k(w_l))
 *       (Eq. cgstop1; from j >= 2, reading R10), where the decrease of
 *       step j is 1/2 alpha_j rho_j'z_j (reading R17; z = rho without M);
 *   (b) sqrt(rho_j'z_j) <= 1e-14 (1 + sqrt(rho_0'z_0))   (machine-precision guard,
 *       SPEC S:371; the M^{-1}-norm of the residual under PCG, reading R28);
 *   (c) j = cap.
 * Returns w_j at that j (reading R11).  Returns the iteration count, or
 * ORA_ENOTSPD (negative) on <p, A_k p> <= 0.  work: 4n doubles. decs (nullable,
 * length >= cap) receives the per-step decreases. */
void ora_bjilu_factor(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                      const unsigned char *free_, int64_t nx, int64_t tx, int64_t ty, double *d);
void ora_bjilu_apply(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                     const unsigned char *free_, int64_t nx, int64_t tx, int64_t ty, const double *d,
                     const double *r, double *t, double *z);

/* block-Jacobi ILU(k) factor (kind 3, below): rows of L (unit, strictly lower) and U (upper,
 * with the diagonal) of every block, in natural order; row v holds ent[beg[v] .. beg[v+1]) */
typedef struct {
    int64_t n, cap, used;
    int64_t *beg;               /* n + 1 */
    int64_t *col;
    int64_t *lev;
    double *val;                /* L entries (col < v): l_vc;  U entries (col >= v): u_vc */
} ora_iluk;

int ora_bjiluk_factor(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                      const unsigned char *free_, int64_t nx, int64_t tx, int64_t ty, int64_t level, ora_iluk *F);
void ora_bjiluk_apply(const ora_iluk *F, const unsigned char *free_, const double *r, double *t, double *z);
void ora_iluk_free(ora_iluk *F);

/* preconditioner of ora_pcg_m: kind 0 none, 1 point Jacobi (dinv), 2 block-Jacobi ILU(0),
 * 3 block-Jacobi ILU(level) (grid nx, tiles tx x ty; factored at the start of every CG call
 * on its free set) */
typedef struct {
    int kind;
    const double *dinv;
    int64_t nx, tx, ty;
    double *d, *t;              /* kind 2: pivots and forward-solve scratch (n each); kind 3: t only */
    int64_t level;              /* kind 3 */
    ora_iluk *F;                /* kind 3 */
} ora_prec;

static void prec_apply(const ora_prec *M, int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                       const unsigned char *free_, const double *r, double *z)
{
    if (M->kind == 1) {
        for (int64_t i = 0; i < n; i++) z[i] = free_[i] ? r[i] * M->dinv[i] : 0.0;
    } else if (M->kind == 3) {
        ora_bjiluk_apply(M->F, free_, r, M->t, z);
    } else {
        ora_bjilu_apply(n, rp, ci, val, free_, M->nx, M->tx, M->ty, M->d, r, M->t, z);
    }
}

int64_t ora_pcg_m(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                  const unsigned char *free_, const double *r, const ora_prec *M, double eta2, int64_t cap,
                  double *w, double *work, double *decs, double deadline)
{
    const int pc = M && M->kind != 0;
    double *rho = work, *p = work + n, *a = work + 2 * n;
    double *z = pc ? work + 3 * n : rho;
    if (M && M->kind == 2) ora_bjilu_factor(n, rp, ci, val, free_, M->nx, M->tx, M->ty, M->d);
    if (M && M->kind == 3 &&
        ora_bjiluk_factor(n, rp, ci, val, free_, M->nx, M->tx, M->ty, M->level, M->F) != ORA_OK)
        return ORA_ENOMEM;
    for (int64_t i = 0; i < n; i++) {
        rho[i] = free_[i] ? -r[i] : 0.0;
        w[i] = 0.0;
    }
    if (pc) prec_apply(M, n, rp, ci, val, free_, rho, z);
    for (int64_t i = 0; i < n; i++) p[i] = z[i];
    double rr = dot(n, rho, z);
    double rnorm0 = sqrt(rr);
    double maxdec = 0.0;
    int64_t it = 0;
    if (cap <= 0) return 0;
    for (;;) {
        it++;
        ora_spmv_masked(n, rp, ci, val, free_, p, a);
        double pAp = dot(n, p, a);
        if (!(pAp > 0.0)) return ORA_ENOTSPD;
        double alpha = rr / pAp;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) w[i] = w[i] + alpha * p[i];
        double dec = 0.5 * alpha * rr;
        if (decs) decs[it - 1] = dec;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) rho[i] = rho[i] - alpha * a[i];
        if (pc) prec_apply(M, n, rp, ci, val, free_, rho, z);
        double rr_new = dot(n, rho, z);
        int stop = (it >= 2 && dec <= eta2 * maxdec) ||
                   (sqrt(rr_new) <= 1e-14 * (1.0 + rnorm0)) || (it >= cap) ||
                   (deadline > 0.0 && now_s() > deadline);  /* bounded-sample timing only */
        if (dec > maxdec) maxdec = dec;
        if (stop) break;
        double beta = rr_new / rr;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) p[i] = z[i] + beta * p[i];
        rr = rr_new;
    }
    return it;
}

/* point-Jacobi form (dinv nullable: plain CG) */
int64_t ora_pcg(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                const unsigned char *free_, const double *r, const double *dinv, double eta2, int64_t cap,
                double *w, double *work, double *decs, double deadline)
{
    ora_prec M = {dinv ? 1 : 0, dinv, 0, 0, 0, NULL, NULL, 0, NULL};
    return ora_pcg_m(n, rp, ci, val, free_, r, &M, eta2, cap, w, work, decs, deadline);
}

/* block-Jacobi ILU(0) form (tiles tx x ty of an nx-wide grid); work: 4n, scratch: 2n */
int64_t ora_pcg_bjilu(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                      const unsigned char *free_, const double *r, int64_t nx, int64_t tx, int64_t ty,
                      double eta2, int64_t cap, double *w, double *work, double *scratch, double *decs)
{
    ora_prec M = {2, NULL, nx, tx, ty, scratch, scratch + n, 0, NULL};
    return ora_pcg_m(n, rp, ci, val, free_, r, &M, eta2, cap, w, work, decs, 0.0);
}

/* block-Jacobi ILU(level) form (tiles tx x ty of an nx-wide grid); work: 4n, scratch: n */
int64_t ora_pcg_bjiluk(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                       const unsigned char *free_, const double *r, int64_t nx, int64_t tx, int64_t ty,
                       int64_t level, double eta2, int64_t cap, double *w, double *work, double *scratch,
                       double *decs)
{
    ora_iluk F;
    memset(&F, 0, sizeof F);
    ora_prec M = {3, NULL, nx, tx, ty, NULL, scratch, level, &F};
    int64_t it = ora_pcg_m(n, rp, ci, val, free_, r, &M, eta2, cap, w, work, decs, 0.0);
    ora_iluk_free(&F);
    return it;
}

/* plain CG (the hot path's CG): ora_pcg without a preconditioner */
int64_t ora_cg(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
               const unsigned char *free_, const double *r, double eta2, int64_t cap,
               double *w, double *work, double *decs, double deadline)
{
    return ora_pcg(n, rp, ci, val, free_, r, NULL, eta2, cap, w, work, decs, deadline);
}

/* ------------------------------------------------------------------------ */
/* block-Jacobi ILU(0) ("a block Jacobi preconditioner ... ILU(0),  */
/* which produced a factored matrix that maintained the same sparsity pattern")  */
/* ------------------------------------------------------------------------ */
/* Blocks: the tiles of tile_x x tile_y points of an nx x ny grid (v = i + nx j); within a
 * block the rows of A_k = Z'AZ (free points only) in natural order.  ILU(0) keeps A's
 * pattern: M = (D + L) D^-1 (D + U), L / U the strict lower / upper parts of the block of
 * A_k, D the pivots
 *     d_v = a_vv - sum_{u < v in the block, u free, a_vu != 0} a_vu a_uv / d_u
 * (for a pattern in which no product l_vk u_ku lands on a pattern entry other than the
 * diagonal -- true for the 5-point stencil in natural order -- this is exactly ILU(0)).
 * Entries coupling different blocks are dropped (block Jacobi).  Symmetric A: a_uv = a_vu. */
static int same_tile(int64_t u, int64_t v, int64_t nx, int64_t tx, int64_t ty)
{
    return (u % nx) / tx == (v % nx) / tx && (u / nx) / ty == (v / nx) / ty;
}

void ora_bjilu_factor(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                      const unsigned char *free_, int64_t nx, int64_t tx, int64_t ty, double *d)
{
    /* natural order is a valid elimination order inside every block: u < v globally and in
     * the same tile <=> u precedes v in the tile's row-major order */
    for (int64_t v = 0; v < n; v++) {
        if (!free_[v]) { d[v] = 1.0; continue; }
        double dv = 0.0;
        for (int64_t k = rp[v]; k < rp[v + 1]; k++)
            if (ci[k] == v) dv += val[k];
        for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
            int64_t u = ci[k];
            if (u < v && free_[u] && same_tile(u, v, nx, tx, ty)) dv = dv - val[k] * val[k] / d[u];
        }
        d[v] = dv;
    }
}

/* z = M^-1 r on the free set: (D + L) t = r forward, then D^-1 (D + U) z = t backward */
void ora_bjilu_apply(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                     const unsigned char *free_, int64_t nx, int64_t tx, int64_t ty, const double *d,
                     const double *r, double *t, double *z)
{
    for (int64_t v = 0; v < n; v++) {
        if (!free_[v]) { t[v] = 0.0; continue; }
        double s = r[v];
        for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
            int64_t u = ci[k];
            if (u < v && free_[u] && same_tile(u, v, nx, tx, ty)) s = s - val[k] * t[u];
        }
        t[v] = s / d[v];
    }
    for (int64_t v = n - 1; v >= 0; v--) {
        if (!free_[v]) { z[v] = 0.0; continue; }
        double s = 0.0;
        for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
            int64_t u = ci[k];
            if (u > v && free_[u] && same_tile(u, v, nx, tx, ty)) s = s + val[k] * z[u];
        }
        z[v] = t[v] - s / d[v];
    }
}

/* ------------------------------------------------------------------------ */
/* block-Jacobi ILU(k) ("ILU(2), which allowed two levels of fill")  */
/* ------------------------------------------------------------------------ */
/* ILU(p) with levels of fill, row by row in the IKJ form (the textbook ILU(p) algorithm):
 * on each block (tile) of A_k = Z'AZ in natural order, row v starts as the free, same-tile
 * entries of A, all of level 0; then for every k < v of the row with lev(v,k) <= p, in
 * increasing k:   l_vk = a_vk / u_kk;   a_vj -= l_vk u_kj  for every j > k of U's row k,
 * lev(v,j) = min(lev(v,j), lev(v,k) + lev(k,j) + 1)   (a new position starts at that
 * level); finally the positions with lev(v,j) > p are dropped.  M = L U, L unit lower.
 * ILU(0) keeps A's pattern (= ora_bjilu_* above); p large enough gives the complete LU
 * factorisation of every block. */
static int iluk_reserve(ora_iluk *F, int64_t need)
{
    if (F->used + need <= F->cap) return ORA_OK;
    int64_t c = F->cap ? F->cap : 1024;
    while (c < F->used + need) c *= 2;
    int64_t *col = (int64_t *)realloc(F->col, (size_t)c * sizeof(int64_t));
    if (!col) return ORA_ENOMEM;
    F->col = col;
    int64_t *lev = (int64_t *)realloc(F->lev, (size_t)c * sizeof(int64_t));
    if (!lev) return ORA_ENOMEM;
    F->lev = lev;
    double *v = (double *)realloc(F->val, (size_t)c * sizeof(double));
    if (!v) return ORA_ENOMEM;
    F->val = v;
    F->cap = c;
    return ORA_OK;
}

void ora_iluk_free(ora_iluk *F)
{
    free(F->beg); free(F->col); free(F->lev); free(F->val);
    memset(F, 0, sizeof *F);
}

int ora_bjiluk_factor(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                      const unsigned char *free_, int64_t nx, int64_t tx, int64_t ty, int64_t level, ora_iluk *F)
{
    if (F->n != n) {
        free(F->beg);
        F->beg = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
        if (!F->beg) return ORA_ENOMEM;
        F->n = n;
    }
    F->used = 0;
    /* the working row: positions (col, lev, val) in insertion order, scanned linearly */
    int64_t wcap = 64, wn;
    for (int64_t v = 0; v < n; v++)
        if (4 * (rp[v + 1] - rp[v]) > wcap) wcap = 4 * (rp[v + 1] - rp[v]);
    int64_t *wc = (int64_t *)malloc((size_t)wcap * sizeof(int64_t));
    int64_t *wl = (int64_t *)malloc((size_t)wcap * sizeof(int64_t));
    double *wv = (double *)malloc((size_t)wcap * sizeof(double));
    unsigned char *wd = (unsigned char *)malloc((size_t)wcap);
    if (!wc || !wl || !wv || !wd) { free(wc); free(wl); free(wv); free(wd); return ORA_ENOMEM; }
    for (int64_t v = 0; v < n; v++) {
        F->beg[v] = F->used;
        if (!free_[v]) continue;
        wn = 0;
        for (int64_t k = rp[v]; k < rp[v + 1]; k++) {
            int64_t u = ci[k];
            if (!free_[u] || !same_tile(u, v, nx, tx, ty)) continue;
            int64_t f = -1;
            for (int64_t q = 0; q < wn; q++) if (wc[q] == u) { f = q; break; }
            if (f >= 0) { wv[f] += val[k]; continue; }
            wc[wn] = u; wl[wn] = 0; wv[wn] = val[k]; wd[wn] = 0; wn++;   /* wcap >= 4 x row length */
        }
        for (;;) {
            /* the smallest not yet eliminated k < v with lev(v,k) <= level */
            int64_t qk = -1;
            for (int64_t q = 0; q < wn; q++)
                if (wc[q] < v && !wd[q] && wl[q] <= level && (qk < 0 || wc[q] < wc[qk])) qk = q;
            if (qk < 0) break;
            wd[qk] = 1;
            int64_t k = wc[qk];
            double ukk = 0.0;
            for (int64_t e = F->beg[k]; e < F->beg[k + 1]; e++) if (F->col[e] == k) ukk = F->val[e];
            double lvk = wv[qk] / ukk;
            wv[qk] = lvk;
            for (int64_t e = F->beg[k]; e < F->beg[k + 1]; e++) {
                int64_t j = F->col[e];
                if (j <= k) continue;                       /* U's row k: j > k */
                int64_t nl = wl[qk] + F->lev[e] + 1;
                int64_t f = -1;
                for (int64_t q = 0; q < wn; q++) if (wc[q] == j) { f = q; break; }
                if (f < 0) {
                    if (wn == wcap) {
                        wcap *= 2;
                        int64_t *a = (int64_t *)realloc(wc, (size_t)wcap * sizeof(int64_t)); if (a) wc = a;
                        int64_t *b = (int64_t *)realloc(wl, (size_t)wcap * sizeof(int64_t)); if (b) wl = b;
                        double *c = (double *)realloc(wv, (size_t)wcap * sizeof(double)); if (c) wv = c;
                        unsigned char *d = (unsigned char *)realloc(wd, (size_t)wcap); if (d) wd = d;
                        if (!a || !b || !c || !d) { free(wc); free(wl); free(wv); free(wd); return ORA_ENOMEM; }
                    }
                    f = wn++;
                    wc[f] = j; wl[f] = nl; wv[f] = 0.0; wd[f] = 0;
                }
                wv[f] = wv[f] - lvk * F->val[e];
                if (nl < wl[f]) wl[f] = nl;
            }
        }
        /* keep the positions of level <= p, in increasing column order */
        int64_t keep = 0;
        for (int64_t q = 0; q < wn; q++) keep += wl[q] <= level;
        if (iluk_reserve(F, keep) != ORA_OK) { free(wc); free(wl); free(wv); free(wd); return ORA_ENOMEM; }
        int64_t last = -1;
        for (int64_t m = 0; m < keep; m++) {
            int64_t qb = -1;
            for (int64_t q = 0; q < wn; q++)
                if (wl[q] <= level && wc[q] > last && (qb < 0 || wc[q] < wc[qb])) qb = q;
            F->col[F->used] = wc[qb]; F->lev[F->used] = wl[qb]; F->val[F->used] = wv[qb];
            F->used++;
            last = wc[qb];
        }
    }
    F->beg[n] = F->used;
    free(wc); free(wl); free(wv); free(wd);
    return ORA_OK;
}

/* z = M^-1 r = U^-1 L^-1 r on the free set (forward L t = r, L unit; backward U z = t) */
void ora_bjiluk_apply(const ora_iluk *F, const unsigned char *free_, const double *r, double *t, double *z)
{
    int64_t n = F->n;
    for (int64_t v = 0; v < n; v++) {
        if (!free_[v]) { t[v] = 0.0; continue; }
        double s = r[v];
        for (int64_t e = F->beg[v]; e < F->beg[v + 1]; e++)
            if (F->col[e] < v) s = s - F->val[e] * t[F->col[e]];
        t[v] = s;
    }
    for (int64_t v = n - 1; v >= 0; v--) {
        if (!free_[v]) { z[v] = 0.0; continue; }
        double s = t[v], d = 0.0;
        for (int64_t e = F->beg[v]; e < F->beg[v + 1]; e++) {
            if (F->col[e] > v) s = s - F->val[e] * z[F->col[e]];
            else if (F->col[e] == v) d = F->val[e];
        }
        z[v] = s / d;
    }
}

/* The factor of ora_bjiluk_factor as dense-able triplets (tests): L and U entries with their
 * levels.  Returns the entry count; with out arrays NULL only counts. */
int64_t ora_bjiluk_export(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                          const unsigned char *free_, int64_t nx, int64_t tx, int64_t ty, int64_t level,
                          int64_t *rows, int64_t *cols, int64_t *levs, double *vals, int64_t cap)
{
    ora_iluk F;
    memset(&F, 0, sizeof F);
    if (ora_bjiluk_factor(n, rp, ci, val, free_, nx, tx, ty, level, &F) != ORA_OK) return -1;
    int64_t m = F.used;
    if (rows && m <= cap) {
        for (int64_t v = 0; v < n; v++)
            for (int64_t e = F.beg[v]; e < F.beg[v + 1]; e++) {
                rows[e] = v; cols[e] = F.col[e]; levs[e] = F.lev[e]; vals[e] = F.val[e];
            }
    }
    ora_iluk_free(&F);
    return m;
}

/* dinv_i = 1 / A_ii (the point-Jacobi preconditioner; A SPD => A_ii > 0) */
void ora_jacobi_inverse(int64_t n, const int64_t *rp, const int32_t *ci, const double *val, double *dinv)
{
    for (int64_t i = 0; i < n; i++) {
        double d = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; k++)
            if (ci[k] == i) d += val[k];
        dinv[i] = 1.0 / d;
    }
}

/* ------------------------------------------------------------------------ */
/* Algorithm GPCG                                                */
/* ------------------------------------------------------------------------ */

void ora_params_default(ora_params *p)
{
    p->mu = 0.1; p->eta1 = 0.1; p->eta2 = 0.05; p->eta2_shrink = 0.1; p->eta2_floor = 1e-12;
    p->gp_cap = 100000; p->refine_cap = 30; p->max_halvings = 50; p->cg_cap = 0;
    p->time_budget_s = 0.0;
    p->precond = 0;
    p->grid_nx = 0; p->grid_ny = 0; p->tile_x = 32; p->tile_y = 32;
    p->trace = NULL; p->trace_cap = 0;
    p->ilu_level = 2;
}

/* Solve min q(x) s.t. l <= x <= u.  tol > 0: absolute tau on ||grad_Omega q||_2
 * (Eq. bqp_approximate_sol, Euclidean norm R4); tol < 0: tau =
 * |tol| * ||A P[x0] - b||_2 (R5).  max_it: outer-iteration cap.  Returns the
 * status; x holds the last feasible iterate. */
int ora_gpcg_solve(int64_t n, const int64_t *rp, const int32_t *ci, const double *val,
                   const double *b, const double *l, const double *u, double c,
                   const double *x0, double tol, int64_t max_it, const ora_params *prm,
                   double *x, ora_stats *st)
{
    double t0 = now_s();
    memset(st, 0, sizeof(*st));
    for (int64_t i = 0; i < n; i++)
        if (!(l[i] <= u[i])) { st->status = ORA_EINVAL; return ORA_EINVAL; }

    double *g = (double *)malloc((size_t)n * sizeof(double));
    double *y = (double *)malloc((size_t)n * sizeof(double));
    double *w = (double *)malloc((size_t)n * sizeof(double));
    double *work = (double *)malloc((size_t)4 * n * sizeof(double));
    double *dinv = prm->precond == 1 ? (double *)malloc((size_t)n * sizeof(double)) : NULL;
    double *ilu = prm->precond >= 2 ? (double *)malloc((size_t)2 * n * sizeof(double)) : NULL;
    ora_iluk iluk;
    memset(&iluk, 0, sizeof iluk);
    if (prm->precond >= 2 && (prm->grid_nx <= 0 || prm->grid_nx * prm->grid_ny != n || prm->tile_x <= 0 ||
                              prm->tile_y <= 0)) {
        free(dinv); free(ilu);
        st->status = ORA_EINVAL; return ORA_EINVAL;
    }
    unsigned char *act = (unsigned char *)malloc((size_t)n);
    unsigned char *fr = (unsigned char *)malloc((size_t)n);
    if (!g || !y || !w || !work || !act || !fr || (prm->precond == 1 && !dinv) || (prm->precond >= 2 && !ilu)) {
        free(g); free(y); free(w); free(work); free(act); free(fr); free(dinv); free(ilu);
        st->status = ORA_ENOMEM; return ORA_ENOMEM;
    }
    int status = ORA_NOT_CONVERGED;

    if (dinv) ora_jacobi_inverse(n, rp, ci, val, dinv);
    /* Setup: x <- P[x0] (Alg. GPCG "Choose x0 in Omega" P:504) */
    ora_project(n, l, u, x0, x);
    gradient(n, rp, ci, val, b, x, g); st->full_spmvs++;
    st->g0_norm = sqrt(dot(n, g, g));
    double tau = tol > 0.0 ? tol : -tol * st->g0_norm;
    st->tau = tau;
    if (pgnorm(n, x, g, l, u) <= tau) { status = ORA_OK; goto done; }

    for (int64_t k = 0; k < max_it; k++) {
        st->outer_iters = k + 1;
        /* ---- gradient projection phase : y_0 = x_k ---------- */
        int64_t j = 0;
        double maxdec = 0.0, alpha_first = 0.0;
        for (;;) {
            /* g = A y_j - b holds here */
            if (pgnorm(n, x, g, l, u) <= tau) {
                trace_put(prm, st, 2, k, j, 0, maxdec, alpha_first);
                status = ORA_OK; goto done;
            }
            int cs;
            double alpha0 = ora_cauchy_alpha(n, rp, ci, val, x, g, l, u, work, &cs);
            st->full_spmvs++;
            if (cs != ORA_OK) { status = cs; goto done; }
            /* direction -grad q (Eq. next-y); identical trial points to the
             * -grad_Omega q reading for feasible y (reading R8) */
            for (int64_t i = 0; i < n; i++) w[i] = -g[i];
            double delta, alpha;
            int64_t h = ora_projected_search(n, rp, ci, val, x, g, w, l, u, alpha0, prm->mu,
                                             prm->max_halvings, y, work, &delta, &alpha);
            if (h < 0) { status = ORA_ESEARCH; goto done; }
            st->full_spmvs += h + 1;
            /* A(y_{j-1}) vs A(y_j), compared as index sets (Eq. pgstop1, R9) */
            int same = 1;
            for (int64_t i = 0; i < n; i++) {
                int a_old = is_active(x[i], l[i], u[i]);
                int a_new = is_active(y[i], l[i], u[i]);
                if (a_old != a_new) { same = 0; break; }
            }
            memcpy(x, y, (size_t)n * sizeof(double));
            j++;
            st->gp_iters++;
            gradient(n, rp, ci, val, b, x, g); st->full_spmvs++;
            double dec = -delta;                            /* q(y_{j-1}) - q(y_j) */
            if (j == 1) alpha_first = alpha0;
            trace_put(prm, st, 1, k, j, h, dec, alpha);
            int reason = same ? 1 :                                      /* Eq. pgstop1 */
                         (j >= 2 && dec <= prm->eta1 * maxdec) ? 2 :     /* Eq. pgstop2 (R10) */
                         (j >= prm->gp_cap) ? 3 : 0;                     /* safety net (R13) */
            if (dec > maxdec) maxdec = dec;
            if (reason) { trace_put(prm, st, 2, k, j, reason, maxdec, alpha_first); break; }
        }
        /* x_k = y_{j_k}; convergence test (R13) */
        if (pgnorm(n, x, g, l, u) <= tau) { status = ORA_OK; goto done; }

        /* ---- CG phase with eta2 refinement ------------------- */
        double eta2 = prm->eta2;
        for (int64_t rep = 0; rep < prm->refine_cap; rep++) {
            int64_t m = 0;
            for (int64_t i = 0; i < n; i++) { fr[i] = !is_active(x[i], l[i], u[i]); m += fr[i]; }
            if (m == 0) break;              /* reading R26: next GP phase frees variables */
            int64_t cap = prm->cg_cap > 0 ? prm->cg_cap : m;
            ora_prec M = {(int)prm->precond, dinv, prm->grid_nx, prm->tile_x, prm->tile_y, ilu, ilu ? ilu + n : NULL,
                          prm->ilu_level, &iluk};
            int64_t its = ora_pcg_m(n, rp, ci, val, fr, g, &M, eta2, cap, w, work, NULL,
                                    prm->time_budget_s > 0.0 ? t0 + prm->time_budget_s : 0.0);
            st->cg_calls++;
            if (its < 0) { status = (int)its; goto done; }
            st->cg_iters += its;
            trace_put(prm, st, 3, k, rep, its, eta2, (double)m);
            /* d_k = Z_k w_{j_k} is w itself (zero off F) */
            double delta, alpha;
            int64_t h = ora_projected_search(n, rp, ci, val, x, g, w, l, u, 1.0, prm->mu,
                                             prm->max_halvings, y, work, &delta, &alpha);
            if (h < 0) { status = ORA_ESEARCH; goto done; }
            st->full_spmvs += h + 1;
            memcpy(x, y, (size_t)n * sizeof(double));
            gradient(n, rp, ci, val, b, x, g); st->full_spmvs++;
            /* Eq. cgstop3: B(x_{k+1}) = A(x_{k+1}) -> reduce eta2, continue CG */
            int64_t nonbinding = 0;
            for (int64_t i = 0; i < n; i++)
                if (is_active(x[i], l[i], u[i]) && !is_binding(x[i], g[i], l[i], u[i])) nonbinding++;
            trace_put(prm, st, 4, k, rep, h, -delta, (double)nonbinding);
            if (pgnorm(n, x, g, l, u) <= tau) { status = ORA_OK; goto done; }
            if (nonbinding != 0) break;
            eta2 = eta2 * prm->eta2_shrink;
            if (eta2 < prm->eta2_floor) eta2 = prm->eta2_floor;
            st->refinements++;
            if (prm->time_budget_s > 0.0 && now_s() - t0 > prm->time_budget_s) goto done;
        }
        if (prm->time_budget_s > 0.0 && now_s() - t0 > prm->time_budget_s) goto done;
    }

done:
    {
        int64_t na = 0, nb = 0;
        ora_sets(n, x, g, l, u, NULL, NULL, &na, &nb);
        st->n_active = na;
        st->n_free = n - na;
        st->n_active_nonbinding = na - nb;
        st->pg_norm = pgnorm(n, x, g, l, u);
        st->q = ora_objective(n, rp, ci, val, b, c, x);
        st->status = status;
        st->seconds = now_s() - t0;
    }
    free(g); free(y); free(w); free(work); free(act); free(fr); free(dinv); free(ilu);
    ora_iluk_free(&iluk);
    return status;
}
