/*
 * gpcg.h -- C ABI of the B200-native GPCG hot path (libgpcg.so).
 *
 * Method: GPCG, gradient projection + conjugate gradients for bound-
 * constrained strictly convex QPs, as studied in Benson, McInnes, More,
 * "GPCG: a case study in the performance and scalability of optimization
 * algorithms" (reference PAPER.md; citations "P:a-b" are PAPER.md lines).
 *
 * Problem (Eqs. def_bqp / def_bounds / def-quadratic):
 *
 *     minimise  q(x) = 1/2 x'Ax - b'x + c   subject to  l <= x <= u
 *
 * A symmetric positive definite, l_i in [-inf, inf), u_i in (-inf, +inf],
 * l_i <= u_i (l_i = u_i allowed: a fixed variable).  NOTE the sign: the paper
 * writes +b'x; this ABI follows BASELINE.json and writes -b'x, so
 * b_abi = -b_paper (reading R1).  Gradient g(x) = Ax - b.
 *
 * API shape follows the paper's Fig. 1: create the problem from
 * (A, b, c) and bounds (l, u), solve, destroy.
 *
 * Pointers: every array argument may be HOST memory or DEVICE memory of the
 * handle's device (detected with cudaPointerGetAttributes); host arrays are
 * staged through library-owned device buffers.  fp64 throughout.
 * Ownership: create copies every input into library-owned device memory; the
 * caller keeps ownership of all arrays passed in or out.
 * Streams: all device work is enqueued on the `cuda_stream` passed to create
 * (a cudaStream_t; NULL = the legacy default stream).  solve, project and
 * objective synchronise that stream before returning; hessvec with device
 * pointers is asynchronous (argument errors return immediately, device faults
 * surface at the next synchronising call).
 * Errors: functions never abort or throw; they return a gpcg_status and
 * gpcg_last_error() holds a thread-local message.  There is no CPU fallback:
 * without a CUDA device create returns GPCG_ECUDA.
 * Threading: one handle is used from one host thread at a time.
 * Determinism: results are bitwise reproducible for a fixed (inputs, params,
 * device, build): every reduction is a fixed-order two-stage tree, no float
 * atomics.
 */
#ifndef GPCG_H
#define GPCG_H

#include <stdint.h>

#if defined(__GNUC__)
#define GPCG_API __attribute__((visibility("default")))
#else
#define GPCG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gpcg_problem gpcg_problem; /* opaque; library-owned */

/* return codes */
enum {
    GPCG_OK = 0,
    GPCG_NOT_CONVERGED = 1, /* >0: result valid (feasible), max_it reached       */
    GPCG_EINVAL = -1,       /* bad argument, l_i > u_i, NaN in inputs            */
    GPCG_ENOMEM = -2,       /* device allocation failed                          */
    GPCG_ECUDA = -3,        /* CUDA runtime error / no device                    */
    GPCG_ENCCL = -4,        /* NCCL failure / not loadable (multi-rank path)     */
    GPCG_ENOTSPD = -5,      /* <d,Ad> <= 0 or <p,A_k p> <= 0: A not SPD          */
    GPCG_ESEARCH = -6,      /* projected search found no step in max_halvings    */
    GPCG_ESTATE = -7        /* e.g. reduced hessvec before any project/solve     */
};

/* Algorithm constants (P:788-793 gives eta1 = 0.1, eta2 = 0.05; the others are
 * DESIGN.md readings R6, R12, R13).  Obtain defaults from gpcg_params_default. */
typedef struct {
    double mu;           /* sufficient decrease, Eqs. gplsstop/cglsstop2, in (0,1/2): 0.1 */
    double eta1;         /* Eq. pgstop2: 0.1                                               */
    double eta2;         /* Eq. cgstop1: 0.05                                              */
    double eta2_shrink;  /* Eq. cgstop3 refinement factor: 0.1                             */
    double eta2_floor;   /* 1e-12                                                          */
    int64_t gp_cap;      /* GP iterates per phase: 100000, a safety net (the paper has none)*/
    int64_t refine_cap;  /* cgstop3 repetitions per outer iterate: 30                      */
    int64_t max_halvings;/* projected-search trials: 50                                    */
    int64_t cg_cap;      /* CG iterations per call, 0 => m_k (finite termination P:444-447)*/
    int32_t search_k;    /* step sizes in the first search sweep: 2 (<=2 -> 2, else 8); retries use 8 */
    int32_t cg_chunk;    /* CG iterations per graph launch between host polls: 32          */
    int32_t gp_chunk;    /* GP steps per graph launch between host polls: 8                */
    int32_t precond;     /* 0: plain CG on A_k (the hot path); 1: point-Jacobi PCG with
                            M = diag(A_k) (Table 4 "Diagonal"); 2: block-
                            Jacobi ILU(0) on 32 x 32 tiles of each slab (
                            2-D stencils only, textbook PCG, two sweeps per iteration);
                            3: block-Jacobi ILU(2) on the same tiles (the
                            subdomain solver of the paper's Tables 1-3, "two levels of
                            fill"; 2-D stencils only)                                      */
    int32_t cg_mode;     /* 0: A_k applied in place on masked full-length vectors (the hot
                            path, P:680-683's "alternative technique"); 1: A_k extracted
                            as a compact CSR matrix each CG call, as the paper does with
                            PETSc -- the extraction ablation; one slab / rank;
                            3: A_k applied in place over the compacted free-row list (the
                            CG and the reduced hessvec touch only the free rows; CSR / 3-D
                            operators, one slab / rank); 2 (default): 3 for CSR / 3-D
                            operators with |F| < 0.3 n on one slab and rank, else 0       */
} gpcg_params;

typedef struct {
    int64_t outer_iters;  /* GPCG iterates (Table 1 "iters")                         */
    int64_t gp_iters;     /* gradient-projection iterates (Table 1 n_GP, reading R22) */
    int64_t cg_iters;     /* CG iterations = reduced Hessian-vector products          */
    int64_t cg_calls;     /* CG solves (one per CG phase / refinement)               */
    int64_t refinements;  /* Eq. cgstop3 eta2 reductions                             */
    int64_t full_spmvs;   /* full-operator applications (gradients, searches)        */
    int64_t n_free, n_active, n_active_nonbinding;
    double pg_norm;       /* ||grad_Omega q(x)||_2 at return                         */
    double q;             /* q(x) at return                                          */
    double g0_norm;       /* ||A P[x0] - b||_2                                       */
    double tau;           /* the absolute tolerance used                             */
    double t_total_ms, t_cg_ms, t_gp_ms;  /* CUDA-event times (CG chunks, GP sweeps) */
    int32_t status;
    int32_t kernel_launches; /* library kernels launched during the call (low 31 bits) */
    /* CG timing: CUDA events around every persistent CG launch (one slab, one rank:
     * the whole call) or, on the graph-chunk path (slabs / ranks), around every chunk
     * in which no iteration had finished; cg_iters_timed iterations took
     * t_cg_timed_ms of device time; cg_free_iters_timed = sum of |F| over them. */
    int64_t cg_iters_timed, cg_free_iters_timed;
    double t_cg_timed_ms;
    double t_extract_ms;   /* cg_mode = 1: device time spent building A_F and r_F          */
    /* GP phase sweeps (2-D persistent GP loop): gp_spec_rejected = GP steps whose speculative
     * accept sweep at alpha_0 was rejected by Eq. gplsstop (each then ran a search sweep and
     * an accept sweep as well); 0 on the other paths. */
    int64_t gp_spec_rejected;
} gpcg_stats;

GPCG_API gpcg_params gpcg_params_default(void);

/*
 * Row-slab distribution (the paper's row-block distribution of
 * A, b, l, u over processes, without its redistribution
 * of A_k after every free-set change).  One process per GPU; rank r
 * owns the contiguous global rows [row_begin, row_end): grid rows j for
 * stencil2d (each nx unknowns), matrix rows for CSR.  Ranks must cover the
 * rows in rank order (rank 0 first).  Every rank calls every function with its
 * own slab (same sequence on all ranks); user arrays hold the rank's rows only.
 * Each operator application reads ghost rows of the neighbouring ranks
 * (stencil2d: 3 grid rows; stencil3d: 1 plane; CSR: the band of rows its columns reach -- columns of
 * a rank may only refer to rows of itself and of ranks r-1, r+1), exchanged by
 * NCCL send/recv after every sweep that writes a vector a neighbour reads, and
 * every global sum is one ncclAllReduce (one per CG iteration, one per search
 * and accept sweep).  NCCL is the process's own libnccl.so.2, bound at run time.
 *   rank, nranks: this process's rank, number of ranks (1 = single process).
 *   nccl_id:      128-byte ncclUniqueId from gpcg_nccl_unique_id on rank 0,
 *                 identical on every rank (broadcast it, e.g. with
 *                 torch.distributed); ignored when nranks == 1.
 *   local_slabs:  >= 1; > 1 splits this rank's rows further into that many
 *                 slabs on the same device, exchanging ghost rows by device
 *                 copies and summing slab totals in slab order -- the same
 *                 arithmetic as nranks * local_slabs ranks (used to test the
 *                 slab path on one GPU).  stencil2d with broadcast faces: the
 *                 slabs of one device run the CG call / GP phase as ONE
 *                 persistent launch whose sweeps write their neighbours' ghost
 *                 rows directly (no exchange step).
 * Environment GPCG_XRANK=1 (read at create; stencil2d with broadcast faces, up
 * to 8 ranks): those persistent launches span the ranks -- each rank maps its
 * neighbours' ghost rows and every rank's counters / partial-sum mailbox over
 * CUDA IPC (exported and all-gathered over the NCCL communicator at create),
 * one NVLink round trip per global sum; the memory pool is off.  Built, not yet
 * run on several GPUs.
 * Errors: GPCG_EINVAL for a bad range or a slab of < 3 stencil2d rows (< 1 plane
 * / CSR row) or a CSR band beyond the neighbouring slab; GPCG_ENCCL if NCCL fails
 * (GPCG_XRANK: also if ncclAllGather is missing); GPCG_ECUDA if a CUDA IPC call
 * fails or a cross-rank wait exceeds 20 s.
 */
typedef struct {
    int32_t rank, nranks;
    const void *nccl_id;
    int64_t row_begin, row_end;
    int32_t local_slabs;
} gpcg_dist;

/* Balanced contiguous split: part k of `parts` gets [begin, end) of [0, total)
 * (host-only helper; the split gpcg_dist's local_slabs uses internally). */
GPCG_API void gpcg_partition_rows(int64_t total, int32_t parts, int32_t part, int64_t *begin, int64_t *end);

/* ncclGetUniqueId of the process's NCCL into out128 (128 bytes).  GPCG_ENCCL
 * if libnccl.so.2 cannot be loaded. */
GPCG_API int gpcg_nccl_unique_id(void *out128);

/*
 * gpcg_create_stencil2d -- A is the 5-point face-weight operator on an nx x ny
 * grid (BASELINE.json configs[0-3]; the paper's journal-bearing discretisation
 * P:742-779 under reading R2).  Grid point (i, j), 0-based, linear index
 * v = i + nx*j (i fastest).
 *   wx: x-face weights, nx+1 per grid row; wx[j*wx_ld + k] joins points
 *       (k-1, j) and (k, j); k = 0 and k = nx are Dirichlet boundary faces.
 *       wx_ld = 0: one row of nx+1 weights broadcast to every grid row;
 *       otherwise wx_ld >= nx+1 and wx holds ny rows.
 *   wy: y-face weights, ny+1 face rows of nx; wy[f*wy_ld + i] joins (i, f-1)
 *       and (i, f).  wy_ld = 0: one row of nx broadcast; else wy_ld >= nx.
 *   shift: nullable diagonal added to A (n entries).
 *   (Ap)_v = (w_W + w_E + w_S + w_N + shift_v) p_v - w_W p_{v-1} - w_E p_{v+1}
 *            - w_S p_{v-nx} - w_N p_{v+nx}   (missing neighbours are 0).
 *   Weights must be finite and >= 0 with A SPD (e.g. all > 0); not checked
 *   beyond finiteness -- non-SPD operators surface as GPCG_ENOTSPD in solve.
 *   b, l, u: n entries each.  c: constant term.
 * Returns GPCG_EINVAL on nx,ny <= 0, n >= 2^31, bad ld, l_i > u_i or NaN.
 */
GPCG_API int gpcg_create_stencil2d(gpcg_problem **out, void *cuda_stream, int64_t nx, int64_t ny,
                          const double *wx, int64_t wx_ld, const double *wy, int64_t wy_ld,
                          const double *shift, const double *b, const double *l,
                          const double *u, double c);

/*
 * gpcg_create_stencil2d_dist -- as gpcg_create_stencil2d for the rank's slab
 * (gpcg_dist above; NULL = the whole grid on one slab).  ny is the GLOBAL
 * number of grid rows; b, l, u, shift hold the rank's rows (row_end-row_begin)
 * * nx entries; wx (wx_ld != 0) the rank's grid rows; wy (wy_ld != 0) the
 * face rows row_begin .. row_end inclusive (row_end-row_begin+1 rows, so the
 * face row shared by two ranks is passed by both).  Broadcast faces (ld 0)
 * are passed whole by every rank.
 */
GPCG_API int gpcg_create_stencil2d_dist(gpcg_problem **out, const gpcg_dist *dist, void *cuda_stream, int64_t nx,
                               int64_t ny, const double *wx, int64_t wx_ld, const double *wy, int64_t wy_ld,
                               const double *shift, const double *b, const double *l, const double *u, double c);

/*
 * gpcg_create_stencil3d -- A is the 3-D 7-point face-weight operator on an
 * nx x ny x nz grid (C4's operator without CSR
 * storage), the 3-D analogue of gpcg_create_stencil2d: A = sum over faces of
 * w_f (e_a - e_b)(e_a - e_b)', boundary faces w_f e_a e_a', plus diag(shift).
 * Point (i, j, k) <-> v = i + nx (j + ny k).  Full face arrays:
 *   wx[(k ny + j)(nx+1) + i'] joins (i'-1, j, k)-(i', j, k), i' = 0..nx;
 *   wy[(k (ny+1) + j') nx + i] joins (i, j'-1, k)-(i, j', k), j' = 0..ny;
 *   wz[k' nx ny + j nx + i]   joins (i, j, k'-1)-(i, j, k'), k' = 0..nz.
 * shift nullable (n).  b, l, u: n.  Errors as gpcg_create_stencil2d.
 * gpcg_create_stencil3d_dist: slabs of z-planes (gpcg_dist rows = planes; one
 * ghost plane per side); wx, wy, b, l, u, shift hold the rank's planes, wz its
 * face planes row_begin .. row_end inclusive.
 */
GPCG_API int gpcg_create_stencil3d(gpcg_problem **out, void *cuda_stream, int64_t nx, int64_t ny, int64_t nz,
                          const double *wx, const double *wy, const double *wz, const double *shift,
                          const double *b, const double *l, const double *u, double c);
GPCG_API int gpcg_create_stencil3d_dist(gpcg_problem **out, const gpcg_dist *dist, void *cuda_stream, int64_t nx,
                               int64_t ny, int64_t nz, const double *wx, const double *wy, const double *wz,
                               const double *shift, const double *b, const double *l, const double *u, double c);

/*
 * gpcg_create_csr -- A given in CSR with BOTH triangles stored:
 * row_ptr[n+1] (int64, row_ptr[0] = 0), col[nnz] (int32, sorted within each
 * row, 0 <= col < n), val[nnz] (fp64).  The paper's PETSc "standard
 * compressed, sparse row" format.  Symmetry is the
 * caller's contract (not checked).  Returns GPCG_EINVAL on n <= 0,
 * n >= 2^31, a non-monotone row_ptr, l_i > u_i or NaN.
 */
GPCG_API int gpcg_create_csr(gpcg_problem **out, void *cuda_stream, int64_t n, const int64_t *row_ptr,
                    const int32_t *col, const double *val, const double *b, const double *l,
                    const double *u, double c);

/*
 * gpcg_create_csr_dist -- as gpcg_create_csr for the rank's rows: n is the
 * GLOBAL size; row_ptr has row_end-row_begin+1 entries (row_ptr[0] = 0), col
 * holds GLOBAL column ids, val, b, l, u the rank's rows.
 */
GPCG_API int gpcg_create_csr_dist(gpcg_problem **out, const gpcg_dist *dist, void *cuda_stream, int64_t n,
                         const int64_t *row_ptr, const int32_t *col, const double *val, const double *b,
                         const double *l, const double *u, double c);

/* Replace the algorithm constants (validated: 0 < mu < 1/2, 0 < eta1, eta2 < 1, ...). */
GPCG_API int gpcg_set_params(gpcg_problem *h, const gpcg_params *p);

/*
 * gpcg_solve -- Algorithm GPCG from x0 (projected first).
 *   tol > 0: stop when ||grad_Omega q(x)||_2 <= tol (Eq. bqp_approximate_sol
 *            P:296-299, Euclidean norm R4);
 *   tol < 0: tau = |tol| * ||A P[x0] - b||_2 (BASELINE.json convention, R5).
 *   max_it:  outer-iteration cap.
 *   x_out:   n entries (host or device), receives the last feasible iterate
 *            (also on GPCG_NOT_CONVERGED, GPCG_ESEARCH, GPCG_ENOTSPD).
 *   stats:   nullable.
 * Records the free set of x_out for gpcg_hessvec(reduced = 1).
 */
GPCG_API int gpcg_solve(gpcg_problem *h, const double *x0, double tol, int64_t max_it, double *x_out,
               gpcg_stats *stats);

/*
 * gpcg_hessvec -- y = A v (reduced = 0), or the reduced Hessian product
 * y = Z Z' A Z Z' v on the free set F recorded by the last gpcg_project or
 * gpcg_solve (reduced = 1): A_k = Z_k' A Z_k, P:411-442 (Eq. cg2), applied
 * in place with no extraction (the "alternative technique" of P:680-683).
 * v is read only on F and y is 0 off F.  Returns GPCG_ESTATE if reduced = 1
 * and no free set has been recorded.  v, y: n entries, must not alias.
 */
GPCG_API int gpcg_hessvec(gpcg_problem *h, const double *v, double *y, int reduced);

/*
 * gpcg_free_count -- |F| of the free set recorded by the last gpcg_project /
 * gpcg_solve, or -1 if none is recorded or the handle has no
 * compacted free-row list (2-D stencils, several slabs or ranks).
 */
GPCG_API int64_t gpcg_free_count(gpcg_problem *h);

/*
 * gpcg_hessvec_free -- the reduced Hessian product in the reduced space:
 * y_free[k] = (A_k Z_k' v)_k = sum_{j in F} A_{f_k j} v_j for k < |F|, where
 * F = [f_0 < f_1 < ...] is the recorded free set in index order and
 * A_k = Z_k' A Z_k (Eq. cg2).  Applied in place over the
 * compacted free-row list (the "alternative technique"; SURVEY
 * 8(a) a4 (iii)): only the free rows of A are read, no extraction, no n-long
 * output.  v: n entries (read on F only); y_free: gpcg_free_count(h)
 * entries; host or device, must not alias.  CSR and 3-D stencil handles on
 * one slab and rank (GPCG_EINVAL otherwise); GPCG_ESTATE if no free set has
 * been recorded.  Equals gpcg_hessvec(reduced = 1) at the free rows, bit for bit.
 */
GPCG_API int gpcg_hessvec_free(gpcg_problem *h, const double *v, double *y_free);

/*
 * gpcg_project -- px = P[x] = mid(l, u, x) and records its free
 * set F = {i : l_i < px_i < u_i}.  Optional outputs (nullable):
 * ||grad_Omega q(px)||_2^2 (Eq. proj-gradient), |A(px)| and
 * |A(px) \ B(px)| (active but not binding).
 */
GPCG_API int gpcg_project(gpcg_problem *h, const double *x, double *px, double *pg_norm2,
                 int64_t *n_active, int64_t *n_active_nonbinding);

/* q(x) = 1/2 x'Ax - b'x + c for any x (no projection). */
GPCG_API int gpcg_objective(gpcg_problem *h, const double *x, double *q);

/* Entries owned by this handle (n; the rank's rows with gpcg_dist). */
GPCG_API int64_t gpcg_size(const gpcg_problem *h);

GPCG_API void gpcg_destroy(gpcg_problem *h);

/* Thread-local message of the last error ("" if none). */
GPCG_API const char *gpcg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* GPCG_H */
