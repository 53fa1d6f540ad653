// kernels.cuh -- the sm_100a kernels of the GPCG hot path.
//
//   a1 k_accept      fused project / accept step / regrad / free mask / sets
//   a2 k_cauchy      Cauchy step alpha_0 = ||d||^2 / <d, A d>, d = grad_Omega q
//   a3 k_search      projected search: K step sizes in one sweep
//   a4 k_hessvec     full or free-set-masked A v (reduced Hessian, in place)
//   a5 k_cg_init / k_cg_iter   single-reduction (Chronopoulos-Gear) CG on A_F
//   a6 reduce_and_finish (common.cuh) deterministic reductions + finalize
//
// Every kernel is templated on the operator (StencilOp | CsrOp) and on scalar
// vs per-point bounds, and streams its vectors once from HBM: neighbour values
// needed by the operator are recomputed on the fly from the inputs at the
// neighbour (so e.g. the accepted step and the new gradient are one sweep).
#pragma once

#include "common.cuh"
#include "fin.cuh"

namespace gpcg {

// ----------------------------------------------------------------------------
// a1: y_out = mid(l, u, y_in + alpha * sgn * dir)   (alpha from the search, or
//     project-only when dir == nullptr: y_out = mid(l, u, y_in))
//     g_out = A y_out - b,  mask_out = [l < y_out < u]
//     sums: ||grad_Omega q||^2 (Eq. proj-gradient), ||g||^2, |A|, #changed
//     (Eq. pgstop1 as index sets, R9), |A \ B| (Eq. cgstop3).
// Skipped entirely (no writes) when the preceding search found no step.
// ----------------------------------------------------------------------------
template <class Op, bool SB>
__global__ void __launch_bounds__(kThreads)
k_accept(Op A, Bounds Bd, const double* __restrict__ y_in, const double* __restrict__ dir,
         double sgn, const double* __restrict__ b, const unsigned char* __restrict__ mask_prev,
         double* __restrict__ y_out, double* __restrict__ g_out, unsigned char* __restrict__ mask_out,
         Scal* S, RedScratch R, int gp) {
    if (gp && gp_skip(S)) return;                    // device-driven GP phase over / k_spec accepted
    double alpha = 0.0;
    if (dir) {
        if (S->s_h < 0) return;          // uniform across the grid
        alpha = S->s_alpha;
    }
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    A.for_each_point([&](const Pt& p) {
        double ax = 0.0, yv = 0.0;
        A.for_each_nbr(p, [&](int c, double a) {
            const double lc = lo<SB>(Bd, c), uc = hi<SB>(Bd, c);
            const double yc = dir ? trial(__ldg(y_in + c), __ldg(dir + c), sgn, alpha, lc, uc)
                                  : mid(lc, uc, __ldg(y_in + c));
            if (c == p.v) yv = yc;
            ax = fma(a, yc, ax);
        });
        const double l = lo<SB>(Bd, p.v), u = hi<SB>(Bd, p.v);
        const double g = ax - __ldg(b + p.v);
        y_out[p.v] = yv;
        g_out[p.v] = g;
        const bool act = (yv == l) || (yv == u);
        const unsigned char m = act ? 0 : 1;
        mask_out[p.v] = m;
        const double pg = pgrad(yv, g, l, u);
        acc[0] = fma(pg, pg, acc[0]);
        acc[1] = fma(g, g, acc[1]);
        acc[2] += act ? 1.0 : 0.0;
        if (mask_prev) acc[3] += (mask_prev[p.v] != m) ? 1.0 : 0.0;
        const bool binding = (yv == l && g >= 0.0) || (yv == u && g <= 0.0);
        acc[4] += (act && !binding) ? 1.0 : 0.0;
    });
    reduce_and_finish<5>(acc, R, [&](double* t) { fin_accept(t, false, S); });
}

// ----------------------------------------------------------------------------
// a2: d = grad_Omega q(y) (formed on the fly at each neighbour); alpha_0 =
//     ||d||^2 / <d, A d>, the minimiser of alpha -> q(y - alpha d) (Eq. bqpls,
//     P:362-374; <g, d> = ||d||^2 since d_i in {g_i, 0}).  Full operator A.
// ----------------------------------------------------------------------------
template <class Op, bool SB>
__global__ void __launch_bounds__(kThreads)
k_cauchy(Op A, Bounds Bd, const double* __restrict__ y, const double* __restrict__ g,
         Scal* S, RedScratch R, int gp) {
    if (gp && *(volatile int*)&S->gp_done) return;   // device-driven GP phase already over
    double acc[2] = {0.0, 0.0};
    A.for_each_point([&](const Pt& p) {
        double ad = 0.0, dv = 0.0;
        A.for_each_nbr(p, [&](int c, double a) {
            const double dc = pgrad(__ldg(y + c), __ldg(g + c), lo<SB>(Bd, c), hi<SB>(Bd, c));
            if (c == p.v) dv = dc;
            ad = fma(a, dc, ad);
        });
        acc[0] = fma(dv, dv, acc[0]);
        acc[1] = fma(dv, ad, acc[1]);
    });
    reduce_and_finish<2>(acc, R, [&](double* t) { fin_cauchy(t, S); });
}

// ----------------------------------------------------------------------------
// a3: projected search sweep.  For h < K, alpha_h = base * 2^-(h0 + h) with
//     base = alpha_0 (GP, Eqs. next-y/gplsstop) or 1 (CG, Eq. cglsstop2):
//     s_h = mid(l, u, y + alpha_h sgn dir) - y;  sums <g, s_h>, <s_h, A s_h>.
//     q(y + s) - q(y) = <g,s> + 1/2 <s,As> exactly (R17).  The finaliser picks
//     the first h with  <g,s_h> + 1/2 <s_h,A s_h> <= mu <g,s_h>  (S->s_h = -1:
//     none in this batch; the host launches the next batch).
// ----------------------------------------------------------------------------
template <class Op, bool SB, int K>
__global__ void __launch_bounds__(kThreads)
k_search(Op A, Bounds Bd, const double* __restrict__ y, const double* __restrict__ g,
         const double* __restrict__ dir, double sgn, int use_alpha0, int h0, double mu,
         Scal* S, RedScratch R, int gp) {
    if (gp && gp_skip(S)) return;                    // device-driven GP phase over / k_spec accepted
    if (use_alpha0 && !S->cauchy_ok) {           // <d,Ad> <= 0: no step (host reports ENOTSPD)
        if (blockIdx.x == 0 && threadIdx.x == 0) S->s_h = -1;
        return;
    }
    const double base = use_alpha0 ? S->alpha0 : 1.0;
    double al[K];
#pragma unroll
    for (int h = 0; h < K; ++h) al[h] = scalbn(base, -(h0 + h));
    double acc[2 * K];
#pragma unroll
    for (int s = 0; s < 2 * K; ++s) acc[s] = 0.0;
    A.for_each_point([&](const Pt& p) {
        double as[K], sv[K];
#pragma unroll
        for (int h = 0; h < K; ++h) { as[h] = 0.0; sv[h] = 0.0; }
        A.for_each_nbr(p, [&](int c, double a) {
            const double yc = __ldg(y + c), dc = __ldg(dir + c);
            const double lc = lo<SB>(Bd, c), uc = hi<SB>(Bd, c);
            const bool self = (c == p.v);
#pragma unroll
            for (int h = 0; h < K; ++h) {
                const double s = trial(yc, dc, sgn, al[h], lc, uc) - yc;
                if (self) sv[h] = s;
                as[h] = fma(a, s, as[h]);
            }
        });
        const double gv = __ldg(g + p.v);
#pragma unroll
        for (int h = 0; h < K; ++h) {
            acc[2 * h] = fma(gv, sv[h], acc[2 * h]);
            acc[2 * h + 1] = fma(sv[h], as[h], acc[2 * h + 1]);
        }
    });
    reduce_and_finish<2 * K>(acc, R, [&](double* t) { fin_search(t, K, h0, base, mu, S); });
}

// ----------------------------------------------------------------------------
// a1 + a3 speculative (generic operators: CSR, 3-D): a projected-search step at h = 0 and its
// accept in ONE sweep.  GP phase: alpha = alpha_0 along -g (Eq. next-y); CG phase: alpha = 1
// along w (Eq. cglsstop2).  At the point and its neighbours (pointwise):
//   y'_c = mid(l, u, y_c + alpha sgn dir_c),  s_c = y'_c - y_c;
//   g' = A y' - b,  A s,  mask' = [l < y' < u];
//   sums <g, s>, <s, A s> (the search's h = 0 sums) and the accept sums of y'.
// Each quantity with the arithmetic (and order of operator terms) of k_search / k_accept, so the
// result is bit for bit theirs: fin_spec keeps the step when q(y') - q(y) = <g,s> + 1/2 <s,As>
// <= mu <g,s> (the step's search / accept sweeps then return at once), otherwise they run from
// h = 1 and overwrite y', g', mask' (the next ping-pong buffers).  One sweep instead of two per
// accepted step; the next Cauchy step cannot join (d' needs g' at the neighbours' neighbours).
// ----------------------------------------------------------------------------
template <class Op, bool SB>
__global__ void __launch_bounds__(kThreads)
k_spec(Op A, Bounds Bd, const double* __restrict__ y, const double* __restrict__ dir, double sgn, int use_alpha0,
       const double* __restrict__ g, const double* __restrict__ b, double* __restrict__ y_out,
       double* __restrict__ g_out, unsigned char* __restrict__ mask_out, double mu, Scal* S, RedScratch R, int gp) {
    if (gp && *(volatile int*)&S->gp_done) return;
    if (use_alpha0 && !S->cauchy_ok) {            // <d,Ad> <= 0: no step (uniform; k_finalize mirrors it)
        if (blockIdx.x == 0 && threadIdx.x == 0) { S->spec_ok = 0; S->s_h = -1; }
        return;
    }
    const double alpha = use_alpha0 ? S->alpha0 : 1.0;
    double acc[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    A.for_each_point([&](const Pt& p) {
        double ax = 0.0, as = 0.0, sv = 0.0, yn = 0.0;
        A.for_each_nbr(p, [&](int c, double a) {
            const double yc = __ldg(y + c);
            const double tc = trial(yc, __ldg(dir + c), sgn, alpha, lo<SB>(Bd, c), hi<SB>(Bd, c));
            const double sc = tc - yc;
            if (c == p.v) { sv = sc; yn = tc; }
            ax = fma(a, tc, ax);
            as = fma(a, sc, as);
        });
        const double l = lo<SB>(Bd, p.v), u = hi<SB>(Bd, p.v);
        const double yv = __ldg(y + p.v), gv = __ldg(g + p.v);
        const double gn = ax - __ldg(b + p.v);
        y_out[p.v] = yn;
        g_out[p.v] = gn;
        const bool act = (yn == l) || (yn == u);
        mask_out[p.v] = act ? 0 : 1;
        const bool act_prev = (yv == l) || (yv == u);     // = !mask(y): y is feasible
        acc[0] = fma(gv, sv, acc[0]);
        acc[1] = fma(sv, as, acc[1]);
        const double pg = pgrad(yn, gn, l, u);
        acc[2] = fma(pg, pg, acc[2]);
        acc[3] = fma(gn, gn, acc[3]);
        acc[4] += act ? 1.0 : 0.0;
        acc[5] += (act_prev != act) ? 1.0 : 0.0;
        const bool binding = (yn == l && gn >= 0.0) || (yn == u && gn <= 0.0);
        acc[6] += (act && !binding) ? 1.0 : 0.0;
    });
    const double base = alpha;
    reduce_and_finish<7>(acc, R, [&](double* t) { fin_spec(t, base, mu, S); });
}

// ----------------------------------------------------------------------------
// a4: y = A v (reduced = false) or y = Z Z' A Z Z' v on the free mask
//     (reduced = true), A_k = Z'AZ applied in place.
// ----------------------------------------------------------------------------
template <class Op, bool kReduced>
__global__ void __launch_bounds__(kThreads)
k_hessvec(Op A, const double* __restrict__ v, double* __restrict__ y,
          const unsigned char* __restrict__ mask) {
    A.for_each_point([&](const Pt& p) {
        double r = 0.0;
        if (!kReduced || mask[p.v]) {
            A.for_each_nbr(p, [&](int c, double a) {
                if (kReduced && !mask[c]) return;
                r = fma(a, __ldg(v + c), r);
            });
        }
        y[p.v] = r;
    });
}

// q(x) = 1/2 x'Ax - b'x + c: sums x'(Ax) and b'x.
template <class Op>
__global__ void __launch_bounds__(kThreads)
k_objective(Op A, const double* __restrict__ x, const double* __restrict__ b, Scal* S, RedScratch R) {
    double acc[2] = {0.0, 0.0};
    A.for_each_point([&](const Pt& p) {
        double ax = 0.0;
        A.for_each_nbr(p, [&](int c, double a) { ax = fma(a, __ldg(x + c), ax); });
        const double xv = __ldg(x + p.v);
        acc[0] = fma(xv, ax, acc[0]);
        acc[1] = fma(__ldg(b + p.v), xv, acc[1]);
    });
    reduce_and_finish<2>(acc, R, [&](double* t) { S->r0 = t[0]; S->r1 = t[1]; });
}

// ----------------------------------------------------------------------------
// a5: CG on A_k w = -r_k (Eq. cg2), w_0 = 0 (Alg. GPCG), in the
// Chronopoulos-Gear single-reduction form (same iterates as textbook CG in
// exact arithmetic, reading R19).  Notation: rho = residual -(r + A_k w),
// q = A_F rho, p = direction, s = A_F p, all zero off F.
//
// init: rho_0 = -[v in F] g_v;  q_0 = A_F rho_0;  gamma_0 = rho_0'rho_0,
//       delta_0 = rho_0'q_0;  alpha_0 = gamma_0/delta_0, beta_0 = 0.
// iter i:  p_i = rho_i + beta_i p_{i-1}      s_i = q_i + beta_i s_{i-1}
//          w_{i+1} = w_i + alpha_i p_i       rho_{i+1} = rho_i - alpha_i s_i
//          q_{i+1} = A_F rho_{i+1}  (rho_{i+1} at neighbours formed on the fly)
//          gamma_{i+1} = rho'rho, delta_{i+1} = rho'q  -> one reduction
// finalize (last block), j = i+1, decrease of step j = 1/2 alpha_i gamma_i:
//   stop if j >= 2 and dec_j <= eta2 max_{l<j} dec_l  (Eq. cgstop1, R10)
//        or ||rho_j|| <= 1e-14 (1 + ||r_k||)         (S:371 guard)
//        or j >= cap;
//   else beta = gamma_j/gamma_i, alpha = gamma_j / (delta_j - beta gamma_j/alpha_i)
//        (= gamma_j / <p_j, A_k p_j>; <= 0 -> ENOTSPD).
// rho, q, s ping-pong between two buffers (neighbours read the old values);
// p and w are updated in place.  After cg_done every launch is a no-op.
// ----------------------------------------------------------------------------
// PC: point-Jacobi PCG with dinv = 1 / diag(A) (k_jacobi_inverse): u = dinv * rho, q = A_F u,
// gamma = rho'u, delta = u'q; p_i = u_i + beta p_{i-1}.
template <class Op, bool PC>
__global__ void __launch_bounds__(kThreads)
k_cg_init(Op A, const double* __restrict__ g, const unsigned char* __restrict__ mask,
          unsigned char* __restrict__ mask_cg, double* __restrict__ rho, double* __restrict__ q, double* __restrict__ s,
          double* __restrict__ rho2, double* __restrict__ q2, double* __restrict__ s2,
          double* __restrict__ p, double* __restrict__ w, const double* __restrict__ dinv, double eta2, long long cap,
          Scal* S, RedScratch R) {
    double acc[2] = {0.0, 0.0};
    A.for_each_point([&](const Pt& pt) {
        const int v = pt.v;
        const unsigned char mv = mask[v];
        mask_cg[v] = mv;                       // the CG graph reads this fixed buffer
        p[v] = 0.0; w[v] = 0.0; s[v] = 0.0;
        rho2[v] = 0.0; q2[v] = 0.0; s2[v] = 0.0;
        if (!mv) { rho[v] = 0.0; q[v] = 0.0; return; }
        double qv = 0.0, uv = 0.0;
        A.for_each_nbr(pt, [&](int c, double a) {
            const double rc = mask[c] ? -__ldg(g + c) : 0.0;
            const double uc = PC ? rc * __ldg(dinv + c) : rc;
            if (c == v) uv = uc;
            qv = fma(a, uc, qv);
        });
        const double rv = -__ldg(g + v);
        rho[v] = rv;
        q[v] = qv;
        acc[0] = fma(rv, uv, acc[0]);
        acc[1] = fma(uv, qv, acc[1]);
    });
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_init_finalize(t[0], t[1], eta2, cap, S); });
}

template <class Op, bool PC>
__global__ void __launch_bounds__(kThreads)
k_cg_iter(Op A, const unsigned char* __restrict__ mask,
          const double* __restrict__ rho, const double* __restrict__ q, const double* __restrict__ s,
          double* __restrict__ rho_n, double* __restrict__ q_n, double* __restrict__ s_n,
          double* __restrict__ p, double* __restrict__ w, const double* __restrict__ dinv, Scal* S, RedScratch R) {
    if (*(volatile int*)&S->cg_done) return;
    const double alpha = S->cg_alpha, beta = S->cg_beta;
    double acc[2] = {0.0, 0.0};
    A.for_each_point([&](const Pt& pt) {
        const int v = pt.v;
        if (!mask[v]) return;
        const double rv = rho[v], qv = q[v], sv = s[v];
        const double pn = fma(beta, p[v], PC ? rv * __ldg(dinv + v) : rv);
        const double sn = fma(beta, sv, qv);
        w[v] = fma(alpha, pn, w[v]);
        p[v] = pn;
        s_n[v] = sn;
        double rnv = 0.0, unv = 0.0, qn = 0.0;
        A.for_each_nbr(pt, [&](int c, double a) {
            double uc;
            if (c == v) {
                rnv = fma(-alpha, sn, rv);
                unv = PC ? rnv * __ldg(dinv + v) : rnv;
                uc = unv;
            } else {
                if (!mask[c]) return;
                const double rc = fma(-alpha, fma(beta, s[c], q[c]), rho[c]);
                uc = PC ? rc * __ldg(dinv + c) : rc;
            }
            qn = fma(a, uc, qn);
        });
        rho_n[v] = rnv;
        q_n[v] = qn;
        acc[0] = fma(rnv, unv, acc[0]);
        acc[1] = fma(unv, qn, acc[1]);
    });
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_finalize(t[0], t[1], S); });
}

// 1 / A_vv for every owned point (point-Jacobi preconditioner)
template <class Op>
__global__ void __launch_bounds__(kThreads)
k_jacobi_inverse(Op A, double* __restrict__ dinv) {
    A.for_each_point([&](const Pt& p) {
        double d = 0.0;
        A.for_each_nbr(p, [&](int c, double a) { if (c == p.v) d += a; });
        dinv[p.v] = 1.0 / d;
    });
}

// #entries of the owned rows that differ from row[] (the row-broadcast test for b)
__global__ void __launch_bounds__(kThreads)
k_count_row_mismatch(int cols, int rows, int pitch, const double* __restrict__ a, const double* __restrict__ row,
                     Scal* S, RedScratch R) {
    double acc[2] = {0.0, 0.0};
    const long long n = (long long)cols * rows;
    for (long long k = blockIdx.x * (long long)kThreads + threadIdx.x; k < n; k += (long long)gridDim.x * kThreads) {
        const long long i = k % cols, v = i + (k / cols) * (long long)pitch;
        acc[0] += (a[v] != row[i]) ? 1.0 : 0.0;
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { S->r0 = t[0]; S->r1 = t[1]; });
}

// ----------------------------------------------------------------------------
// input validation at create: #(l > u or NaN), #(b NaN), l / u constant?
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
k_check_inputs(int cols, int rows, int pitch, const double* __restrict__ b, const double* __restrict__ l,
               const double* __restrict__ u, const double* __restrict__ lu0, Scal* S, RedScratch R) {
    // sums: #bad entries, #entries differing from the global first (l, u) pair lu0
    double acc[2] = {0.0, 0.0};
    const double l0 = lu0[0], u0 = lu0[1];
    const long long n = (long long)cols * rows;
    for (long long k = blockIdx.x * (long long)kThreads + threadIdx.x; k < n; k += (long long)gridDim.x * kThreads) {
        const long long v = (k % cols) + (k / cols) * (long long)pitch;
        const double lv = l[v], uv = u[v], bv = b[v];
        acc[0] += (!(lv <= uv) || isnan(bv) || isinf(bv) || lv == INFINITY || uv == -INFINITY) ? 1.0 : 0.0;
        acc[1] += (lv != l0 || uv != u0) ? 1.0 : 0.0;
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { S->r0 = t[0]; S->r1 = t[1]; });
}

// create-time validation of a one-slab CSR operator uploaded as given: r0 = #rows with
// row_ptr[i + 1] < row_ptr[i], r1 = #column indices outside [0, n)
__global__ void k_check_csr(long long n, const long long* __restrict__ rp, const int* __restrict__ ci, long long nnz,
                            Scal* S, RedScratch R) {
    double acc[2] = {0.0, 0.0};
    const long long t0 = blockIdx.x * (long long)kThreads + threadIdx.x, st = (long long)gridDim.x * kThreads;
    for (long long i = t0; i < n; i += st) acc[0] += (rp[i + 1] < rp[i]) ? 1.0 : 0.0;
    for (long long k = t0; k < nnz; k += st) acc[1] += (ci[k] < 0 || ci[k] >= n) ? 1.0 : 0.0;
    reduce_and_finish<2>(acc, R, [&](double* t) { S->r0 = t[0]; S->r1 = t[1]; });
}

__global__ void k_count_nonfinite(long long n, const double* __restrict__ a, Scal* S, RedScratch R) {
    double acc[2] = {0.0, 0.0};
    for (long long v = blockIdx.x * (long long)kThreads + threadIdx.x; v < n; v += (long long)gridDim.x * kThreads)
        acc[0] += isfinite(a[v]) ? 0.0 : 1.0;
    reduce_and_finish<2>(acc, R, [&](double* t) { S->r0 = t[0]; S->r1 = t[1]; });
}

}  // namespace gpcg
