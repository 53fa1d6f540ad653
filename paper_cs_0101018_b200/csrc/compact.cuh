// compact.cuh -- the reduced Hessian applied IN PLACE over a compacted free-row list (SURVEY.md
// 8(a) a4 (iii); the paper's "alternative technique" of running CG on the full operator
// restricted to the free index set) for the small-free regime (C4: ~5 % free).
//
// F = [v_0 < v_1 < ... < v_{m-1}], the free points of the current mask in owned-point order,
// is built by the deterministic prefix sums of extract.cuh (k_scan_*).  The kernels iterate
// k < m with v = F[k] instead of every point: A's rows are read in place (no copy of its
// values, unlike the extraction ablation), the CG vectors stay full-length and zero off F
// (neighbour values are read only where the mask says free), so a CG iteration touches the
// free rows and their neighbours only -- O(m) instead of O(n) work and bytes.  Same arithmetic
// (and order of the operator terms) as k_cg_init / k_cg_iter / k_hessvec of kernels.cuh.
#pragma once

#include "common.cuh"
#include "fin.cuh"

namespace gpcg {

// grid-stride over the free list
template <class Body>
__device__ __forceinline__ void for_each_free_row(long long m, const int* __restrict__ rows, Body&& body) {
    for (long long k = blockIdx.x * (long long)kThreads + threadIdx.x; k < m; k += (long long)gridDim.x * kThreads)
        body(__ldg(rows + k));
}

template <class Op, bool PC>
__global__ void __launch_bounds__(kThreads)
k_cg_init_rows(Op A, long long m, const int* __restrict__ rows, const double* __restrict__ g,
               const unsigned char* __restrict__ mask, double* __restrict__ rho, double* __restrict__ q,
               double* __restrict__ s, double* __restrict__ p, double* __restrict__ w,
               const double* __restrict__ dinv, double eta2, long long cap, Scal* S, RedScratch R) {
    double acc[2] = {0.0, 0.0};
    for_each_free_row(m, rows, [&](int v) {
        const Pt pt = A.point(v);
        p[v] = 0.0; w[v] = 0.0; s[v] = 0.0;
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
k_cg_iter_rows(Op A, long long m, const int* __restrict__ rows, const unsigned char* __restrict__ mask,
               const double* __restrict__ rho, const double* __restrict__ q, const double* __restrict__ s,
               double* __restrict__ rho_n, double* __restrict__ q_n, double* __restrict__ s_n,
               double* __restrict__ p, double* __restrict__ w, const double* __restrict__ dinv, Scal* S,
               RedScratch R) {
    if (*(volatile int*)&S->cg_done) return;
    const double alpha = S->cg_alpha, beta = S->cg_beta;
    double acc[2] = {0.0, 0.0};
    for_each_free_row(m, rows, [&](int v) {
        const Pt pt = A.point(v);
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

// y_v = sum_{c in F} a_vc x_c on the free rows (y must be zero elsewhere: the caller clears it)
template <class Op>
__global__ void __launch_bounds__(kThreads)
k_hessvec_rows(Op A, long long m, const int* __restrict__ rows, const unsigned char* __restrict__ mask,
               const double* __restrict__ x, double* __restrict__ y) {
    for_each_free_row(m, rows, [&](int v) {
        double t = 0.0;
        A.for_each_nbr(A.point(v), [&](int c, double a) {
            if (mask[c]) t = fma(a, __ldg(x + c), t);
        });
        y[v] = t;
    });
}

}  // namespace gpcg
