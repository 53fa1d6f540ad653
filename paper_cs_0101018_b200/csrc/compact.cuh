// compact.cuh -- the reduced Hessian applied IN PLACE over a compacted free-row list (SURVEY.md
// 8(a) a4 (iii); the paper's "alternative technique" of running CG on the full operator
// restricted to the free index set) for the small-free regime (C4: ~5 % free).
//
// F = [v_0 < v_1 < ... < v_{m-1}], the free points of the current mask in owned-point order,
// is built by the deterministic prefix sums of extract.cuh (k_scan_*), with pos[v] = k for v in F
// and the same set as bits.  The kernels iterate k < m with v = F[k] instead of every point: A's
// rows are read in place (no copy of its values, unlike the extraction ablation), the CG vectors
// live in the reduced space (m entries, coalesced), and neighbours are visited only where the
// free bits say so -- O(m) instead of O(n) work and bytes.  Same arithmetic (and order of the
// operator terms) as k_cg_init / k_cg_iter / k_hessvec of kernels.cuh.
#pragma once

#include "common.cuh"
#include "fin.cuh"

namespace gpcg {

// ---------------------------------------------------------------- free bits + reduced product
// The free set as bits: word w holds the mask bytes 32 w .. 32 w + 31 (n / 8 bytes -- 2 MB at
// C4's 16.8M points, L2-resident, where the byte mask's scattered neighbour tests each cost a
// DRAM sector).  One warp per word: the ballot of its 32 bytes.
__global__ void __launch_bounds__(kThreads)
k_pack_bits(long long n, const unsigned char* __restrict__ mask, unsigned* __restrict__ bits) {
    const long long i = blockIdx.x * (long long)kThreads + threadIdx.x;
    const unsigned b = __ballot_sync(0xffffffffu, i < n && mask[i] != 0);
    if ((threadIdx.x & 31) == 0 && i < n) bits[i >> 5] = b;
}

__device__ __forceinline__ bool free_bit(const unsigned* __restrict__ bits, int c) {
    return (__ldg(bits + (c >> 5)) >> (c & 31)) & 1u;
}

// The CG vectors live in the REDUCED space (index k of F, the w of Eq. cg2 itself): rho, q, s,
// p, w of m entries each, read and written coalesced; only the operator's rows of A (in place),
// the free bits and -- for free neighbours -- pos[c] (the k of point c) and their compact values
// are gathered.  Same recurrences, arithmetic and order of operator terms as k_cg_init /
// k_cg_iter (kernels.cuh), so the same iterates as the masked full-length kernels.
template <class Op, bool PC>
__global__ void __launch_bounds__(kThreads)
k_cg_init_c(Op A, long long m, const int* __restrict__ rows, const unsigned* __restrict__ bits,
            const double* __restrict__ g, double* __restrict__ rho, double* __restrict__ q, double* __restrict__ s,
            double* __restrict__ p, double* __restrict__ w, const double* __restrict__ dinv, double eta2,
            long long cap, Scal* S, RedScratch R) {
    double acc[2] = {0.0, 0.0};
    for (long long k = blockIdx.x * (long long)kThreads + threadIdx.x; k < m; k += (long long)gridDim.x * kThreads) {
        const int v = __ldg(rows + k);
        p[k] = 0.0; w[k] = 0.0; s[k] = 0.0;
        double qv = 0.0, uv = 0.0;
        A.for_each_nbr(A.point(v), [&](int c, double a) {
            const double rc = free_bit(bits, c) ? -__ldg(g + c) : 0.0;
            const double uc = PC ? rc * __ldg(dinv + c) : rc;
            if (c == v) uv = uc;
            qv = fma(a, uc, qv);
        });
        const double rv = -__ldg(g + v);
        rho[k] = rv;
        q[k] = qv;
        acc[0] = fma(rv, uv, acc[0]);
        acc[1] = fma(uv, qv, acc[1]);
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_init_finalize(t[0], t[1], eta2, cap, S); });
}

template <class Op, bool PC>
__global__ void __launch_bounds__(kThreads)
k_cg_iter_c(Op A, long long m, const int* __restrict__ rows, const unsigned* __restrict__ bits,
            const int* __restrict__ pos, const double* __restrict__ rho, const double* __restrict__ q,
            const double* __restrict__ s, double* __restrict__ rho_n, double* __restrict__ q_n,
            double* __restrict__ s_n, double* __restrict__ p, double* __restrict__ w,
            const double* __restrict__ dinv, Scal* S, RedScratch R) {
    if (*(volatile int*)&S->cg_done) return;
    const double alpha = S->cg_alpha, beta = S->cg_beta;
    double acc[2] = {0.0, 0.0};
    for (long long k = blockIdx.x * (long long)kThreads + threadIdx.x; k < m; k += (long long)gridDim.x * kThreads) {
        const int v = __ldg(rows + k);
        const double rv = rho[k], qv = q[k], sv = s[k];
        const double dv = PC ? __ldg(dinv + v) : 1.0;
        const double pn = fma(beta, p[k], PC ? rv * dv : rv);
        const double sn = fma(beta, sv, qv);
        w[k] = fma(alpha, pn, w[k]);
        p[k] = pn;
        s_n[k] = sn;
        double rnv = 0.0, unv = 0.0, qn = 0.0;
        A.for_each_nbr(A.point(v), [&](int c, double a) {
            double uc;
            if (c == v) {
                rnv = fma(-alpha, sn, rv);
                unv = PC ? rnv * dv : rnv;
                uc = unv;
            } else {
                if (!free_bit(bits, c)) return;
                const int kc = __ldg(pos + c);
                const double rc = fma(-alpha, fma(beta, s[kc], q[kc]), rho[kc]);
                uc = PC ? rc * __ldg(dinv + c) : rc;
            }
            qn = fma(a, uc, qn);
        });
        rho_n[k] = rnv;
        q_n[k] = qn;
        acc[0] = fma(rnv, unv, acc[0]);
        acc[1] = fma(unv, qn, acc[1]);
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_finalize(t[0], t[1], S); });
}

// w (full length, cleared by the caller) at the free points from the reduced-space w
__global__ void __launch_bounds__(kThreads)
k_scatter_free(long long m, const int* __restrict__ rows, const double* __restrict__ wc, double* __restrict__ w) {
    const long long k = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (k < m) w[__ldg(rows + k)] = wc[k];
}

// y = (A_F x) on the free rows: y_free[k] = sum_{c in F} a_{F[k] c} x_c (compact output, the
// reduced space of A_k = Z'AZ, Eq. cg2) and / or y_full[F[k]] (the full-length layout
// of gpcg_hessvec; the caller clears y_full off F).  Same fma chain (CSR order, free columns
// only) as the masked full-length k_hessvec<Op, true>.
//
// CSR ("CSR-vector"): a group of kRowLanes lanes per free row, kRowUnroll
// rows per group in flight (4 lanes x 2 rows at 64 registers measured fastest at C4 of 8 x 4 /
// 8 x 2 / 8 x 8 / 4 x 4 at 40-136 registers, r2h2: 99.6 vs 101-171 us).  Lane j of a group loads entry j of its row (the row's columns and
// values are contiguous: one or two sectors each, instead of one thread walking a chain of
// dependent loads), tests the column's free bit and gathers x there; every lane of the group
// then forms the sum in the row's CSR order from the group's shuffled (a, x) pairs, and the
// group's first lane stores it.  Rows longer than kRowLanes take several chunks.
#ifndef GPCG_HVF_LANES
#define GPCG_HVF_LANES 4        // lanes per free row (A/B: scripts/build_variant.sh; r2h2)
#endif
#ifndef GPCG_HVF_UNROLL
#define GPCG_HVF_UNROLL 2       // rows per lane group in flight
#endif
#ifndef GPCG_HVF_MINB
#define GPCG_HVF_MINB 4         // __launch_bounds__ min CTAs per SM (register budget: 64)
#endif
constexpr int kRowLanes = GPCG_HVF_LANES, kRowUnroll = GPCG_HVF_UNROLL;
__global__ void __launch_bounds__(kThreads, GPCG_HVF_MINB)
k_hessvec_free_csr(CsrOp A, long long m, const int* __restrict__ rows, const unsigned* __restrict__ bits,
                   const double* __restrict__ x, double* __restrict__ y_free, double* __restrict__ y_full) {
    constexpr int kGroups = 32 / kRowLanes;                  // row groups per warp
    const int lane = threadIdx.x & 31, sub = lane & (kRowLanes - 1), base = lane & ~(kRowLanes - 1);
    const long long warp = (blockIdx.x * (long long)kThreads + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * kThreads) >> 5;
    for (long long k0 = warp * kGroups * kRowUnroll; k0 < m; k0 += nwarps * kGroups * kRowUnroll) {
        long long k[kRowUnroll], e0[kRowUnroll];
        int v[kRowUnroll], len[kRowUnroll];
        int maxlen = 0;
#pragma unroll
        for (int u = 0; u < kRowUnroll; ++u) {
            k[u] = k0 + u * kGroups + lane / kRowLanes;
            v[u] = k[u] < m ? __ldg(rows + k[u]) : -1;
        }
#pragma unroll
        for (int u = 0; u < kRowUnroll; ++u) {
            e0[u] = 0;
            len[u] = 0;
            if (v[u] >= 0) {
                e0[u] = __ldg(A.rp + v[u]);
                len[u] = (int)(__ldg(A.rp + v[u] + 1) - e0[u]);
            }
            maxlen = max(maxlen, len[u]);
        }
        maxlen = __reduce_max_sync(0xffffffffu, maxlen);
        double r[kRowUnroll];
#pragma unroll
        for (int u = 0; u < kRowUnroll; ++u) r[u] = 0.0;
        for (int j0 = 0; j0 < maxlen; j0 += kRowLanes) {
            double a[kRowUnroll], xv[kRowUnroll];
            int c[kRowUnroll];
            bool f[kRowUnroll];
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) {
                const bool in = j0 + sub < len[u];
                c[u] = in ? __ldg(A.ci + e0[u] + j0 + sub) : -1;
                a[u] = in ? __ldg(A.val + e0[u] + j0 + sub) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) f[u] = c[u] >= 0 && free_bit(bits, c[u]);
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) xv[u] = f[u] ? __ldg(x + c[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) {
                const unsigned fb = __ballot_sync(0xffffffffu, f[u]);
#pragma unroll
                for (int t = 0; t < kRowLanes; ++t) {
                    const double at = __shfl_sync(0xffffffffu, a[u], base + t);
                    const double xt = __shfl_sync(0xffffffffu, xv[u], base + t);
                    if ((fb >> (base + t)) & 1u) r[u] = fma(at, xt, r[u]);
                }
            }
        }
        if (sub == 0) {
#pragma unroll
            for (int u = 0; u < kRowUnroll; ++u) {
                if (v[u] < 0) continue;
                if (y_free) y_free[k[u]] = r[u];
                if (y_full) y_full[v[u]] = r[u];
            }
        }
    }
}

// 3-D stencil (and any operator with a generic for_each_nbr): one thread per free row, no grid
// stride (every row's dependent loads in flight at once), neighbour tests on the free bits.
template <class Op>
__global__ void __launch_bounds__(kThreads)
k_hessvec_free(Op A, long long m, const int* __restrict__ rows, const unsigned* __restrict__ bits,
               const double* __restrict__ x, double* __restrict__ y_free, double* __restrict__ y_full) {
    const long long k = blockIdx.x * (long long)kThreads + threadIdx.x;
    if (k >= m) return;
    const int v = __ldg(rows + k);
    double t = 0.0;
    A.for_each_nbr(A.point(v), [&](int c, double a) {
        if (free_bit(bits, c)) t = fma(a, __ldg(x + c), t);
    });
    if (y_free) y_free[k] = t;
    if (y_full) y_full[v] = t;
}

}  // namespace gpcg
