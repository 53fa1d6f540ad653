// march3.cuh -- stencil-specialised sweeps for the 3-D 7-point operator (SURVEY.md 8(f) NEXT-2,
// gpcg_create_stencil3d): a1 accept, a2 Cauchy, a3 search, a4 hessvec, a5 CG init / iteration.
//
// Execution model ("plane march"): a 256-thread CTA owns a 32 x 8 column block of the (x, y)
// plane -- lane = x, warp = y -- and marches up a chunk of KZ planes.  At every plane step each
// thread loads the raw inputs of its column two planes ahead (software pipeline), forms the
// derived value the operator is applied to (trial point, projected gradient, search step, CG
// vector) ONCE per point, and publishes it in a 3-slot shared-memory ring of planes.  After one
// CTA barrier the interior threads (lanes 1..30, warps 1..6) apply the operator at the plane
// below: x / y neighbours from shared memory, z neighbours from the thread's own registers
// (previous / next plane), face weights prefetched with the raw inputs.  Outputs are written
// by the interior threads only; the one-cell halo ring is recomputed by the neighbouring block.
//
// Per point every kernel does exactly the arithmetic of its generic counterpart in
// kernels.cuh with Stencil3Op (same derived values, operator terms accumulated in the same
// order: diagonal, west, east, south, north, down, up; a neighbour outside the readable grid
// contributes fma(-w, 0, .), which leaves the sum unchanged), so only the order of the block
// partial sums differs.
#pragma once

#include "common.cuh"
#include "fin.cuh"

namespace gpcg {
namespace m3 {
#ifndef GPCG_M3_TY
#define GPCG_M3_TY 8
#endif
constexpr int TX = 32, TY = GPCG_M3_TY;   // threads per block: lanes x, warps y
constexpr int OX = TX - 2, OY = TY - 2;   // outputs per block in x, y
constexpr int KZ = 32;                    // planes per work item
constexpr int kThreads = TX * TY;
constexpr int kMinBlocks = TY >= 16 ? 1 : 2;
}  // namespace m3

// face weights of point (i, j, k) (Stencil3Op layout) + diagonal shift; wu is the next plane's wd
struct Faces7 {
    double ww, we, ws, wn, wd, sh;
};

// Faces of the owned point (i, j, k) for an interior thread (ok = in-grid column and interior);
// at k = nz only wd (the top face plane, which enters the diagonal of plane nz - 1 as wu).
__device__ __forceinline__ Faces7 faces7(const Stencil3Op& A, int i, int j, int k, bool ok) {
    Faces7 f{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (!ok || k < 0 || k > A.nz) return f;
    const long long ij = (long long)j * A.nx + i;
    f.wd = __ldg(A.wz + (long long)k * A.plane + ij);
    if (k == A.nz) return f;
    const double* wxl = A.wx + ((long long)k * A.ny + j) * (A.nx + 1) + i;
    const double* wyl = A.wy + (long long)k * (A.plane + A.nx) + ij;
    f.ww = __ldg(wxl);
    f.we = __ldg(wxl + 1);
    f.ws = __ldg(wyl);
    f.wn = __ldg(wyl + A.nx);
    if (A.shift) f.sh = __ldg(A.shift + (long long)k * A.plane + ij);
    return f;
}

// (A u)_v with the terms in Stencil3Op::for_each_nbr's order
__device__ __forceinline__ double apply7(const Faces7& f, double wu, double uc, double uw, double ue, double us,
                                         double un, double ud, double uu, bool shift) {
    double d = ((f.ww + f.we) + (f.ws + f.wn)) + (f.wd + wu);
    if (shift) d += f.sh;
    double q = d * uc;
    q = fma(-f.ww, uw, q);
    q = fma(-f.we, ue, q);
    q = fma(-f.ws, us, q);
    q = fma(-f.wn, un, q);
    q = fma(-f.wd, ud, q);
    return fma(-wu, uu, q);
}

struct M3Item {
    int i, j, k0, k1;   // this thread's column (may be outside the grid), plane range of the item
    bool out;           // interior thread on an owned in-grid column
};

__device__ __forceinline__ int m3_items(const Stencil3Op& A) {
    return ((A.nx + m3::OX - 1) / m3::OX) * ((A.ny + m3::OY - 1) / m3::OY) * ((A.nz + m3::KZ - 1) / m3::KZ);
}

__device__ __forceinline__ M3Item m3_item(const Stencil3Op& A, int item) {
    const int ntx = (A.nx + m3::OX - 1) / m3::OX, nty = (A.ny + m3::OY - 1) / m3::OY;
    const int bx = item % ntx, r = item / ntx, by = r % nty, bz = r / nty;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    M3Item it;
    it.i = bx * m3::OX - 1 + tx;
    it.j = by * m3::OY - 1 + ty;
    it.k0 = bz * m3::KZ;
    it.k1 = min(it.k0 + m3::KZ, A.nz);
    it.out = tx >= 1 && tx <= m3::TX - 2 && ty >= 1 && ty <= m3::TY - 2 && it.i >= 0 && it.i < A.nx && it.j >= 0 &&
             it.j < A.ny;
    return it;
}

// The plane march over one work item.  Raw: per-point inputs incl. Faces7 f; load(k) -> Raw
// (k may lie outside the readable planes: load must then give derived values 0); derive(k, raw,
// u[NV]); emit(k, raw_c, uc[NV], Au[NV]) for interior threads at owned plane k.
template <int NV, class Raw, class LoadF, class DeriveF, class EmitF>
__device__ __forceinline__ void march3(const Stencil3Op& A, const M3Item& it, double* U /* 3*NV*kThreads */,
                                       LoadF&& load, DeriveF&& derive, EmitF&& emit) {
    const int tid = threadIdx.x;
    const bool shift = A.shift != nullptr;
    auto slot = [&](int s, int v) { return U + (s * NV + v) * m3::kThreads; };
    Raw rm = load(it.k0 - 1), rc = load(it.k0), rn = load(it.k0 + 1);
    double um[NV], uc[NV], un[NV];
    derive(it.k0 - 1, rm, um);
    derive(it.k0, rc, uc);
#pragma unroll
    for (int v = 0; v < NV; ++v) slot(0, v)[tid] = uc[v];
    int s0 = 0, s1 = 1, s2 = 2;                  // slots of planes k, k + 1, k - 1
    for (int k = it.k0; k < it.k1; ++k) {
        const Raw rnn = load(k + 2);             // two planes ahead
        derive(k + 1, rn, un);
#pragma unroll
        for (int v = 0; v < NV; ++v) slot(s1, v)[tid] = un[v];
        __syncthreads();
        if (it.out) {
            double au[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const double* P = slot(s0, v);
                au[v] = apply7(rc.f, rn.f.wd, uc[v], P[tid - 1], P[tid + 1], P[tid - m3::TX], P[tid + m3::TX], um[v], un[v],
                               shift);
            }
            emit(k, rc, uc, au);
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) { um[v] = uc[v]; uc[v] = un[v]; }
        rc = rn;
        rn = rnn;
        const int t = s2; s2 = s0; s0 = s1; s1 = t;
    }
    __syncthreads();                             // the ring is reused by the next item
}

// readable-grid test of (i, j, k) and its flat index
__device__ __forceinline__ bool m3_in(const Stencil3Op& A, int i, int j, int k) {
    return i >= 0 && i < A.nx && j >= 0 && j < A.ny && k >= A.klo && k < A.khi;
}
__device__ __forceinline__ long long m3_v(const Stencil3Op& A, int i, int j, int k) {
    return i + (long long)A.nx * j + A.plane * k;
}

#define M3_SMEM(NV) __shared__ double U_[3 * (NV) * m3::kThreads]

// ---------------------------------------------------------------- a1 accept (k_accept)
template <bool SB>
struct RawAcc3 {
    double y, d, b, l, u;
    unsigned char mp;
    bool in;
    Faces7 f;
};

template <bool SB>
__global__ void __launch_bounds__(m3::kThreads, m3::kMinBlocks)
k7_accept(Stencil3Op A, Bounds Bd, const double* __restrict__ y_in, const double* __restrict__ dir, double sgn,
          const double* __restrict__ b, const unsigned char* __restrict__ mask_prev, double* __restrict__ y_out,
          double* __restrict__ g_out, unsigned char* __restrict__ mask_out, Scal* S, RedScratch R, int gp) {
    M3_SMEM(1);
    if (gp && gp_skip(S)) return;      // GP phase over / k_spec accepted
    double alpha = 0.0;
    if (dir) {
        if (S->s_h < 0) return;
        alpha = S->s_alpha;
    }
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    using Raw = RawAcc3<SB>;
    for (int item = blockIdx.x; item < m3_items(A); item += gridDim.x) {
        const M3Item it = m3_item(A, item);
        march3<1, Raw>(
            A, it, U_,
            [&](int k) {
                Raw r{0.0, 0.0, 0.0, 0.0, 0.0, 0, false, Faces7{}};
                r.in = m3_in(A, it.i, it.j, k);
                if (r.in) {
                    const long long v = m3_v(A, it.i, it.j, k);
                    r.y = __ldg(y_in + v);
                    if (dir) r.d = __ldg(dir + v);
                    r.l = SB ? Bd.lc : __ldg(Bd.l + v);
                    r.u = SB ? Bd.uc : __ldg(Bd.u + v);
                    if (it.out) {
                        r.b = __ldg(b + v);
                        if (mask_prev) r.mp = mask_prev[v];
                    }
                }
                r.f = faces7(A, it.i, it.j, k, it.out);
                return r;
            },
            [&](int, const Raw& r, double* u) {
                u[0] = r.in ? (dir ? trial(r.y, r.d, sgn, alpha, r.l, r.u) : mid(r.l, r.u, r.y)) : 0.0;
            },
            [&](int k, const Raw& r, const double* uc, const double* au) {
                const long long v = m3_v(A, it.i, it.j, k);
                const double yv = uc[0];
                const double g = au[0] - r.b;
                y_out[v] = yv;
                g_out[v] = g;
                const bool act = (yv == r.l) || (yv == r.u);
                const unsigned char m = act ? 0 : 1;
                mask_out[v] = m;
                const double pg = pgrad(yv, g, r.l, r.u);
                acc[0] = fma(pg, pg, acc[0]);
                acc[1] = fma(g, g, acc[1]);
                acc[2] += act ? 1.0 : 0.0;
                if (mask_prev) acc[3] += (r.mp != m) ? 1.0 : 0.0;
                const bool binding = (yv == r.l && g >= 0.0) || (yv == r.u && g <= 0.0);
                acc[4] += (act && !binding) ? 1.0 : 0.0;
            });
    }
    reduce_and_finish<5>(acc, R, [&](double* t) { fin_accept(t, false, S); });
}

// ---------------------------------------------------------------- a2 Cauchy (k_cauchy)
struct RawCy3 {
    double y, g, l, u;
    bool in;
    Faces7 f;
};

template <bool SB>
__global__ void __launch_bounds__(m3::kThreads, m3::kMinBlocks)
k7_cauchy(Stencil3Op A, Bounds Bd, const double* __restrict__ y, const double* __restrict__ g, Scal* S, RedScratch R,
          int gp) {
    M3_SMEM(1);
    if (gp && *(volatile int*)&S->gp_done) return;
    double acc[2] = {0.0, 0.0};
    for (int item = blockIdx.x; item < m3_items(A); item += gridDim.x) {
        const M3Item it = m3_item(A, item);
        march3<1, RawCy3>(
            A, it, U_,
            [&](int k) {
                RawCy3 r{0.0, 0.0, 0.0, 0.0, false, Faces7{}};
                r.in = m3_in(A, it.i, it.j, k);
                if (r.in) {
                    const long long v = m3_v(A, it.i, it.j, k);
                    r.y = __ldg(y + v);
                    r.g = __ldg(g + v);
                    r.l = SB ? Bd.lc : __ldg(Bd.l + v);
                    r.u = SB ? Bd.uc : __ldg(Bd.u + v);
                }
                r.f = faces7(A, it.i, it.j, k, it.out);
                return r;
            },
            [&](int, const RawCy3& r, double* u) { u[0] = r.in ? pgrad(r.y, r.g, r.l, r.u) : 0.0; },
            [&](int, const RawCy3&, const double* uc, const double* au) {
                acc[0] = fma(uc[0], uc[0], acc[0]);
                acc[1] = fma(uc[0], au[0], acc[1]);
            });
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { fin_cauchy(t, S); });
}

// ---------------------------------------------------------------- a3 search (k_search)
struct RawSr3 {
    double y, d, g, l, u;
    bool in;
    Faces7 f;
};

template <bool SB, int K>
__global__ void __launch_bounds__(m3::kThreads, m3::kMinBlocks)
k7_search(Stencil3Op A, Bounds Bd, const double* __restrict__ y, const double* __restrict__ g,
          const double* __restrict__ dir, double sgn, int use_alpha0, int h0, double mu, Scal* S, RedScratch R,
          int gp) {
    M3_SMEM(K);
    if (gp && gp_skip(S)) return;      // GP phase over / k_spec accepted
    if (use_alpha0 && !S->cauchy_ok) {
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
    for (int item = blockIdx.x; item < m3_items(A); item += gridDim.x) {
        const M3Item it = m3_item(A, item);
        march3<K, RawSr3>(
            A, it, U_,
            [&](int k) {
                RawSr3 r{0.0, 0.0, 0.0, 0.0, 0.0, false, Faces7{}};
                r.in = m3_in(A, it.i, it.j, k);
                if (r.in) {
                    const long long v = m3_v(A, it.i, it.j, k);
                    r.y = __ldg(y + v);
                    r.d = __ldg(dir + v);
                    if (it.out) r.g = __ldg(g + v);
                    r.l = SB ? Bd.lc : __ldg(Bd.l + v);
                    r.u = SB ? Bd.uc : __ldg(Bd.u + v);
                }
                r.f = faces7(A, it.i, it.j, k, it.out);
                return r;
            },
            [&](int, const RawSr3& r, double* u) {
#pragma unroll
                for (int h = 0; h < K; ++h) u[h] = r.in ? trial(r.y, r.d, sgn, al[h], r.l, r.u) - r.y : 0.0;
            },
            [&](int, const RawSr3& r, const double* uc, const double* au) {
#pragma unroll
                for (int h = 0; h < K; ++h) {
                    acc[2 * h] = fma(r.g, uc[h], acc[2 * h]);
                    acc[2 * h + 1] = fma(uc[h], au[h], acc[2 * h + 1]);
                }
            });
    }
    reduce_and_finish<2 * K>(acc, R, [&](double* t) { fin_search(t, K, h0, base, mu, S); });
}

// ---------------------------------------------------------------- a4 hessvec (k_hessvec)
struct RawHv3 {
    double x;
    unsigned char m;
    bool in;
    Faces7 f;
};

template <bool kReduced>
__global__ void __launch_bounds__(m3::kThreads, m3::kMinBlocks)
k7_hessvec(Stencil3Op A, const double* __restrict__ x, double* __restrict__ y, const unsigned char* __restrict__ mask) {
    M3_SMEM(1);
    for (int item = blockIdx.x; item < m3_items(A); item += gridDim.x) {
        const M3Item it = m3_item(A, item);
        march3<1, RawHv3>(
            A, it, U_,
            [&](int k) {
                RawHv3 r{0.0, 0, false, Faces7{}};
                r.in = m3_in(A, it.i, it.j, k);
                if (r.in) {
                    const long long v = m3_v(A, it.i, it.j, k);
                    r.x = __ldg(x + v);
                    r.m = kReduced ? mask[v] : 1;
                }
                // (loads not predicated on the mask: a dependent mask -> value chain measured slower
                // at C4's 5 % free set, 431 vs 322 us)
                r.f = faces7(A, it.i, it.j, k, it.out);
                return r;
            },
            [&](int, const RawHv3& r, double* u) { u[0] = (r.in && r.m) ? r.x : 0.0; },
            [&](int k, const RawHv3& r, const double*, const double* au) {
                y[m3_v(A, it.i, it.j, k)] = r.m ? au[0] : 0.0;
            });
    }
}

// ---------------------------------------------------------------- a5 CG init (k_cg_init)
struct RawCi3 {
    double g, dinv;
    unsigned char m;
    bool in;
    Faces7 f;
};

template <bool PC>
__global__ void __launch_bounds__(m3::kThreads, m3::kMinBlocks)
k7_cg_init(Stencil3Op A, const double* __restrict__ g, const unsigned char* __restrict__ mask,
           unsigned char* __restrict__ mask_cg, double* __restrict__ rho, double* __restrict__ q, double* __restrict__ s,
           double* __restrict__ rho2, double* __restrict__ q2, double* __restrict__ s2, double* __restrict__ p,
           double* __restrict__ w, const double* __restrict__ dinv, double eta2, long long cap, Scal* S, RedScratch R) {
    M3_SMEM(1);
    double acc[2] = {0.0, 0.0};
    for (int item = blockIdx.x; item < m3_items(A); item += gridDim.x) {
        const M3Item it = m3_item(A, item);
        march3<1, RawCi3>(
            A, it, U_,
            [&](int k) {
                RawCi3 r{0.0, 0.0, 0, false, Faces7{}};
                r.in = m3_in(A, it.i, it.j, k);
                if (r.in) {
                    const long long v = m3_v(A, it.i, it.j, k);
                    r.m = mask[v];
                    r.g = __ldg(g + v);
                    if (PC) r.dinv = __ldg(dinv + v);
                }
                r.f = faces7(A, it.i, it.j, k, it.out);
                return r;
            },
            [&](int, const RawCi3& r, double* u) {
                const double rc = r.m ? -r.g : 0.0;
                u[0] = PC ? rc * r.dinv : rc;
            },
            [&](int k, const RawCi3& r, const double* uc, const double* au) {
                const long long v = m3_v(A, it.i, it.j, k);
                mask_cg[v] = r.m;
                p[v] = 0.0; w[v] = 0.0; s[v] = 0.0;
                rho2[v] = 0.0; q2[v] = 0.0; s2[v] = 0.0;
                if (!r.m) { rho[v] = 0.0; q[v] = 0.0; return; }
                const double rv = -r.g;
                rho[v] = rv;
                q[v] = au[0];
                acc[0] = fma(rv, uc[0], acc[0]);
                acc[1] = fma(uc[0], au[0], acc[1]);
            });
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_init_finalize(t[0], t[1], eta2, cap, S); });
}

// ---------------------------------------------------------------- a5 CG iteration (k_cg_iter)
struct RawCg3 {
    double rho, q, s, dinv, p, w;
    unsigned char m;
    Faces7 f;
};

template <bool PC>
__global__ void __launch_bounds__(m3::kThreads, m3::kMinBlocks)
k7_cg_iter(Stencil3Op A, const unsigned char* __restrict__ mask, const double* __restrict__ rho,
           const double* __restrict__ q, const double* __restrict__ s, double* __restrict__ rho_n,
           double* __restrict__ q_n, double* __restrict__ s_n, double* __restrict__ p, double* __restrict__ w,
           const double* __restrict__ dinv, Scal* S, RedScratch R) {
    M3_SMEM(1);
    if (*(volatile int*)&S->cg_done) return;
    const double alpha = S->cg_alpha, beta = S->cg_beta;
    double acc[2] = {0.0, 0.0};
    for (int item = blockIdx.x; item < m3_items(A); item += gridDim.x) {
        const M3Item it = m3_item(A, item);
        march3<1, RawCg3>(
            A, it, U_,
            [&](int k) {
                RawCg3 r{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0, Faces7{}};
                if (m3_in(A, it.i, it.j, k)) {
                    const long long v = m3_v(A, it.i, it.j, k);
                    r.m = mask[v];
                    if (r.m) {
                        r.rho = rho[v];
                        r.q = q[v];
                        r.s = s[v];
                        if (PC) r.dinv = __ldg(dinv + v);
                        if (it.out) { r.p = p[v]; r.w = w[v]; }
                    }
                }
                r.f = faces7(A, it.i, it.j, k, it.out);
                return r;
            },
            [&](int, const RawCg3& r, double* u) {
                const double rc = r.m ? fma(-alpha, fma(beta, r.s, r.q), r.rho) : 0.0;   // rho_{i+1}
                u[0] = PC ? rc * r.dinv : rc;
            },
            [&](int k, const RawCg3& r, const double* uc, const double* au) {
                if (!r.m) return;
                const long long v = m3_v(A, it.i, it.j, k);
                const double pn = fma(beta, r.p, PC ? r.rho * r.dinv : r.rho);
                const double sn = fma(beta, r.s, r.q);
                w[v] = fma(alpha, pn, r.w);
                p[v] = pn;
                s_n[v] = sn;
                const double rnv = fma(-alpha, sn, r.rho);
                const double unv = uc[0];
                rho_n[v] = rnv;
                q_n[v] = au[0];
                acc[0] = fma(rnv, unv, acc[0]);
                acc[1] = fma(unv, au[0], acc[1]);
            });
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_finalize(t[0], t[1], S); });
}

#undef M3_SMEM

}  // namespace gpcg
