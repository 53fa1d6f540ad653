// bjilu.cuh -- block-Jacobi ILU(0) preconditioned CG on the free set (SURVEY.md 8(f)
// NEXT-3; the paper's block Jacobi with ILU(0) subdomain solves, Table 4)
// for 2-D 5-point stencils (gpcg_params.precond = 2).
//
// Blocks: 32 x 32 tiles of a slab's owned grid (tile (bi, bj) = columns 32 bi .., rows
// 32 bj .. of the slab; entries coupling tiles are dropped).  Within a tile the rows of
// A_k in natural order; ILU(0) keeps the 5-point pattern, so only the pivots change:
//     d_v = a_vv - a_vs^2 / d_s - a_vw^2 / d_w      (south / west neighbour in the tile, free)
// and M = (D + L) D^-1 (D + U) (oracle/gpcg_oracle.c ora_bjilu_*).  One warp owns a tile:
// lane i is column i, and anti-diagonal l = i + j is step l of a 63-step wavefront -- the
// west neighbour of (i, j) was computed by lane i-1 one step earlier (warp shuffle), the
// south neighbour by the same lane one step earlier (register) -- so the factorisation and
// both triangular solves run in registers with no barrier.
//
// PCG (textbook form, the oracle's ora_pcg_m): per iteration
//   k_pcg2_matvec: p = z + beta p (at the point and its neighbours), q = A_F p, sum p'q
//                  -> alpha = gamma / p'q
//   k_pcg2_update: w += alpha p, r -= alpha q, z = M^-1 r (tile wavefronts), sum r'z
//                  -> decrease 1/2 alpha gamma, cgstop1 / exact guard / cap, beta
// Vectors (full length, zero off F): r, z, p (ping-pong), q, w, 1/d.
#pragma once

#include "common.cuh"
#include "fin.cuh"

namespace gpcg {

constexpr int kTile = 32;

// face weights / diagonal of point (i, j) of the slab (StencilOp layout)
struct Faces5 {
    double w, e, s, n, d;
};
__device__ __forceinline__ Faces5 faces_at(const StencilOp& A, int i, int j) {
    Faces5 f;
    f.w = __ldg(A.wx + (long long)j * A.wx_ld + i);
    f.e = __ldg(A.wx + (long long)j * A.wx_ld + i + 1);
    f.s = __ldg(A.wy + (long long)j * A.wy_ld + i);
    f.n = __ldg(A.wy + (long long)(j + 1) * A.wy_ld + i);
    f.d = (f.w + f.e) + (f.s + f.n);
    if (A.shift) f.d += __ldg(A.shift + i + (long long)A.pitch * j);
    return f;
}

// tiles of the slab, one per warp (grid-stride over tiles)
template <class Body>
__device__ __forceinline__ void for_each_tile(const StencilOp& A, Body&& body) {
    const int ntx = (A.nx + kTile - 1) / kTile, nty = (A.ny + kTile - 1) / kTile;
    const int nt = ntx * nty;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int t = warp; t < nt; t += nw) body((t % ntx) * kTile, (t / ntx) * kTile);
}

// ILU(0) pivots of every tile on the CG mask -> dinv = 1 / d (1 off F)
__global__ void __launch_bounds__(256)
k_bjilu_factor(StencilOp A, const unsigned char* __restrict__ mask, double* __restrict__ dinv) {
    const int lane = threadIdx.x & 31;
    for_each_tile(A, [&](int x0, int y0) {
        const int i = x0 + lane;
        double d_prev = 1.0;                              // d of (i, j-1): this lane, previous step
        for (int l = 0; l < 2 * kTile - 1; ++l) {
            const double d_west = __shfl_up_sync(0xffffffffu, d_prev, 1);   // (i-1, j) from step l-1
            const int j = y0 + l - lane;
            double d_new = d_prev;
            if (l - lane >= 0 && l - lane < kTile && i < A.nx && j < A.ny) {
                const long long v = i + (long long)A.pitch * j;
                if (mask[v]) {
                    const Faces5 f = faces_at(A, i, j);
                    double dv = f.d;
                    if (j > y0 && mask[v - A.pitch]) dv = dv - f.s * f.s / d_prev;          // south
                    if (lane > 0 && mask[v - 1]) dv = dv - f.w * f.w / d_west;              // west
                    d_new = dv;
                    dinv[v] = 1.0 / dv;
                } else {
                    d_new = 1.0;
                    dinv[v] = 1.0;
                }
            }
            d_prev = d_new;
        }
    });
}

// z = M^-1 r on one tile (r already updated): forward (D + L) t = r, backward D^-1 (D + U) z = t.
// The tile's r, 1/d and mask are first staged in shared memory by coalesced row loads (the
// wavefront steps then wait on shared memory, not on dependent global loads); z overwrites t
// in place during the backward sweep and is stored row by row.  Returns this lane's r'z.
struct TileSmem {
    double r[kTile * kTile], dinv[kTile * kTile], t[kTile * kTile];
    unsigned char m[kTile * kTile];
};

__device__ __forceinline__ double tile_solve(const StencilOp& A, int x0, int y0, const unsigned char* __restrict__ mask,
                                             const double* __restrict__ dinv, const double* __restrict__ r,
                                             double* __restrict__ z, TileSmem& T) {
    const int lane = threadIdx.x & 31;
    const int i = x0 + lane;
    const bool col_ok = i < A.nx;
    // stage (coalesced rows; unrolled so that many rows' loads are in flight at once)
    const int ic = col_ok ? i : x0;                       // in-grid address for the predicated-off lanes
#pragma unroll 8
    for (int jl = 0; jl < kTile; ++jl) {
        const int j = y0 + jl;
        const bool in = col_ok && j < A.ny;
        const long long v = ic + (long long)A.pitch * min(j, A.ny - 1);
        const unsigned char mv = in ? mask[v] : 0;
        const double rv = r[v], dv = dinv[v];
        const int q = jl * kTile + lane;
        T.m[q] = mv;
        T.r[q] = mv ? rv : 0.0;
        T.dinv[q] = mv ? dv : 0.0;
    }
    __syncwarp();
    double t_prev = 0.0;                                  // t of (i, j-1)
    for (int l = 0; l < 2 * kTile - 1; ++l) {
        const double t_west = __shfl_up_sync(0xffffffffu, t_prev, 1);
        const int jl = l - lane;
        double t_new = t_prev;
        if (jl >= 0 && jl < kTile) {
            const int q = jl * kTile + lane;
            double tv = 0.0;
            if (T.m[q]) {
                const int j = y0 + jl;
                double s = T.r[q];
                if (jl > 0 && T.m[q - kTile]) s = s + __ldg(A.wy + (long long)j * A.wy_ld + i) * t_prev;   // a_vs = -w_s
                if (lane > 0 && T.m[q - 1]) s = s + __ldg(A.wx + (long long)j * A.wx_ld + i) * t_west;     // a_vw = -w_w
                tv = s * T.dinv[q];
            }
            T.t[q] = tv;
            t_new = tv;
        }
        t_prev = t_new;
    }
    __syncwarp();
    double z_prev = 0.0;                                  // z of (i, j+1)
    for (int l = 2 * kTile - 2; l >= 0; --l) {
        const double z_east = __shfl_down_sync(0xffffffffu, z_prev, 1);
        const int jl = l - lane;
        double z_new = z_prev;
        if (jl >= 0 && jl < kTile) {
            const int q = jl * kTile + lane;
            double zv = 0.0;
            if (T.m[q]) {
                const int j = y0 + jl;
                double s = 0.0;
                if (jl < kTile - 1 && T.m[q + kTile]) s = s - __ldg(A.wy + (long long)(j + 1) * A.wy_ld + i) * z_prev;  // a_vn
                if (lane < kTile - 1 && T.m[q + 1]) s = s - __ldg(A.wx + (long long)j * A.wx_ld + i + 1) * z_east;     // a_ve
                zv = T.t[q] - s * T.dinv[q];
            }
            T.t[q] = zv;                                  // z overwrites t (t_v is not read again)
            z_new = zv;
        }
        z_prev = z_new;
    }
    __syncwarp();
    double rz = 0.0;
#pragma unroll 8
    for (int jl = 0; jl < kTile; ++jl) {                  // store z (coalesced rows), r'z
        const int j = y0 + jl;
        if (col_ok && j < A.ny) {
            const int q = jl * kTile + lane;
            const double zv = T.t[q];
            z[i + (long long)A.pitch * j] = zv;
            rz = fma(T.r[q], zv, rz);
        }
    }
    __syncwarp();
    return rz;
}

// init: r = -[v in F] (A y - b)_v, w = 0, p = 0, mask copy; then z = M^-1 r, gamma = r'z
// (two launches: the gradient sweep below, then k_pcg2_solve)
__global__ void __launch_bounds__(kThreads)
k_pcg2_init(StencilOp A, const double* __restrict__ y, const double* __restrict__ b,
            const unsigned char* __restrict__ mask, unsigned char* __restrict__ mask_cg, double* __restrict__ r,
            double* __restrict__ p0, double* __restrict__ p1, double* __restrict__ w) {
    A.for_each_point([&](const Pt& pt) {
        const int v = pt.v;
        mask_cg[v] = mask[v];
        double g = 0.0;
        A.for_each_nbr(pt, [&](int c, double a) { g = fma(a, __ldg(y + c), g); });
        g -= __ldg(b + v);
        r[v] = mask[v] ? -g : 0.0;
        p0[v] = 0.0;
        p1[v] = 0.0;
        w[v] = 0.0;
    });
}

constexpr int kSolveThreads = 128;      // 4 tiles per CTA, one warp each
constexpr int kSolveSmem = (kSolveThreads / 32) * (int)sizeof(TileSmem);

template <int KIND>   // 0: init solve (gamma_0), 1: iteration update + solve (gamma_{j+1})
__global__ void __launch_bounds__(kSolveThreads)
k_pcg2_solve(StencilOp A, const unsigned char* __restrict__ mask, const double* __restrict__ dinv,
             double* __restrict__ r, const double* __restrict__ q, const double* __restrict__ p,
             double* __restrict__ w, double* __restrict__ z, double eta2, long long cap, Scal* S, RedScratch R) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (KIND == 1 && *(volatile int*)&S->cg_done) return;
    const double alpha = KIND == 1 ? S->cg_alpha : 0.0;
    double acc[1] = {0.0};
    const int lane = threadIdx.x & 31;
    TileSmem& T = reinterpret_cast<TileSmem*>(smem_raw)[threadIdx.x >> 5];
    for_each_tile(A, [&](int x0, int y0) {
        if (KIND == 1) {                                  // w += alpha p, r -= alpha q on the tile
            const int i = x0 + lane;
            const int ic = i < A.nx ? i : x0;
#pragma unroll 8
            for (int jl = 0; jl < kTile; ++jl) {          // unconditional loads: rows in flight together
                const int j = y0 + jl;
                const bool in = i < A.nx && j < A.ny;
                const long long v = ic + (long long)A.pitch * min(j, A.ny - 1);
                const unsigned char mv = mask[v];
                const double pv = p[v], wv = w[v], qv = q[v], rv = r[v];
                if (in && mv) {
                    w[v] = fma(alpha, pv, wv);
                    r[v] = fma(-alpha, qv, rv);
                }
            }
            __syncwarp();
        }
        acc[0] += tile_solve(A, x0, y0, mask, dinv, r, z, T);
    });
    reduce_and_finish<1>(acc, R, [&](double* t) {
        if (KIND == 0) pcg2_init_fin(t[0], eta2, cap, S);
        else pcg2_beta_fin(t[0], S);
    });
}

// p_new = z + beta p_old (zero off F; formed at the neighbours too), q = A_F p_new, sum p'q
__global__ void __launch_bounds__(kThreads)
k_pcg2_matvec(StencilOp A, const unsigned char* __restrict__ mask, const double* __restrict__ z,
              const double* __restrict__ p_old, double* __restrict__ p_new, double* __restrict__ q, Scal* S,
              RedScratch R) {
    if (*(volatile int*)&S->cg_done) return;
    const double beta = S->cg_beta;
    double acc[1] = {0.0};
    A.for_each_point([&](const Pt& pt) {
        const int v = pt.v;
        if (!mask[v]) { p_new[v] = 0.0; q[v] = 0.0; return; }
        double qv = 0.0, pv = 0.0;
        A.for_each_nbr(pt, [&](int c, double a) {
            if (!mask[c]) return;
            const double pc = fma(beta, p_old[c], z[c]);
            if (c == v) pv = pc;
            qv = fma(a, pc, qv);
        });
        p_new[v] = pv;
        q[v] = qv;
        acc[0] = fma(pv, qv, acc[0]);
    });
    reduce_and_finish<1>(acc, R, [&](double* t) { pcg2_alpha_fin(t[0], S); });
}

}  // namespace gpcg
