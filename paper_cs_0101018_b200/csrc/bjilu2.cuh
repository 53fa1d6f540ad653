// bjilu2.cuh -- block-Jacobi ILU(2) preconditioned CG on the free set (SURVEY.md 8(f)
// NEXT-3; the paper's block Jacobi whose subdomain solver is "ILU(2), which allowed two
// levels of fill", Tables 1-4) for 2-D 5-point stencils (gpcg_params.precond = 3).
//
// Blocks: the 32 x 32 tiles of bjilu.cuh.  Within a tile, the rows of A_k = Z'AZ in natural
// order (point (i, jl) <-> i + 32 jl).  For the 5-point pattern the level-2 fill of row v =
// (i, jl) is (oracle/gpcg_oracle.c ora_bjiluk_factor, pinned by the fill-path theorem in
// tests/test_oracle_iluk.py):
//     L: S = (i, jl-1) [level 0], SE = (i+1, jl-1) [1], SEE = (i+2, jl-1) [2], W = (i-1, jl) [0]
//     U: E = (i+1, jl) [0], NWW = (i-2, jl+1) [2], NW = (i-1, jl+1) [1], N = (i, jl+1) [0]
// and, on the masked graph, SE exists iff S, SE are free; SEE iff S, SE, SEE are (the only fill
// paths run through S and SE).  A is symmetric, so U = D L' (u_vj = l_jv d_v) and only L and
// d = diag(U) are formed.  The IKJ elimination of row v (pivots S, SE, SEE, W in column order):
//     l_S   = a_vS / d_S
//     l_SE  = -l_S  l_{SE,W} d_S / d_SE                       (u_{S,SE}  = l_{SE,W}  d_S)
//     l_SEE = -l_SE l_{SEE,W} d_SE / d_SEE                    (u_{SE,SEE}= l_{SEE,W} d_SE)
//     l_W   = (a_vW - l_S l_{W,SE} d_S - l_SE l_{W,SEE} d_SE) / d_W
//     d_v   = a_vv - l_S^2 d_S - l_SE^2 d_SE - l_SEE^2 d_SEE - l_W^2 d_W
// (l_{X,Y}: the L entry of row X in its column Y; W's SE is S and W's SEE is SE).  Entries of
// points off F, or outside the tile or the grid, are 0 (d = 1), which drops every coupling
// that does not exist in the masked tile graph.
// Solves: forward L y = r (unit L), backward z_v = y_v / d_v - (l_{E,W} z_E + l_{NW,SE} z_NW +
// l_{NWW,SEE} z_NWW + l_{N,S} z_N).  Row v depends on S, SE, SEE, W, so the tile runs as a
// skewed wavefront: lane i (column i) handles row jl at step t = i + 3 jl (W at t-1, SEE at
// t-1, SE at t-2, S at t-3), 125 steps per sweep; the backward sweep in reverse step order.
// r'z = y' D^-1 y (M = L D L'), accumulated in the forward sweep.
#pragma once

#include "bjilu.cuh"

namespace gpcg {

constexpr int kIlu2Steps = (kTile - 1) + 3 * (kTile - 1) + 1;       // 125

// per tile, natural layout (i + 32 jl), kTile^2 doubles per tile and array
struct Bj2Factor {
    double *lS, *lSE, *lSEE, *lW, *dinv;
};

constexpr int kBj2FactorWarps = 2;
constexpr int kBj2FactorSmem = kBj2FactorWarps * 4 * kTile * kTile * 8;   // d, lW, lSE, lSEE per warp

__device__ __forceinline__ bool ilu2_step(int t, int lane, int& jl) {
    const int q = t - lane;
    if (q < 0) return false;
    jl = q / 3;
    return q - 3 * jl == 0 && jl < kTile;
}

__global__ void __launch_bounds__(32 * kBj2FactorWarps)
k_bjilu2_factor(StencilOp A, const unsigned char* __restrict__ mask, Bj2Factor F) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* Dd = reinterpret_cast<double*>(smem_raw) + wid * 4 * kTile * kTile;
    double* Dw = Dd + kTile * kTile;
    double* Dse = Dw + kTile * kTile;
    double* Dsee = Dse + kTile * kTile;
    const int ntx = (A.nx + kTile - 1) / kTile, nty = (A.ny + kTile - 1) / kTile;
    const int nt = ntx * nty;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int tt = warp; tt < nt; tt += nw) {
        const int x0 = (tt % ntx) * kTile, y0 = (tt / ntx) * kTile;
        const long long tb = (long long)tt * kTile * kTile;
        const int i = x0 + lane;
        for (int t = 0; t < kIlu2Steps; ++t) {
            int jl;
            if (ilu2_step(t, lane, jl)) {
                const int j = y0 + jl;
                const int q = jl * kTile + lane;
                double d = 1.0, lS = 0.0, lSE = 0.0, lSEE = 0.0, lW = 0.0, di = 0.0;
                if (i < A.nx && j < A.ny) {
                    const long long v = i + (long long)A.pitch * j;
                    if (mask[v]) {
                        const Faces5 fc = faces_at(A, i, j);
                        const double aS = (jl > 0 && mask[v - A.pitch]) ? -fc.s : 0.0;
                        const double aW = (lane > 0 && mask[v - 1]) ? -fc.w : 0.0;
                        const double dS = jl > 0 ? Dd[q - kTile] : 1.0;
                        const bool se = jl > 0 && lane + 1 < kTile, see = jl > 0 && lane + 2 < kTile;
                        const double dSE = se ? Dd[q - kTile + 1] : 1.0;
                        const double dSEE = see ? Dd[q - kTile + 2] : 1.0;
                        const double dW = lane > 0 ? Dd[q - 1] : 1.0;
                        lS = aS / dS;
                        lSE = se ? -lS * Dw[q - kTile + 1] * dS / dSE : 0.0;
                        lSEE = see ? -lSE * Dw[q - kTile + 2] * dSE / dSEE : 0.0;
                        double xW = aW;
                        if (lane > 0) xW = xW - lS * Dse[q - 1] * dS - lSE * Dsee[q - 1] * dSE;
                        lW = xW / dW;
                        d = fc.d - lS * lS * dS - lSE * lSE * dSE - lSEE * lSEE * dSEE - lW * lW * dW;
                        di = 1.0 / d;
                    }
                }
                Dd[q] = d;
                Dw[q] = lW;
                Dse[q] = lSE;
                Dsee[q] = lSEE;
                F.lS[tb + q] = lS;
                F.lSE[tb + q] = lSE;
                F.lSEE[tb + q] = lSEE;
                F.lW[tb + q] = lW;
                F.dinv[tb + q] = di;
            }
            __syncwarp();
        }
    }
}

// z = M^-1 r on one tile staged in T (natural layout), in place; returns this lane's part of r'z.
// The wavefront step t = i + 3 jl is run as groups G = t / 3 of three sub-steps s = t mod 3:
// in group G lane i handles its single point jl = G - i / 3 at sub-step i mod 3, so the five
// factor values it needs in a group are known in advance -- they are loaded kIlu2Pre groups
// ahead (a register ring) and the recurrence waits on shared memory and shuffles only.
constexpr int kIlu2Groups = 42;                    // (31 + 3 * 31) / 3 + 1
constexpr int kIlu2Pre = 4;                        // groups of factor loads in flight
struct F5 {
    double a, b, c, d, e;
};

__device__ __forceinline__ double tile_solve_ilu2(const StencilOp& A, int x0, int y0, long long tb,
                                                  const Bj2Factor& F, double* __restrict__ z, double* T) {
    const int lane = threadIdx.x & 31;
    const int i3 = lane / 3, sl = lane - 3 * i3;
    // forward L y = r: values of the lane's point of group G (lS, lSE, lSEE, lW, 1/d)
    auto ldf = [&](int G) {
        const int jl = G - i3;
        F5 v{0.0, 0.0, 0.0, 0.0, 0.0};
        if (jl >= 0 && jl < kTile) {
            const long long q = tb + jl * kTile + lane;
            v.a = __ldg(F.lS + q); v.b = __ldg(F.lSE + q); v.c = __ldg(F.lSEE + q);
            v.d = __ldg(F.lW + q); v.e = __ldg(F.dinv + q);
        }
        return v;
    };
    double rz = 0.0;
    F5 ring[kIlu2Pre];
#pragma unroll
    for (int d = 0; d < kIlu2Pre; ++d) ring[d] = ldf(d);
    __syncwarp();
#pragma unroll 1
    for (int G0 = 0; G0 < kIlu2Groups; G0 += kIlu2Pre) {
#pragma unroll
        for (int d = 0; d < kIlu2Pre; ++d) {
            const int G = G0 + d;
            const F5 f = ring[d];
            ring[d] = ldf(G + kIlu2Pre);
            const int jl = G - i3;
            const bool act = jl >= 0 && jl < kTile;
#pragma unroll
            for (int s3 = 0; s3 < 3; ++s3) {
                if (act && sl == s3) {
                    const int q = jl * kTile + lane;
                    double y = T[q];
                    if (jl > 0) {
                        y = fma(-f.a, T[q - kTile], y);
                        if (lane + 1 < kTile) y = fma(-f.b, T[q - kTile + 1], y);
                        if (lane + 2 < kTile) y = fma(-f.c, T[q - kTile + 2], y);
                    }
                    if (lane > 0) y = fma(-f.d, T[q - 1], y);
                    T[q] = y;
                    rz = fma(y * y, f.e, rz);
                }
                __syncwarp();
            }
        }
    }
    // backward: z_v = y_v / d_v - (l_{E,W} z_E + l_{N,S} z_N + l_{NW,SE} z_NW + l_{NWW,SEE} z_NWW)
    auto ldb = [&](int G) {
        const int jl = G - i3;
        F5 v{0.0, 0.0, 0.0, 0.0, 0.0};
        if (jl >= 0 && jl < kTile) {
            const long long q = tb + jl * kTile + lane;
            if (lane + 1 < kTile) v.a = __ldg(F.lW + q + 1);                    // E
            if (jl + 1 < kTile) {
                v.b = __ldg(F.lS + q + kTile);                                  // N
                if (lane > 0) v.c = __ldg(F.lSE + q + kTile - 1);               // NW
                if (lane > 1) v.d = __ldg(F.lSEE + q + kTile - 2);              // NWW
            }
            v.e = __ldg(F.dinv + q);
        }
        return v;
    };
#pragma unroll
    for (int d = 0; d < kIlu2Pre; ++d) ring[d] = ldb(kIlu2Groups - 1 - d);
#pragma unroll 1
    for (int G0 = kIlu2Groups - 1; G0 >= 0; G0 -= kIlu2Pre) {
#pragma unroll
        for (int d = 0; d < kIlu2Pre; ++d) {
            const int G = G0 - d;
            const F5 f = ring[d];
            ring[d] = ldb(G - kIlu2Pre);
            const int jl = G - i3;
            const bool act = jl >= 0 && jl < kTile;
#pragma unroll
            for (int s3 = 2; s3 >= 0; --s3) {
                if (act && sl == s3) {
                    const int q = jl * kTile + lane;
                    double sacc = 0.0;
                    if (lane + 1 < kTile) sacc = fma(f.a, T[q + 1], sacc);
                    if (jl + 1 < kTile) {
                        sacc = fma(f.b, T[q + kTile], sacc);
                        if (lane > 0) sacc = fma(f.c, T[q + kTile - 1], sacc);
                        if (lane > 1) sacc = fma(f.d, T[q + kTile - 2], sacc);
                    }
                    T[q] = fma(T[q], f.e, -sacc);
                }
                __syncwarp();
            }
        }
    }
    const int i = x0 + lane;
#pragma unroll 8
    for (int jl = 0; jl < kTile; ++jl) {
        const int j = y0 + jl;
        if (i < A.nx && j < A.ny) z[i + (long long)A.pitch * j] = T[jl * kTile + lane];
    }
    __syncwarp();
    return rz;
}

// as k_pcg2_solve (bjilu.cuh) with the ILU(2) tile solve
template <int KIND>   // 0: init solve (gamma_0), 1: iteration update + solve (gamma_{j+1})
__global__ void __launch_bounds__(kBjThreads, kBjMinBlocks)
k_pcg3_solve(StencilOp A, Bj2Factor F, const __grid_constant__ CUtensorMap m_r, int row0, double* __restrict__ r,
             const double* __restrict__ q, double* __restrict__ z, double eta2, long long cap, Scal* S,
             RedScratch R) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint64_t bars[kBjThreads / 32];
    if (KIND == 1 && *(volatile int*)&S->cg_done) return;
    const double alpha = KIND == 1 ? S->cg_alpha : 0.0;
    double acc[1] = {0.0};
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    double* T = reinterpret_cast<double*>(base) + wid * kTile * kTile;
    uint64_t* bar = &bars[wid];
    if (lane == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t phase = 0;
    for_each_tile(A, [&](int x0, int y0, int tt) {
        if (lane == 0) {
            fence_proxy_async();
            mbar_expect_tx(bar, kTile * kTile * 8);
            tma_load_2d(T, &m_r, x0, y0 + row0, bar);
        }
        const int i = x0 + lane;
        const int ic = i < A.nx ? i : x0;
        mbar_wait(bar, phase);
        phase ^= 1;
#pragma unroll 16
        for (int jl = 0; jl < kTile; ++jl) {
            const int j = y0 + jl;
            const bool in = i < A.nx && j < A.ny;
            double rv = T[jl * kTile + lane];
            if (KIND == 1) {
                rv = fma(-alpha, q[ic + (long long)A.pitch * min(j, A.ny - 1)], rv);
                if (in) r[i + (long long)A.pitch * j] = rv;
            }
            T[jl * kTile + lane] = in ? rv : 0.0;
        }
        acc[0] += tile_solve_ilu2(A, x0, y0, (long long)tt * kTile * kTile, F, z, T);
    });
    reduce_and_finish<1>(acc, R, [&](double* t) {
        if (KIND == 0) pcg2_init_fin(t[0], eta2, cap, S);
        else pcg2_beta_fin(t[0], S);
    });
}

}  // namespace gpcg
