// tile.cuh -- TMA-tiled stencil sweeps (sm_100a) for the broadcast-face
// 5-point operator of the journal-bearing family (C0 / C2 / C3).
//
// A CTA owns a tile of 60 x 32 output points.  The inputs of the tile plus a
// 2-point halo (a 64 x 36 box) are brought into shared memory by the Tensor
// Memory Accelerator (cp.async.bulk.tensor.2d, one instruction per array,
// completion counted on an mbarrier); points outside the grid are zero-filled
// by the TMA unit, which is exactly the Dirichlet boundary.  The levels of a
// fused sweep (e.g. p_i, then rho - alpha A p_i, then A rho) are then computed
// for the whole tile from shared memory with every thread working on
// independent points, separated by __syncthreads.  CTAs are persistent over a
// fixed tile sequence; with NSTAGE = 2 the next tile's TMA load is in flight
// while the current one is computed.
//
// Same arithmetic and same reduction structure as the column-march kernels
// (march.cuh) -- both are checked against the CPU oracle.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "march.cuh"

namespace gpcg {

constexpr int kTileThreads = 256;
constexpr int TBW = 64;                 // box width (columns), incl. halo
constexpr int TBH = 36;                 // box height (rows), incl. halo
constexpr int THALO = 2;
constexpr int TOX = TBW - 2 * THALO;    // 60 output columns
constexpr int TOY = TBH - 2 * THALO;    // 32 output rows
constexpr int kBoxF64 = TBW * TBH * 8;  // 18432 bytes
// u8 boxes (free masks): the TMA box start must be 16-byte aligned in the inner
// dimension, so mask boxes start at floor16(x) and are 80 columns wide; the
// tile's 64 columns then sit at offset moff = x - floor16(x) in [0, 16).
constexpr int MBW = 80;
constexpr int kBoxU8 = 2944;            // MBW * TBH = 2880, padded to a multiple of 128
constexpr int kCtrF64 = TOX * TOY * 8;  // 15360 bytes (centre box, CG w)

struct TileGeom {
    int nx, ny, pitch;
    int ntx, nty;       // tiles per row / column (over the owned rows)
    int rlo, rhi;       // readable rows (owned + ghost, StencilOp); the tensor maps start at row rlo
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ int floor16(int x) { return x & ~15; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 2-D tile load: box at element coordinates (x, y) of the tensor (may be negative / out of range:
// those elements are zero-filled).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// Broadcast face weights of the 64 box columns of a tile (zero outside the grid).
struct ColFaces {
    double fw[TBW], fe[TBW], fs[TBW], dg[TBW];
};
__device__ __forceinline__ void load_colfaces(ColFaces& F, const StencilOp& A, int gx0) {
    for (int c = threadIdx.x; c < TBW; c += blockDim.x) {
        const int gc = gx0 + c;
        double w = 0.0, e = 0.0, s = 0.0;
        if (gc >= 0 && gc < A.nx) {
            w = __ldg(A.wx + gc);
            e = __ldg(A.wx + gc + 1);
            s = __ldg(A.wy + gc);
        }
        F.fw[c] = w; F.fe[c] = e; F.fs[c] = s; F.dg[c] = (w + e) + (s + s);
    }
}
// (A v) at box point (r, c) of a box-shaped smem array
__device__ __forceinline__ double apply_box(const ColFaces& F, const double* v, int r, int c) {
    const int k = r * TBW + c;
    double t = F.dg[c] * v[k];
    t = fma(-F.fw[c], v[k - 1], t);
    t = fma(-F.fe[c], v[k + 1], t);
    return fma(-F.fs[c], v[k - TBW] + v[k + TBW], t);
}

// ============================================================================
// a5: CG iteration (same recurrences as k2_cg_iter).  Stage layout:
//   rho [TBH][TBW] f64 | p [TBH][TBW] f64 | w [TOY][TOX] f64 | mask [TBH][TBW] u8
// level 1 (whole box):        pn = [m] (rho + beta p)            -> in place of p
// level 2 (rows/cols 1..-2):  rn = [m] (rho - alpha (A pn))      -> in place of rho
// level 3 (centre 60 x 32):   q = A rn; gamma += rn^2, delta += rn q;
//                             w += alpha pn, rho' = rn, p' = pn  (free points only)
// ============================================================================
template <int NSTAGE>
struct CgStage {
    static constexpr int kRho = 0, kP = kBoxF64, kW = 2 * kBoxF64, kMask = 2 * kBoxF64 + kCtrF64;
    static constexpr int kBytes = 2 * kBoxF64 + kCtrF64 + kBoxU8;   // multiple of 128
    static constexpr int kTx = 2 * kBoxF64 + kCtrF64 + MBW * TBH;   // bytes the TMA delivers
    static constexpr int kSmem = NSTAGE * kBytes + (int)sizeof(ColFaces) + 64;
};

template <int NSTAGE>
__global__ void __launch_bounds__(kTileThreads, 2)
k3_cg_iter(StencilOp A, TileGeom T, const __grid_constant__ CUtensorMap m_rho, const __grid_constant__ CUtensorMap m_p,
           const __grid_constant__ CUtensorMap m_w, const __grid_constant__ CUtensorMap m_mask,
           double* __restrict__ rho_n, double* __restrict__ p_n, double* __restrict__ w, Scal* S, RedScratch R) {
    if (*(volatile int*)&S->cg_done) return;
    using L = CgStage<NSTAGE>;
    extern __shared__ __align__(128) unsigned char smem[];
    ColFaces& F = *reinterpret_cast<ColFaces*>(smem + NSTAGE * L::kBytes);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + NSTAGE * L::kBytes + sizeof(ColFaces));
    const double alpha = S->cg_alpha, beta = S->cg_beta;
    const int ntiles = T.ntx * T.nty;
    auto issue = [&](int stage, int t) {
        unsigned char* st = smem + stage * L::kBytes;
        const int x0 = (t % T.ntx) * TOX, y0 = (t / T.ntx) * TOY;
        mbar_expect_tx(&bar[stage], L::kTx);
        tma_load_2d(st + L::kRho, &m_rho, x0 - THALO, y0 - THALO - T.rlo, &bar[stage]);
        tma_load_2d(st + L::kP, &m_p, x0 - THALO, y0 - THALO - T.rlo, &bar[stage]);
        tma_load_2d(st + L::kW, &m_w, x0, y0 - T.rlo, &bar[stage]);
        tma_load_2d(st + L::kMask, &m_mask, floor16(x0 - THALO), y0 - THALO - T.rlo, &bar[stage]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (int s = 0; s < NSTAGE; ++s) {
            const int t = blockIdx.x + s * gridDim.x;
            if (t < ntiles) issue(s, t);
        }
    }
    __syncthreads();
    double acc[2] = {0.0, 0.0};
    int k = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int stage = k % NSTAGE;
        const uint32_t parity = (k / NSTAGE) & 1;
        unsigned char* st = smem + stage * L::kBytes;
        double* rho = reinterpret_cast<double*>(st + L::kRho);
        double* p = reinterpret_cast<double*>(st + L::kP);
        const double* ws = reinterpret_cast<const double*>(st + L::kW);
        const unsigned char* m = st + L::kMask;
        const int x0 = (t % T.ntx) * TOX, y0 = (t / T.ntx) * TOY;
        const int moff = (x0 - THALO) - floor16(x0 - THALO);
        load_colfaces(F, A, x0 - THALO);
        mbar_wait(&bar[stage], parity);
        // level 1: pn over the whole box
        for (int q = threadIdx.x; q < TBW * TBH; q += kTileThreads) {
            const int r = q / TBW, c = q % TBW;
            p[q] = m[r * MBW + c + moff] ? fma(beta, p[q], rho[q]) : 0.0;
        }
        __syncthreads();
        // level 2: rn on rows 1..TBH-2, cols 1..TBW-2
        for (int q = threadIdx.x; q < (TBH - 2) * (TBW - 2); q += kTileThreads) {
            const int r = 1 + q / (TBW - 2), c = 1 + q % (TBW - 2);
            const int kk = r * TBW + c;
            if (m[r * MBW + c + moff]) rho[kk] = fma(-alpha, apply_box(F, p, r, c), rho[kk]);
            else rho[kk] = 0.0;
        }
        __syncthreads();
        // level 3: centre
        for (int q = threadIdx.x; q < TOX * TOY; q += kTileThreads) {
            const int r = THALO + q / TOX, c = THALO + q % TOX;
            const int kk = r * TBW + c;
            if (m[r * MBW + c + moff] && y0 + r - THALO < T.ny) {     // owned rows only (ghost rows: the exchange)
                const double rn = rho[kk];
                const double qv = apply_box(F, rho, r, c);
                acc[0] = fma(rn, rn, acc[0]);
                acc[1] = fma(rn, qv, acc[1]);
                const long long v = (long long)(x0 + c - THALO) + (long long)T.pitch * (y0 + r - THALO);
                const double pn = p[kk];
                w[v] = fma(alpha, pn, ws[q]);
                rho_n[v] = rn;
                p_n[v] = pn;
            }
        }
        __syncthreads();                          // stage and face table free again
        if (threadIdx.x == 0 && t + NSTAGE * (int)gridDim.x < ntiles) {
            fence_proxy_async();                  // generic-proxy smem writes before the async-proxy refill
            issue(stage, t + NSTAGE * gridDim.x);
        }
    }
    reduce_and_finish<2>(acc, R, [&](double* tt) { cg_finalize(tt[0], tt[1], S); });
}

// ============================================================================
// a1 + a2 fused (accept / project + regrad + mask + counts + next Cauchy form).
// Stage: y | dir | b | l | u | mask_prev   (boxes; dir, l/u, mask_prev optional)
// level 1 (box):        yn = mid(l, u, y + alpha sgn dir)       -> in place of y
// level 2 (inner box):  gn = A yn - b -> GN;  d = pgrad(yn, gn)  -> in place of b
// level 3 (centre):     Ad = A d; sums; y_out = yn, g_out = gn, mask_out
// ============================================================================
template <bool SB>
struct AccStage {
    static constexpr int kY = 0, kD = kBoxF64, kB = 2 * kBoxF64;
    static constexpr int kL = 3 * kBoxF64, kU = SB ? kL : 4 * kBoxF64;
    static constexpr int kMP = SB ? 3 * kBoxF64 : 5 * kBoxF64;
    static constexpr int kBytes = kMP + kBoxU8;         // kBoxU8 = 18 * 128: stays 128-byte aligned
    static constexpr int kGN = kBytes;                  // single-buffered derived array
    static constexpr int kSmem = kBytes + kBoxF64 + (int)sizeof(ColFaces) + 64;
};

template <bool SB>
__global__ void __launch_bounds__(kTileThreads, 1)
k3_accept(StencilOp A, TileGeom T, Bounds Bd, const __grid_constant__ CUtensorMap m_y,
          const __grid_constant__ CUtensorMap m_dir, const __grid_constant__ CUtensorMap m_b,
          const __grid_constant__ CUtensorMap m_l, const __grid_constant__ CUtensorMap m_u,
          const __grid_constant__ CUtensorMap m_mp, int has_dir, double sgn, int has_mp,
          double* __restrict__ y_out, double* __restrict__ g_out, unsigned char* __restrict__ mask_out,
          Scal* S, RedScratch R, int gp) {
    if (gp && *(volatile int*)&S->gp_done) return;   // device-driven GP phase already over
    double alpha = 0.0;
    if (has_dir) {
        if (S->s_h < 0) return;
        alpha = S->s_alpha;
    }
    using L = AccStage<SB>;
    extern __shared__ __align__(128) unsigned char smem[];
    double* y = reinterpret_cast<double*>(smem + L::kY);
    double* dir = reinterpret_cast<double*>(smem + L::kD);
    double* bd = reinterpret_cast<double*>(smem + L::kB);
    const double* lb = reinterpret_cast<const double*>(smem + L::kL);
    const double* ub = reinterpret_cast<const double*>(smem + L::kU);
    const unsigned char* mp = smem + L::kMP;
    double* gn = reinterpret_cast<double*>(smem + L::kGN);
    ColFaces& F = *reinterpret_cast<ColFaces*>(smem + L::kGN + kBoxF64);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kGN + kBoxF64 + sizeof(ColFaces));
    const int ntiles = T.ntx * T.nty;
    const uint32_t bytes = kBoxF64 * (2 + (has_dir ? 1 : 0) + (SB ? 0 : 2)) + (has_mp ? MBW * TBH : 0);
    auto issue = [&](int t) {
        const int x0 = (t % T.ntx) * TOX - THALO, y0 = (t / T.ntx) * TOY - THALO - T.rlo;
        mbar_expect_tx(&bar[0], bytes);
        tma_load_2d(y, &m_y, x0, y0, &bar[0]);
        if (has_dir) tma_load_2d(dir, &m_dir, x0, y0, &bar[0]);
        tma_load_2d(bd, &m_b, x0, y0, &bar[0]);
        if (!SB) {
            tma_load_2d(smem + L::kL, &m_l, x0, y0, &bar[0]);
            tma_load_2d(smem + L::kU, &m_u, x0, y0, &bar[0]);
        }
        if (has_mp) tma_load_2d(smem + L::kMP, &m_mp, floor16(x0), y0, &bar[0]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        fence_mbar_init();
        if ((int)blockIdx.x < ntiles) issue(blockIdx.x);
    }
    __syncthreads();
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int k = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int x0 = (t % T.ntx) * TOX, y0 = (t / T.ntx) * TOY;
        const int moff = (x0 - THALO) - floor16(x0 - THALO);
        load_colfaces(F, A, x0 - THALO);
        mbar_wait(&bar[0], k & 1);
        // level 1: yn over the box; out-of-grid points: y = dir = 0, bounds forced to 0 -> yn = 0
        for (int q = threadIdx.x; q < TBW * TBH; q += kTileThreads) {
            const int r = q / TBW, c = q % TBW;
            const int gi = x0 - THALO + c, gj = y0 - THALO + r;
            const bool in = gi >= 0 && gi < T.nx && gj >= T.rlo && gj < T.rhi;
            const double l = in ? (SB ? Bd.lc : lb[q]) : 0.0, u = in ? (SB ? Bd.uc : ub[q]) : 0.0;
            y[q] = has_dir ? trial(y[q], dir[q], sgn, alpha, l, u) : mid(l, u, y[q]);
        }
        __syncthreads();
        // level 2: gn and d on the inner box
        for (int q = threadIdx.x; q < (TBH - 2) * (TBW - 2); q += kTileThreads) {
            const int r = 1 + q / (TBW - 2), c = 1 + q % (TBW - 2);
            const int kk = r * TBW + c;
            const int gi = x0 - THALO + c, gj = y0 - THALO + r;
            const bool in = gi >= 0 && gi < T.nx && gj >= T.rlo && gj < T.rhi;
            const double g = apply_box(F, y, r, c) - bd[kk];
            gn[kk] = g;
            const double l = in ? (SB ? Bd.lc : lb[kk]) : 0.0, u = in ? (SB ? Bd.uc : ub[kk]) : 0.0;
            bd[kk] = in ? pgrad(y[kk], g, l, u) : 0.0;
        }
        __syncthreads();
        // level 3: centre
        for (int q = threadIdx.x; q < TOX * TOY; q += kTileThreads) {
            const int r = THALO + q / TOX, c = THALO + q % TOX;
            const int gi = x0 + c - THALO, gj = y0 + r - THALO;
            if (gi < T.nx && gj < T.ny) {
                const int kk = r * TBW + c;
                const double yn = y[kk], g = gn[kk], d = bd[kk];
                const double ad = apply_box(F, bd, r, c);
                const double l = SB ? Bd.lc : lb[kk], u = SB ? Bd.uc : ub[kk];
                const long long v = (long long)gi + (long long)T.pitch * gj;
                y_out[v] = yn;
                g_out[v] = g;
                const bool act = (yn == l) || (yn == u);
                const unsigned char mm = act ? 0 : 1;
                mask_out[v] = mm;
                acc[0] = fma(d, d, acc[0]);
                acc[1] = fma(g, g, acc[1]);
                acc[2] += act ? 1.0 : 0.0;
                if (has_mp) acc[3] += (mp[r * MBW + c + moff] != mm) ? 1.0 : 0.0;
                const bool binding = (yn == l && g >= 0.0) || (yn == u && g <= 0.0);
                acc[4] += (act && !binding) ? 1.0 : 0.0;
                acc[5] = fma(d, ad, acc[5]);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && t + (int)gridDim.x < ntiles) {
            fence_proxy_async();
            issue(t + gridDim.x);
        }
    }
    reduce_and_finish<6>(acc, R, [&](double* tt) { fin_accept(tt, true, S); });
}

// ============================================================================
// a3: projected search with K = 2 step sizes per sweep.
// Stage: y | dir | g (if !DG) | l | u (if !SB);  derived: s_0, s_1 (boxes)
// level 1 (box):    s_h = mid(l, u, y + alpha_h sgn dir) - y
// level 2 (centre): <g, s_h>, <s_h, A s_h>
// ============================================================================
template <bool SB, bool DG>
struct SrchStage {
    static constexpr int kY = 0, kD = kBoxF64;
    static constexpr int kG = DG ? kD : 2 * kBoxF64;
    static constexpr int kL = (DG ? 2 : 3) * kBoxF64;
    static constexpr int kU = SB ? kL : kL + kBoxF64;
    static constexpr int kBytes = SB ? kL : kL + 2 * kBoxF64;
    static constexpr int kS = kBytes;
    static constexpr int kSmem = kBytes + 2 * kBoxF64 + (int)sizeof(ColFaces) + 64;
};

template <bool SB, bool DG>
__global__ void __launch_bounds__(kTileThreads, 1)
k3_search(StencilOp A, TileGeom T, Bounds Bd, const __grid_constant__ CUtensorMap m_y,
          const __grid_constant__ CUtensorMap m_dir, const __grid_constant__ CUtensorMap m_g,
          const __grid_constant__ CUtensorMap m_l, const __grid_constant__ CUtensorMap m_u, double sgn,
          int use_alpha0, int h0, double mu, Scal* S, RedScratch R, int gp) {
    constexpr int K = 2;
    if (gp && *(volatile int*)&S->gp_done) return;   // device-driven GP phase already over
    if (use_alpha0 && !S->cauchy_ok) {
        if (blockIdx.x == 0 && threadIdx.x == 0) S->s_h = -1;
        return;
    }
    const double base = use_alpha0 ? S->alpha0 : 1.0;
    const double al0 = scalbn(base, -h0), al1 = scalbn(base, -(h0 + 1));
    using L = SrchStage<SB, DG>;
    extern __shared__ __align__(128) unsigned char smem[];
    const double* y = reinterpret_cast<const double*>(smem + L::kY);
    const double* dir = reinterpret_cast<const double*>(smem + L::kD);
    const double* g = reinterpret_cast<const double*>(smem + L::kG);
    const double* lb = reinterpret_cast<const double*>(smem + L::kL);
    const double* ub = reinterpret_cast<const double*>(smem + L::kU);
    double* s0 = reinterpret_cast<double*>(smem + L::kS);
    double* s1 = reinterpret_cast<double*>(smem + L::kS + kBoxF64);
    ColFaces& F = *reinterpret_cast<ColFaces*>(smem + L::kS + 2 * kBoxF64);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kS + 2 * kBoxF64 + sizeof(ColFaces));
    const int ntiles = T.ntx * T.nty;
    auto issue = [&](int t) {
        const int x0 = (t % T.ntx) * TOX - THALO, y0 = (t / T.ntx) * TOY - THALO - T.rlo;
        mbar_expect_tx(&bar[0], L::kBytes);
        tma_load_2d(smem + L::kY, &m_y, x0, y0, &bar[0]);
        tma_load_2d(smem + L::kD, &m_dir, x0, y0, &bar[0]);
        if (!DG) tma_load_2d(smem + L::kG, &m_g, x0, y0, &bar[0]);
        if (!SB) {
            tma_load_2d(smem + L::kL, &m_l, x0, y0, &bar[0]);
            tma_load_2d(smem + L::kU, &m_u, x0, y0, &bar[0]);
        }
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        fence_mbar_init();
        if ((int)blockIdx.x < ntiles) issue(blockIdx.x);
    }
    __syncthreads();
    double acc[2 * K] = {0.0, 0.0, 0.0, 0.0};
    int k = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int x0 = (t % T.ntx) * TOX, y0 = (t / T.ntx) * TOY;
        load_colfaces(F, A, x0 - THALO);
        mbar_wait(&bar[0], k & 1);
        for (int q = threadIdx.x; q < TBW * TBH; q += kTileThreads) {
            const int r = q / TBW, c = q % TBW;
            const int gi = x0 - THALO + c, gj = y0 - THALO + r;
            const bool in = gi >= 0 && gi < T.nx && gj >= T.rlo && gj < T.rhi;
            const double l = in ? (SB ? Bd.lc : lb[q]) : 0.0, u = in ? (SB ? Bd.uc : ub[q]) : 0.0;
            const double yv = y[q], dv = dir[q];
            s0[q] = trial(yv, dv, sgn, al0, l, u) - yv;
            s1[q] = trial(yv, dv, sgn, al1, l, u) - yv;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < TOX * TOY; q += kTileThreads) {
            const int r = THALO + q / TOX, c = THALO + q % TOX;
            const int gi = x0 + c - THALO, gj = y0 + r - THALO;
            if (gi < T.nx && gj < T.ny) {
                const int kk = r * TBW + c;
                const double gv = g[kk];
                const double a0 = apply_box(F, s0, r, c), a1 = apply_box(F, s1, r, c);
                acc[0] = fma(gv, s0[kk], acc[0]);
                acc[1] = fma(s0[kk], a0, acc[1]);
                acc[2] = fma(gv, s1[kk], acc[2]);
                acc[3] = fma(s1[kk], a1, acc[3]);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && t + (int)gridDim.x < ntiles) {
            fence_proxy_async();
            issue(t + gridDim.x);
        }
    }
    reduce_and_finish<2 * K>(acc, R, [&](double* tt) { fin_search(tt, K, h0, base, mu, S); });
}

}  // namespace gpcg
