// bjilu.cuh -- block-Jacobi ILU(0) preconditioned CG on the free set (SURVEY.md 8(f)
// NEXT-3; the paper's block Jacobi with ILU(0) subdomain solves, Table 4)
// for 2-D 5-point stencils (gpcg_params.precond = 2).
//
// Blocks: 32 x 32 tiles of a slab's owned grid (tile (bi, bj) = columns 32 bi .., rows
// 32 bj .. of the slab; entries coupling tiles are dropped).  Within a tile the rows of
// A_k in natural order; ILU(0) keeps the 5-point pattern, so only the pivots change:
//     d_v = a_vv - a_vs^2 / d_s - a_vw^2 / d_w      (south / west neighbour in the tile, free)
// and M = (D + L) D^-1 (D + U) (oracle/gpcg_oracle.c ora_bjilu_*).  One warp owns a tile:
// lane i is column i, and anti-diagonal l = i + jl is step l of a 63-step wavefront -- the
// west neighbour of (i, jl) was computed by lane i-1 one step earlier (warp shuffle), the
// south neighbour by the same lane one step earlier (register).  The factor is stored, and
// the tile staged, in a skewed layout (sk() below) in which every wavefront step is one
// contiguous row, so a step costs a shared-memory access, two FMAs and a shuffle; the factor
// loads are independent of the recurrence and run ahead of it.
//
// PCG (textbook form, the oracle's ora_pcg_m): per iteration
//   k_pcg2_matvec: w += alpha_prev p_old, p = z + beta p (at the point and its neighbours),
//                  q = A_F p, sum p'q
//                  -> alpha = gamma / p'q
//   k_pcg2_solve<1>: r -= alpha q, z = M^-1 r (tile wavefronts), sum r'z
//                  -> decrease 1/2 alpha gamma, cgstop1 / exact guard / cap, beta
// Vectors (full length, zero off F): r, z, p (ping-pong), q; the factor (BjFactor) per slab.
#pragma once

#include "common.cuh"
#include "fin.cuh"
#include "tma.cuh"

namespace gpcg {

constexpr int kTile = 32;
#ifndef GPCG_BJ_UNROLL
#define GPCG_BJ_UNROLL 4
#endif

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

// tiles of the slab, one per warp (grid-stride over tiles); body(x0, y0, tile index)
template <class Body>
__device__ __forceinline__ void for_each_tile(const StencilOp& A, Body&& body) {
    const int ntx = (A.nx + kTile - 1) / kTile, nty = (A.ny + kTile - 1) / kTile;
    const int nt = ntx * nty;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int t = warp; t < nt; t += nw) body((t % ntx) * kTile, (t / ntx) * kTile, t);
}

// Skewed tile layout of the factor (and of the per-warp shared-memory staging): element
// (i, jl) of a tile sits at row (i + jl) mod 32, column i.  Wavefront step l touches the
// points with i + jl = l, i.e. row l mod 32 -- 32 consecutive doubles (lanes with
// i + jl = l and i + jl = l - 32 never coexist in one step, so the map is a bijection and
// each step is one coalesced 256-byte access); a row-major pass over the tile (fixed jl,
// lane i) hits 32 distinct bank pairs.
__device__ __forceinline__ int sk(int i, int jl) { return ((i + jl) & (kTile - 1)) * kTile + i; }

// The factor of every tile in the skewed layout, kTile^2 doubles per tile and array:
//   dinv = 1 / d_v on F, 0 off F (so the solves need no mask: off F every t, z is 0),
//   cs   = w_s (the coupling -a_vs) if v, s in F and s in the tile, else 0,
//   cw   = w_w likewise for the west neighbour.
// The backward solve reads the north / east couplings as cs of (i, jl + 1) and cw of (i + 1, jl)
// (A symmetric; cs of a tile's row 0 and cw of its column 0 are 0, which drops the couplings
// across tile edges).
// Broadcast faces (journal bearing: the couplings of column i are the same in every row):
// instead of cs / cw the factor stores one code byte per element -- bit 0: the south
// coupling is present (v, s in F, s in the tile), bit 1: the west one -- and the solve forms
// cs = bit0 ? w_s(i) : 0, cw = bit1 ? w_w(i) : 0 from the lane's column faces held in
// registers: 9 instead of 24 bytes of factor per element and wavefront step.
struct BjFactor {
    double *dinv, *cs, *cw;
    unsigned char* code;
};

constexpr int kBjThreads = 64;                                        // 2 tiles per CTA
constexpr int kBjMinBlocks = 9;                                       // 18 tiles / SM in flight
constexpr int kFactorSmem = (kBjThreads / 32) * kTile * kTile * (3 * 8 + 1);
constexpr int kSolveSmem = (kBjThreads / 32) * kTile * kTile * 8 + 128;   // + alignment pad

// ILU(0) pivots of every tile on the CG mask: d_v = a_vv - cs^2 / d_s - cw^2 / d_w (south first,
// the oracle's column order).  Staged per warp in shared memory (skewed), then one 63-step
// wavefront; cs / cw go out as soon as they are formed, dinv at its wavefront step.
__global__ void __launch_bounds__(kBjThreads)
k_bjilu_factor(StencilOp A, const unsigned char* __restrict__ mask, BjFactor F) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* Da = reinterpret_cast<double*>(smem_raw) + wid * 3 * kTile * kTile;
    double* Ds = Da + kTile * kTile;
    double* Dw = Ds + kTile * kTile;
    unsigned char* Mf = smem_raw + (kBjThreads / 32) * 3 * kTile * kTile * 8 + wid * kTile * kTile;
    for_each_tile(A, [&](int x0, int y0, int tt) {
        const long long tb = (long long)tt * kTile * kTile;
        const int i = x0 + lane;
        for (int jl = 0; jl < kTile; ++jl) {
            const int j = y0 + jl;
            const int q = sk(lane, jl);
            double a = 0.0, cs = 0.0, cw = 0.0;
            unsigned char f = 0;
            if (i < A.nx && j < A.ny) {
                const long long v = i + (long long)A.pitch * j;
                if (mask[v]) {
                    const Faces5 fc = faces_at(A, i, j);
                    a = fc.d;
                    if (jl > 0 && mask[v - A.pitch]) cs = fc.s;
                    if (lane > 0 && mask[v - 1]) cw = fc.w;
                    f = 1;
                }
            }
            Da[q] = a;
            Ds[q] = cs;
            Dw[q] = cw;
            Mf[q] = f;
            if (F.code) {
                F.code[tb + q] = (unsigned char)((cs != 0.0 ? 1 : 0) | (cw != 0.0 ? 2 : 0));
            } else {
                F.cs[tb + q] = cs;
                F.cw[tb + q] = cw;
            }
        }
        __syncwarp();
        double d_prev = 1.0;                              // d of (i, jl - 1): this lane, previous step
        for (int l = 0; l < 2 * kTile - 1; ++l) {
            const double d_west = __shfl_up_sync(0xffffffffu, d_prev, 1);   // (i - 1, jl), step l - 1
            if ((unsigned)(l - lane) < (unsigned)kTile) {
                const int q = (l & (kTile - 1)) * kTile + lane;
                double dn = 1.0, di = 0.0;
                if (Mf[q]) {
                    const double cs = Ds[q], cw = Dw[q];
                    dn = Da[q] - cs * cs / d_prev - cw * cw / d_west;
                    di = 1.0 / dn;
                }
                F.dinv[tb + q] = di;
                d_prev = dn;
            }
        }
        __syncwarp();
    });
}

// z = M^-1 r on one tile whose r is staged in T (natural layout: (i, jl) at jl * 32 + i):
// forward (D + L) t = r, backward D^-1 (D + U) z = t, both in place in T; then z is stored
// row by row.  Wavefront step l touches T at (l - i) * 32 + i: 32 distinct bank pairs
// (-31 = 1 mod 16), so the diagonal access is conflict-free without skewing T.  Returns this
// lane's share of r'z, formed in the forward sweep as t'D t = sum t_v (D t)_v: with U = L^T,
// r'z = r'(D + U)^-1 D t = ((D + L)^-1 r)' D t = t'D t, and (D t)_v is the sum the step
// forms before scaling by 1/d_v (so r need not be kept or re-read).
// The factor rows (skewed, one contiguous 256-byte row per step) are loaded in groups of
// kBjGroup steps, double-buffered: group g + 1 is in flight while group g runs, so the
// recurrence waits on shared memory and shuffles, not on the loads.
constexpr int kBjGroup = GPCG_BJ_UNROLL;
constexpr int kBjSteps = 2 * kTile;                      // 63 wavefront steps + 1 idle (no active lane)

template <bool BC>
struct FacGroup {
    double d[kBjGroup], s[kBjGroup], w[kBjGroup];
    unsigned int c[BC ? kBjGroup : 1];
};

// BC: s / w are formed from the code byte and the lane's column faces fs / fw (0 when absent)
template <bool BWD, bool BC>
__device__ __forceinline__ void load_group(FacGroup<BC>& G, const double* Fd, const double* Fs, const double* Fw,
                                           const unsigned char* Fc, int g) {
#pragma unroll
    for (int k = 0; k < kBjGroup; ++k) {
        const int l = BWD ? kBjSteps - 1 - (g * kBjGroup + k) : g * kBjGroup + k;
        const int row = (l & (kTile - 1)) * kTile;
        const int nrow = BWD ? ((l + 1) & (kTile - 1)) * kTile : row;
        G.d[k] = __ldg(Fd + row);
        if constexpr (BC) {
            G.c[k] = __ldg(Fc + nrow);                   // fwd: code of (i, jl); bwd: of (i, jl + 1)
        } else {
            G.s[k] = __ldg(Fs + nrow);                   // fwd: cs of (i, jl); bwd: cs of (i, jl + 1)
            G.w[k] = __ldg(Fw + nrow);                   // fwd: cw of (i, jl); bwd: lane i+1 has cw of (i+1, jl)
        }
    }
}

template <bool BC>
__device__ __forceinline__ void decode_group(FacGroup<BC>& G, double fs, double fw) {
    if constexpr (BC) {
#pragma unroll
        for (int k = 0; k < kBjGroup; ++k) {
            G.s[k] = (G.c[k] & 1u) ? fs : 0.0;
            G.w[k] = (G.c[k] & 2u) ? fw : 0.0;
        }
    }
}

template <bool BC>
__device__ __forceinline__ double tile_solve(const StencilOp& A, int x0, int y0, long long tb, const BjFactor& F,
                                             double* __restrict__ z, double* T) {
    const int lane = threadIdx.x & 31;
    const double* Fd = F.dinv + tb + lane;
    const double* Fs = BC ? nullptr : F.cs + tb + lane;
    const double* Fw = BC ? nullptr : F.cw + tb + lane;
    const unsigned char* Fc = BC ? F.code + tb + lane : nullptr;
    double fs = 0.0, fw = 0.0;                            // BC: this column's south / west faces
    if (BC && x0 + lane < A.nx) {
        fs = __ldg(A.wy + x0 + lane);
        fw = __ldg(A.wx + x0 + lane);
    }
    constexpr int NG = kBjSteps / kBjGroup;
    __syncwarp();
    double t_prev = 0.0;                                  // t of (i, jl - 1)
    double rz = 0.0;
    FacGroup<BC> cur, nxt;
    load_group<false, BC>(cur, Fd, Fs, Fw, Fc, 0);
#pragma unroll 1
    for (int g = 0; g < NG; ++g) {
        if (g + 1 < NG) load_group<false, BC>(nxt, Fd, Fs, Fw, Fc, g + 1);
        decode_group<BC>(cur, fs, fw);
#pragma unroll
        for (int k = 0; k < kBjGroup; ++k) {
            const int l = g * kBjGroup + k;
            const int q = ((l - lane) & (kTile - 1)) * kTile + lane;
            const double t_west = __shfl_up_sync(0xffffffffu, t_prev, 1);   // (i - 1, jl), step l - 1
            const double sv = T[q] + cur.s[k] * t_prev + cur.w[k] * t_west;  // (D t)_v
            const double tv = sv * cur.d[k];
            if ((unsigned)(l - lane) < (unsigned)kTile) {
                T[q] = tv;
                t_prev = tv;
                rz = fma(tv, sv, rz);
            }
        }
        cur = nxt;
    }
    __syncwarp();
    double z_prev = 0.0;                                  // z of (i, jl + 1)
    load_group<true, BC>(cur, Fd, Fs, Fw, Fc, 0);
#pragma unroll 1
    for (int g = 0; g < NG; ++g) {
        if (g + 1 < NG) load_group<true, BC>(nxt, Fd, Fs, Fw, Fc, g + 1);
        decode_group<BC>(cur, fs, fw);
#pragma unroll
        for (int k = 0; k < kBjGroup; ++k) {
            const int l = kBjSteps - 1 - (g * kBjGroup + k);
            const int q = ((l - lane) & (kTile - 1)) * kTile + lane;
            const double z_east = __shfl_down_sync(0xffffffffu, z_prev, 1);  // (i + 1, jl), step l + 1
            const double cwe = __shfl_down_sync(0xffffffffu, cur.w[k], 1);   // all lanes take part
            const double ce = lane < kTile - 1 ? cwe : 0.0;
            const double cn = cur.s[k];                                     // 0 when jl = 31 (row 0's cs)
            const double zv = T[q] + (ce * z_east + cn * z_prev) * cur.d[k];
            if ((unsigned)(l - lane) < (unsigned)kTile) {
                T[q] = zv;
                z_prev = zv;
            }
        }
        cur = nxt;
    }
    __syncwarp();
    const int i = x0 + lane;
#pragma unroll 8
    for (int jl = 0; jl < kTile; ++jl) {                  // store z (coalesced rows)
        const int j = y0 + jl;
        if (i < A.nx && j < A.ny) z[i + (long long)A.pitch * j] = T[jl * kTile + lane];
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

template <int KIND, bool BC>   // KIND 0: init solve (gamma_0), 1: iteration update + solve (gamma_{j+1})
__global__ void __launch_bounds__(kBjThreads, kBjMinBlocks)
k_pcg2_solve(StencilOp A, BjFactor F, const __grid_constant__ CUtensorMap m_r, int row0, double* __restrict__ r,
             const double* __restrict__ q, double* __restrict__ z, double eta2, long long cap, Scal* S,
             RedScratch R) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint64_t bars[kBjThreads / 32];
    if (KIND == 1 && *(volatile int*)&S->cg_done) return;
    const double alpha = KIND == 1 ? S->cg_alpha : 0.0;
    double acc[1] = {0.0};
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // TMA destinations must be 128-byte aligned; the dynamic block is padded by 128 for this
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
        // r tile -> T by TMA (zero outside the stored grid)
        if (lane == 0) {
            fence_proxy_async();                          // T's previous generic accesses before the async write
            mbar_expect_tx(bar, kTile * kTile * 8);
            tma_load_2d(T, &m_r, x0, y0 + row0, bar);
        }
        const int i = x0 + lane;
        const int ic = i < A.nx ? i : x0;
        mbar_wait(bar, phase);
        phase ^= 1;
        // KIND 1: r -= alpha q (r and q are 0 off F, so no mask), written back; rows / columns
        // outside the slab's owned grid are zeroed in T (the tile is the owned part).  w += alpha p
        // is deferred to the next matvec (k_pcg2_wlast after the last iteration).
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
        acc[0] += tile_solve<BC>(A, x0, y0, (long long)tt * kTile * kTile, F, z, T);
    });
    reduce_and_finish<1>(acc, R, [&](double* t) {
        if (KIND == 0) pcg2_init_fin(t[0], eta2, cap, S);
        else pcg2_beta_fin(t[0], S);
    });
}

// p_new = z + beta p_old (zero off F; formed at the neighbours too), q = A_F p_new, sum p'q
__global__ void __launch_bounds__(kThreads)
k_pcg2_matvec(StencilOp A, const unsigned char* __restrict__ mask, const double* __restrict__ z,
              const double* __restrict__ p_old, double* __restrict__ p_new, double* __restrict__ q,
              double* __restrict__ w, Scal* S, RedScratch R) {
    if (*(volatile int*)&S->cg_done) return;
    const double beta = S->cg_beta;
    const double alpha_prev = S->cg_alpha;                // alpha of the previous iteration (0 at the first)
    double acc[1] = {0.0};
    A.for_each_point([&](const Pt& pt) {
        const int v = pt.v;
        if (!mask[v]) { p_new[v] = 0.0; q[v] = 0.0; return; }
        w[v] = fma(alpha_prev, p_old[v], w[v]);           // the previous iteration's w += alpha p
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

// The same step as a 2-D tile sweep (the default): a 256-thread CTA owns a 32 x 32 output
// tile; p = z + beta p_old is formed once per point on the 34 x 34 tile + halo in shared
// memory (z and p_old are 0 off F, so no mask there; the loads of the fill are independent),
// then every thread applies the 5-point operator to 4 points from shared memory, in the
// order of Op5::apply.  w += alpha_prev p_old, p_new, q written at the owned points.
constexpr int kMvThreads = 256;
constexpr int kMvH = kTile + 2;

__global__ void __launch_bounds__(kMvThreads)
k_pcg2_matvec_tile(StencilOp A, const unsigned char* __restrict__ mask, const double* __restrict__ z,
                   const double* __restrict__ p_old, double* __restrict__ p_new, double* __restrict__ q,
                   double* __restrict__ w, Scal* S, RedScratch R) {
    __shared__ double P[kMvH][kMvH + 1];
    if (*(volatile int*)&S->cg_done) return;
    const double beta = S->cg_beta;
    const double alpha_prev = S->cg_alpha;                // alpha of the previous iteration (0 at the first)
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int ntx = (A.nx + kTile - 1) / kTile, nty = (A.ny + kTile - 1) / kTile;
    double acc[1] = {0.0};
    for (int t = blockIdx.x; t < ntx * nty; t += gridDim.x) {
        const int x0 = (t % ntx) * kTile, y0 = (t / ntx) * kTile;
        for (int e = threadIdx.x; e < kMvH * kMvH; e += kMvThreads) {
            const int ry = e / kMvH, rx = e - ry * kMvH;
            const int i = x0 - 1 + rx, j = y0 - 1 + ry;
            double pv = 0.0;
            if (i >= 0 && i < A.nx && j >= A.rlo && j < A.rhi) {
                const long long v = i + (long long)A.pitch * j;
                pv = fma(beta, p_old[v], z[v]);
            }
            P[ry][rx] = pv;
        }
        __syncthreads();
        const int i = x0 + tx;
#pragma unroll
        for (int m = 0; m < kTile / 8; ++m) {
            const int jl = ty + 8 * m, j = y0 + jl;
            if (i < A.nx && j < A.ny) {
                const long long v = i + (long long)A.pitch * j;
                const double pc = P[jl + 1][tx + 1];
                if (mask[v]) {
                    const double* wxr = A.wx + (long long)j * A.wx_ld + i;
                    const double fw = __ldg(wxr), fe = __ldg(wxr + 1);
                    const double fs = __ldg(A.wy + (long long)j * A.wy_ld + i);
                    const double fn = __ldg(A.wy + (long long)(j + 1) * A.wy_ld + i);
                    double d = (fw + fe) + (fs + fn);
                    if (A.shift) d += __ldg(A.shift + v);
                    double qv = d * pc;
                    qv = fma(-fw, P[jl + 1][tx], qv);
                    qv = fma(-fe, P[jl + 1][tx + 2], qv);
                    qv = fma(-fs, P[jl][tx + 1], qv);
                    qv = fma(-fn, P[jl + 2][tx + 1], qv);
                    w[v] = fma(alpha_prev, p_old[v], w[v]);
                    p_new[v] = pc;
                    q[v] = qv;
                    acc[0] = fma(pc, qv, acc[0]);
                } else {
                    p_new[v] = 0.0;
                    q[v] = 0.0;
                }
            }
        }
        __syncthreads();
    }
    reduce_and_finish<1>(acc, R, [&](double* tt) { pcg2_alpha_fin(tt[0], S); });
}

// after the last iteration j: w += alpha_j p_j (p is 0 off F)
__global__ void __launch_bounds__(kThreads)
k_pcg2_wlast(StencilOp A, const double* __restrict__ p, double* __restrict__ w, const Scal* S) {
    const double alpha = S->cg_alpha;
    A.for_each_point([&](const Pt& pt) { w[pt.v] = fma(alpha, p[pt.v], w[pt.v]); });
}

}  // namespace gpcg
