// march.cuh -- stencil-specialised sweeps for the 5-point operator (SURVEY.md
// 8(a) a1-a5, "stencil2d" variants).
//
// Execution model ("column march"): a warp owns a strip of 32 consecutive grid
// columns and marches down a chunk of TY rows.  Values needed at the four
// neighbours of a point come from registers: west/east by warp shuffle, south/
// north from a sliding window of rows.  Every input is read from HBM once per
// sweep (plus a few warm-up rows per chunk); all loads are coalesced 256-byte
// row segments; derived values (trial points, projected gradients, CG
// vectors) are computed once per point instead of once per neighbour.  A
// kernel that applies the operator L times in sequence (e.g. the CG iteration
// forms p, then rho - alpha A p, then A rho) keeps H = L halo lanes per side:
// outputs are written by lanes [H, 32-H).
//
// Latency hiding: raw rows are software-pipelined through a register ring of
// depth kPipe (loads for row r + kPipe are issued while row r is consumed);
// where a load is predicated on the free mask, masks run a further kPipe rows
// ahead so no load waits on another.
//
// Reductions go through reduce_and_finish (common.cuh): fixed-order, so every
// result is bitwise reproducible for a fixed grid.
#pragma once

#include "common.cuh"
#include "fin.cuh"

namespace gpcg {

constexpr int kPipe = 4;            // rows in flight per warp
constexpr int kMarchMinBlocks = 4;  // >= 16 resident warps per SM (<= 128 registers)

struct MarchGeom {
    int nstrips;   // ceil(nx / (32 - 2H))
    int nchunks;   // ceil(ny / TY)
    int TY;        // output rows per work item
};

// ---------------------------------------------------------------------------
// Per-lane 5-point operator.  BC = broadcast face weights and no diagonal
// shift (the journal-bearing configs C0/C2/C3): weights live in registers for
// the whole strip and the two y-faces of a point are equal.  Otherwise faces
// (and shift) are loaded per row, at a clamped in-grid address -- results at
// out-of-grid rows/columns are always discarded or multiplied by a zero mask,
// so they only need to be finite.
// Out-of-grid raw inputs are loaded as 0; every derived value (trial step,
// projected gradient, CG vector) is then exactly 0 there as the Dirichlet
// boundary requires (mid(0,0,0) = 0, pgrad of a fixed variable = 0, masks 0).
// ---------------------------------------------------------------------------
template <bool BC>
struct Op5 {
    double fw, fe, fs, fn, dg;     // BC: strip-constant faces and diagonal
    int ic;                        // clamped column
    __device__ __forceinline__ void init(const StencilOp& A, int i) {
        ic = min(max(i, 0), A.nx - 1);
        if constexpr (BC) {
            fw = __ldg(A.wx + ic);
            fe = __ldg(A.wx + ic + 1);
            fs = __ldg(A.wy + ic);
            fn = fs;
            dg = (fw + fe) + (fs + fn);
        }
    }
    // 1 / A_vv at row r of this lane (point-Jacobi preconditioner); BC: per column
    __device__ __forceinline__ double dinv(const StencilOp& A, int r) const {
        if constexpr (BC) {
            return 1.0 / dg;
        } else {
            const int rc = min(max(r, A.rlo), A.rhi - 1);
            const double* wxr = A.wx + (long long)rc * A.wx_ld + ic;
            double d = (__ldg(wxr) + __ldg(wxr + 1)) +
                       (__ldg(A.wy + (long long)rc * A.wy_ld + ic) + __ldg(A.wy + (long long)(rc + 1) * A.wy_ld + ic));
            if (A.shift) d += __ldg(A.shift + ic + A.pitch * rc);
            return 1.0 / d;
        }
    }
    // (A v) at row r of this lane: vc centre, vs / vn rows r-1 / r+1, west/east by shuffle
    __device__ __forceinline__ double apply(const StencilOp& A, int r, double vc, double vs, double vn) const {
        const double vw = __shfl_up_sync(0xffffffffu, vc, 1);
        const double ve = __shfl_down_sync(0xffffffffu, vc, 1);
        if constexpr (BC) {
            double t = dg * vc;
            t = fma(-fw, vw, t);
            t = fma(-fe, ve, t);
            return fma(-fs, vs + vn, t);
        } else {
            const int rc = min(max(r, A.rlo), A.rhi - 1);
            const double* wxr = A.wx + (long long)rc * A.wx_ld + ic;
            const double w = __ldg(wxr), e = __ldg(wxr + 1);
            const double s = __ldg(A.wy + (long long)rc * A.wy_ld + ic);
            const double n = __ldg(A.wy + (long long)(rc + 1) * A.wy_ld + ic);
            double d = (w + e) + (s + n);
            if (A.shift) d += __ldg(A.shift + ic + A.pitch * rc);
            double t = d * vc;
            t = fma(-w, vw, t);
            t = fma(-e, ve, t);
            t = fma(-s, vs, t);
            return fma(-n, vn, t);
        }
    }
};

// One work item per warp: strip column of this lane and output row range.
template <int H>
__device__ __forceinline__ bool march_item(const StencilOp& A, const MarchGeom& G, int& i, int& j0, int& j1) {
    const int item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (item >= G.nstrips * G.nchunks) return false;
    const int s = item % G.nstrips, c = item / G.nstrips;
    i = s * (32 - 2 * H) - H + (threadIdx.x & 31);
    j0 = c * G.TY;
    j1 = min(j0 + G.TY, A.ny);
    return true;
}

struct NoPre {};

// Software pipeline over rows r0 .. r0+nsteps-1 (nsteps rounded up to kPipe):
// ring[k] holds raw(r) loaded kPipe steps earlier; pre(r) (e.g. the mask) runs
// 2*kPipe rows ahead so that load(r, pre(r)) never waits on pre.
template <class Pre, class Raw, class PreF, class LoadF, class StepF>
__device__ __forceinline__ void pipeline(int r0, int nsteps, PreF&& pre, LoadF&& load, StepF&& step) {
    Raw ring[kPipe];
    Pre pring[kPipe];
#pragma unroll
    for (int k = 0; k < kPipe; ++k) {
        ring[k] = load(r0 + k, pre(r0 + k));
        pring[k] = pre(r0 + kPipe + k);
    }
    for (int s0 = 0; s0 < nsteps; s0 += kPipe) {
#pragma unroll
        for (int k = 0; k < kPipe; ++k) {
            const int r = r0 + s0 + k;
            const Raw cur = ring[k];
            ring[k] = load(r + kPipe, pring[k]);
            pring[k] = pre(r + 2 * kPipe);
            step(r, cur);
        }
    }
}

// ============================================================================
// a1 + a2 fused: accept / project, regrad, free mask, set counts, and the
// Cauchy quadratic form of the NEW point (so the next GP step's alpha_0 is
// ready without another sweep).  H = 2.
//   level 1  yn(r)   = mid(l, u, y(r) + alpha sgn dir(r))   (or mid(l,u,y) if !dir)
//   level 2  gn(r-1) = (A yn)(r-1) - b,  d(r-1) = grad_Omega q(yn)(r-1)  (Eq. proj-gradient)
//   level 3  Ad(r-2) = (A d)(r-2);  emit row r-2
// sums: ||d||^2 (= ||grad_Omega q||^2), ||gn||^2, |A|, #changed, |A\B|, <d, A d>
// finaliser: alpha_0 = ||d||^2 / <d, A d> (Eq. bqpls) for the next GP step.
// ============================================================================
struct RawAcc {
    double y, d, b, l, u;
    unsigned char mp;
};

template <bool SB, bool BC>
__global__ void __launch_bounds__(kMarchThreads, kMarchMinBlocks)
k2_accept(StencilOp A, MarchGeom G, Bounds Bd, const double* __restrict__ y_in, const double* __restrict__ dir,
          double sgn, const double* __restrict__ b, const unsigned char* __restrict__ mask_prev,
          double* __restrict__ y_out, double* __restrict__ g_out, unsigned char* __restrict__ mask_out,
          Scal* S, RedScratch R, int gp) {
    if (gp && *(volatile int*)&S->gp_done) return;   // device-driven GP phase already over
    double alpha = 0.0;
    if (dir) {
        if (S->s_h < 0) return;                   // uniform: no accepted step in this batch
        alpha = S->s_alpha;
    }
    constexpr int H = 2;
    const int lane = threadIdx.x & 31;
    const bool out_lane = lane >= H && lane < 32 - H;
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int i, j0, j1;
    if (march_item<H>(A, G, i, j0, j1)) {
        const bool col_ok = (i >= 0 && i < A.nx);
        Op5<BC> op;
        op.init(A, i);
        const int rend = min(A.rhi, j1 + H);            // raw rows [j0-H, rend) are needed
        double yn_m2 = 0.0, yn_m1 = 0.0;               // yn(r-2), yn(r-1)
        double b_m1 = 0.0, l_m1 = 0.0, u_m1 = 0.0;      // row r-1
        double l_m2 = 0.0, u_m2 = 0.0;                  // row r-2
        unsigned char mp_m1 = 0, mp_m2 = 0;
        double gn_m2 = 0.0;                             // gn(r-2)
        double d_m3 = 0.0, d_m2 = 0.0;                  // d(r-3), d(r-2)
        pipeline<NoPre, RawAcc>(
            j0 - 2, j1 - j0 + 4, [&](int) { return NoPre{}; },
            [&](int r, NoPre) {                          // loads only; consumed kPipe rows later
                RawAcc x{0.0, 0.0, 0.0, SB ? Bd.lc : 0.0, SB ? Bd.uc : 0.0, 0};
                if (r >= A.rlo && r < rend) {                // warp-uniform
                    if (col_ok) {
                        const int v = i + A.pitch * r;
                        if constexpr (!SB) { x.l = __ldg(Bd.l + v); x.u = __ldg(Bd.u + v); }
                        x.b = __ldg(b + v);
                        x.y = __ldg(y_in + v);
                        if (dir) x.d = __ldg(dir + v);
                        if (mask_prev) x.mp = __ldg(mask_prev + v);
                    }
                }
                if (!(col_ok && r >= A.rlo && r < rend)) { x.l = 0.0; x.u = 0.0; }   // fixed at 0 outside
                return x;
            },
            [&](int r, const RawAcc& x) {
                const double yn0 = dir ? trial(x.y, x.d, sgn, alpha, x.l, x.u) : mid(x.l, x.u, x.y);
                // level 2 at row r-1
                const double ay = op.apply(A, r - 1, yn_m1, yn_m2, yn0);
                const double gn1 = ay - b_m1;
                const double d1 = pgrad(yn_m1, gn1, l_m1, u_m1);      // 0 outside the grid
                // level 3 at row r-2
                const double ad = op.apply(A, r - 2, d_m2, d_m3, d1);
                const int r2 = r - 2;
                if (out_lane && col_ok && r2 >= j0 && r2 < j1) {
                    const int v = i + A.pitch * r2;
                    y_out[v] = yn_m2;
                    g_out[v] = gn_m2;
                    const bool act = (yn_m2 == l_m2) || (yn_m2 == u_m2);
                    const unsigned char m = act ? 0 : 1;
                    mask_out[v] = m;
                    acc[0] = fma(d_m2, d_m2, acc[0]);
                    acc[1] = fma(gn_m2, gn_m2, acc[1]);
                    acc[2] += act ? 1.0 : 0.0;
                    if (mask_prev) acc[3] += (mp_m2 != m) ? 1.0 : 0.0;
                    const bool binding = (yn_m2 == l_m2 && gn_m2 >= 0.0) || (yn_m2 == u_m2 && gn_m2 <= 0.0);
                    acc[4] += (act && !binding) ? 1.0 : 0.0;
                    acc[5] = fma(d_m2, ad, acc[5]);
                }
                yn_m2 = yn_m1; yn_m1 = yn0;
                l_m2 = l_m1; u_m2 = u_m1; mp_m2 = mp_m1;
                l_m1 = x.l; u_m1 = x.u; b_m1 = x.b; mp_m1 = x.mp;
                gn_m2 = gn1;
                d_m3 = d_m2; d_m2 = d1;
            });
    }
    reduce_and_finish<6>(acc, R, [&](double* t) { fin_accept(t, true, S); });
}

// ============================================================================
// a3: projected search, K step sizes per sweep.  H = 1.
//   level 1  s_h(r) = mid(l, u, y + alpha_h sgn dir) - y
//   level 2  sums <g, s_h>(r-1), <s_h, A s_h>(r-1)
// kDirIsG: the GP direction is -g, so dir and g are the same array (one load).
// ============================================================================
struct RawY {
    double y, d, g, l, u;
};

template <bool SB, bool BC, int K, bool kDirIsG>
__global__ void __launch_bounds__(kMarchThreads, (K <= 4 ? kMarchMinBlocks : 2))
k2_search(StencilOp A, MarchGeom G, Bounds Bd, const double* __restrict__ y, const double* __restrict__ g,
          const double* __restrict__ dir, double sgn, int use_alpha0, int h0, double mu, Scal* S,
          RedScratch R, int gp) {
    if (gp && *(volatile int*)&S->gp_done) return;   // device-driven GP phase already over
    if (use_alpha0 && !S->cauchy_ok) {           // <d,Ad> <= 0: no step (host reports ENOTSPD)
        if (blockIdx.x == 0 && threadIdx.x == 0) S->s_h = -1;
        return;
    }
    const double base = use_alpha0 ? S->alpha0 : 1.0;
    double al[K];
#pragma unroll
    for (int h = 0; h < K; ++h) al[h] = scalbn(base, -(h0 + h));
    constexpr int H = 1;
    const int lane = threadIdx.x & 31;
    const bool out_lane = lane >= H && lane < 32 - H;
    double acc[2 * K];
#pragma unroll
    for (int s = 0; s < 2 * K; ++s) acc[s] = 0.0;
    int i, j0, j1;
    if (march_item<H>(A, G, i, j0, j1)) {
        const bool col_ok = (i >= 0 && i < A.nx);
        Op5<BC> op;
        op.init(A, i);
        const int rend = min(A.rhi, j1 + H);
        double s_m2[K], s_m1[K];
        double g_m1 = 0.0;
#pragma unroll
        for (int h = 0; h < K; ++h) { s_m2[h] = 0.0; s_m1[h] = 0.0; }
        pipeline<NoPre, RawY>(
            j0 - 1, j1 - j0 + 2, [&](int) { return NoPre{}; },
            [&](int r, NoPre) {
                RawY x{0.0, 0.0, 0.0, SB ? Bd.lc : 0.0, SB ? Bd.uc : 0.0};
                if (r >= A.rlo && r < rend) {
                    if (col_ok) {
                        const int v = i + A.pitch * r;
                        x.y = __ldg(y + v);
                        x.d = __ldg(dir + v);
                        if constexpr (!kDirIsG) x.g = __ldg(g + v);
                        if constexpr (!SB) { x.l = __ldg(Bd.l + v); x.u = __ldg(Bd.u + v); }
                    }
                }
                if constexpr (kDirIsG) x.g = x.d;
                if (!(col_ok && r >= A.rlo && r < rend)) { x.l = 0.0; x.u = 0.0; }
                return x;
            },
            [&](int r, const RawY& x) {
                double s0[K];
#pragma unroll
                for (int h = 0; h < K; ++h) s0[h] = trial(x.y, x.d, sgn, al[h], x.l, x.u) - x.y;   // 0 outside
                const int r1 = r - 1;
                const bool emit = out_lane && col_ok && r1 >= j0 && r1 < j1;
#pragma unroll
                for (int h = 0; h < K; ++h) {
                    const double as = op.apply(A, r1, s_m1[h], s_m2[h], s0[h]);
                    if (emit) {
                        acc[2 * h] = fma(g_m1, s_m1[h], acc[2 * h]);
                        acc[2 * h + 1] = fma(s_m1[h], as, acc[2 * h + 1]);
                    }
                }
#pragma unroll
                for (int h = 0; h < K; ++h) { s_m2[h] = s_m1[h]; s_m1[h] = s0[h]; }
                g_m1 = x.g;
            });
    }
    reduce_and_finish<2 * K>(acc, R, [&](double* t) { fin_search(t, K, h0, base, mu, S); });
}

// ============================================================================
// a5 init: rho_0 = -[v in F] g_v, p_{-1} = 0, w_0 = 0; gamma_0 = rho_0'rho_0,
// delta_0 = rho_0'A_F rho_0.  Also copies the free mask into the fixed CG mask
// buffer used by the captured CG graph.  H = 1.
// ============================================================================
struct RawInit {
    double rho;
    unsigned char m;
};

// PC: point-Jacobi PCG (u = rho / A_vv): gamma_0 = rho_0'u_0, delta_0 = u_0'A_F u_0.
template <bool BC, bool PC>
__global__ void __launch_bounds__(kMarchThreads, kMarchMinBlocks)
k2_cg_init(StencilOp A, MarchGeom G, const double* __restrict__ g, const unsigned char* __restrict__ mask,
           unsigned char* __restrict__ mask_cg, double* __restrict__ rho, double* __restrict__ p,
           double* __restrict__ w, double eta2, long long cap, Scal* S, RedScratch R) {
    constexpr int H = 1;
    const int lane = threadIdx.x & 31;
    const bool out_lane = lane >= H && lane < 32 - H;
    double acc[2] = {0.0, 0.0};
    int i, j0, j1;
    if (march_item<H>(A, G, i, j0, j1)) {
        const bool col_ok = (i >= 0 && i < A.nx);
        Op5<BC> op;
        op.init(A, i);
        const int rend = min(A.rhi, j1 + H);
        double r_m2 = 0.0, r_m1 = 0.0, rho_m1 = 0.0;   // u (= rho without PC) at r-2, r-1; rho at r-1
        unsigned char m_m1 = 0;
        pipeline<NoPre, RawInit>(
            j0 - 1, j1 - j0 + 2, [&](int) { return NoPre{}; },
            [&](int r, NoPre) {
                RawInit x{0.0, 0};
                if (r >= A.rlo && r < rend) {
                    if (col_ok) {
                        const int v = i + A.pitch * r;
                        x.m = __ldg(mask + v);
                        x.rho = -__ldg(g + v);
                    }
                }
                return x;
            },
            [&](int r, const RawInit& x) {
                const double rho0 = x.m ? x.rho : 0.0;
                const double r0 = PC ? rho0 * op.dinv(A, r) : rho0;
                const int r1 = r - 1;
                const double q = op.apply(A, r1, r_m1, r_m2, r0);
                if (out_lane && col_ok && r1 >= j0 && r1 < j1) {
                    const int v = i + A.pitch * r1;
                    mask_cg[v] = m_m1;
                    rho[v] = rho_m1;
                    p[v] = 0.0;
                    w[v] = 0.0;
                    acc[0] = fma(rho_m1, r_m1, acc[0]);        // 0 off F
                    acc[1] = m_m1 ? fma(r_m1, q, acc[1]) : acc[1];
                }
                r_m2 = r_m1; r_m1 = r0; rho_m1 = rho0; m_m1 = x.m;
            });
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_init_finalize(t[0], t[1], eta2, cap, S); });
}

// ============================================================================
// a5 iteration, stencil form that stores only rho, p, w (49 B per free point
// instead of 81): the products s = A_F p and q = A_F rho are recomputed from
// neighbours instead of being carried as vectors.  H = 2.
//   level 1  pn(r)   = [r in F] (rho(r) + beta p(r))                       p_i
//   level 2  rn(r-1) = [r-1 in F] (rho(r-1) - alpha (A pn)(r-1))          rho_{i+1}
//   level 3  q(r-2)  = [r-2 in F] (A rn)(r-2)                              A_F rho_{i+1}
//   emit r-2: w += alpha pn; rho' = rn; p' = pn; gamma += rn^2; delta += rn q
// Loads of rho, p, w are predicated on the mask (active regions cost 1 B/pt),
// with masks pipelined kPipe rows ahead of the data.
// ============================================================================
struct RawCg {
    double rho, p, w;
    unsigned char m;
};

// PC: point-Jacobi PCG -- level 1 uses u = rho / A_vv, level 3 applies A to un = rn / A_vv and
// accumulates gamma = rn'un, delta = un'A un (reading R19: Chronopoulos-Gear PCG).
template <bool BC, bool PC>
__global__ void __launch_bounds__(kMarchThreads, kMarchMinBlocks)
k2_cg_iter(StencilOp A, MarchGeom G, const unsigned char* __restrict__ mask,
           const double* __restrict__ rho, const double* __restrict__ p,
           double* __restrict__ rho_n, double* __restrict__ p_n, double* __restrict__ w,
           Scal* S, RedScratch R) {
    if (*(volatile int*)&S->cg_done) return;
    const double alpha = S->cg_alpha, beta = S->cg_beta;
    constexpr int H = 2;
    const int lane = threadIdx.x & 31;
    const bool out_lane = lane >= H && lane < 32 - H;
    double acc[2] = {0.0, 0.0};
    int i, j0, j1;
    if (march_item<H>(A, G, i, j0, j1)) {
        const bool col_ok = (i >= 0 && i < A.nx);
        Op5<BC> op;
        op.init(A, i);
        const int rend = min(A.rhi, j1 + H);
        double pn_m2 = 0.0, pn_m1 = 0.0;          // pn(r-2), pn(r-1)
        double rho_m1 = 0.0;                       // rho(r-1)
        double w_m1 = 0.0, w_m2 = 0.0;             // w(r-1), w(r-2)
        unsigned char m_m1 = 0, m_m2 = 0;
        double rn_m3 = 0.0, rn_m2 = 0.0;           // rn(r-3), rn(r-2)   (PC: un)
        double rr_m2 = 0.0;                        // PC: rn(r-2)
        pipeline<unsigned char, RawCg>(
            j0 - 2, j1 - j0 + 4,
            [&](int r) -> unsigned char {
                unsigned char m = 0;
                if (r >= A.rlo && r < rend) {
                    if (col_ok) m = __ldg(mask + i + A.pitch * r);
                }
                return m;
            },
            [&](int r, unsigned char m) {
                RawCg x{0.0, 0.0, 0.0, m};
                if (m) {
                    const int v = i + A.pitch * r;
                    x.rho = rho[v];
                    x.p = p[v];
                    if (out_lane) x.w = w[v];       // w is only needed where this warp writes
                }
                return x;
            },
            [&](int r, const RawCg& x) {
                const double u0 = PC ? x.rho * op.dinv(A, r) : x.rho;
                const double pn0 = x.m ? fma(beta, x.p, u0) : 0.0;
                // level 2 at row r-1
                const double ap = op.apply(A, r - 1, pn_m1, pn_m2, pn0);
                const double rr1 = m_m1 ? fma(-alpha, ap, rho_m1) : 0.0;
                const double rn1 = PC ? rr1 * op.dinv(A, r - 1) : rr1;
                // level 3 at row r-2
                const double q = op.apply(A, r - 2, rn_m2, rn_m3, rn1);
                const int r2 = r - 2;
                const double rres = PC ? rr_m2 : rn_m2;
                if (out_lane && m_m2 && r2 >= j0 && r2 < j1) {   // m_m2 = 0 outside the grid
                    const int v = i + A.pitch * r2;
                    w[v] = fma(alpha, pn_m2, w_m2);
                    rho_n[v] = rres;
                    p_n[v] = pn_m2;
                    acc[0] = fma(rres, rn_m2, acc[0]);
                    acc[1] = fma(rn_m2, q, acc[1]);
                }
                pn_m2 = pn_m1; pn_m1 = pn0;
                rho_m1 = x.rho;
                w_m2 = w_m1; w_m1 = x.w;
                m_m2 = m_m1; m_m1 = x.m;
                rn_m3 = rn_m2; rn_m2 = rn1;
                rr_m2 = rr1;
            });
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_finalize(t[0], t[1], S); });
}

}  // namespace gpcg
