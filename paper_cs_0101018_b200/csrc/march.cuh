// march.cuh -- stencil-specialised sweeps for the 5-point operator (SURVEY.md
// 8(a) a1-a5, "stencil2d" variants).
//
// Execution model ("column march"): a warp owns a strip of 32 consecutive grid
// columns and marches down a chunk of TY rows.  Values needed at the four
// neighbours of a point come from registers: west/east by warp shuffle, south/
// north from a sliding window of rows.  Every input is therefore read from
// HBM once per sweep (plus a few warm-up rows per chunk), all loads are
// coalesced 256-byte rows, and derived values (trial points, projected
// gradients, CG vectors) are computed once per point instead of once per
// neighbour.  A kernel that applies the operator L times in sequence
// (e.g. the CG iteration forms p, then rho = rho - alpha A p, then A rho) keeps
// H = L halo lanes per side: outputs are written by lanes [H, 32-H).
//
// Reductions go through reduce_and_finish (common.cuh): fixed-order, so every
// result is bitwise reproducible for a fixed grid.
#pragma once

#include "common.cuh"

namespace gpcg {

struct MarchGeom {
    int nstrips;   // ceil(nx / (32 - 2H))
    int nchunks;   // ceil(ny / TY)
    int TY;        // output rows per work item
};

// Per-lane face weights of column i at grid row j (zero outside the grid).
struct Faces {
    double w, e, s, n;
};

__device__ __forceinline__ Faces load_faces(const StencilOp& A, int i, int j, bool col_ok) {
    Faces f{0.0, 0.0, 0.0, 0.0};
    if (col_ok && j >= 0 && j < A.ny) {
        const double* wxr = A.wx + (long long)j * A.wx_ld;
        f.w = __ldg(wxr + i);
        f.e = __ldg(wxr + i + 1);
        f.s = __ldg(A.wy + (long long)j * A.wy_ld + i);
        f.n = __ldg(A.wy + (long long)(j + 1) * A.wy_ld + i);
    }
    return f;
}

// (A v) at this lane's point: vc centre, vs/vn rows below/above, west/east by shuffle.
__device__ __forceinline__ double apply5(const Faces& f, double shift, double vc, double vs, double vn) {
    const double vw = __shfl_up_sync(0xffffffffu, vc, 1);
    const double ve = __shfl_down_sync(0xffffffffu, vc, 1);
    const double d = (f.w + f.e) + (f.s + f.n) + shift;
    double r = d * vc;
    r = fma(-f.w, vw, r);
    r = fma(-f.e, ve, r);
    r = fma(-f.s, vs, r);
    r = fma(-f.n, vn, r);
    return r;
}

// Work item -> strip column of this lane and row range.
template <int H>
__device__ __forceinline__ void march_item(const StencilOp& A, const MarchGeom& G, int item, int& i, int& j0,
                                           int& j1) {
    const int s = item % G.nstrips, c = item / G.nstrips;
    i = s * (32 - 2 * H) - H + (threadIdx.x & 31);
    j0 = c * G.TY;
    j1 = min(j0 + G.TY, A.ny);
}

__device__ __forceinline__ int warp_global() { return (blockIdx.x * blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ int warps_total() { return (gridDim.x * blockDim.x) >> 5; }

// Faces cache: broadcast weights are loaded once per strip; full arrays per row.
struct FaceRow {
    bool bcast;
    Faces fb;
    __device__ __forceinline__ void init(const StencilOp& A, int i, bool col_ok) {
        bcast = (A.wx_ld == 0 && A.wy_ld == 0);
        if (bcast) fb = load_faces(A, i, 0, col_ok);
    }
    __device__ __forceinline__ Faces at(const StencilOp& A, int i, int j, bool col_ok) const {
        if (bcast) return (col_ok && j >= 0 && j < A.ny) ? fb : Faces{0.0, 0.0, 0.0, 0.0};
        return load_faces(A, i, j, col_ok);
    }
};

__device__ __forceinline__ double shift_at(const StencilOp& A, int v, bool ok) {
    return (A.shift && ok) ? __ldg(A.shift + v) : 0.0;
}

// ============================================================================
// a1 + a2 fused: accept / project, regrad, free mask, set counts, and the
// Cauchy quadratic form of the NEW point (so the next GP step's alpha_0 is
// ready without another sweep).  H = 2.
//   level 1  yn(r) = mid(l, u, y(r) + alpha sgn dir(r))   (or mid(l,u,y) if !dir)
//   level 2  gn(r) = (A yn)(r) - b(r),  d(r) = grad_Omega q(yn)(r)   (Eq. proj-gradient)
//   level 3  Ad(j) = (A d)(j)
// sums: ||d||^2 (= ||grad_Omega q||^2), ||gn||^2, |A|, #changed, |A\B|, <d, A d>
// finaliser: alpha_0 = ||d||^2 / <d, A d> (Eq. bqpls) for the next GP step.
// ============================================================================
template <bool SB>
__global__ void __launch_bounds__(kThreads)
k2_accept(StencilOp A, MarchGeom G, Bounds Bd, const double* __restrict__ y_in, const double* __restrict__ dir,
          double sgn, const double* __restrict__ b, const unsigned char* __restrict__ mask_prev,
          double* __restrict__ y_out, double* __restrict__ g_out, unsigned char* __restrict__ mask_out,
          Scal* S, RedScratch R) {
    double alpha = 0.0;
    if (dir) {
        if (S->s_h < 0) return;                   // uniform: no accepted step in this batch
        alpha = S->s_alpha;
    }
    constexpr int H = 2;
    const int lane = threadIdx.x & 31;
    const bool out_lane = lane >= H && lane < 32 - H;
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const int nitems = G.nstrips * G.nchunks;
    for (int item = warp_global(); item < nitems; item += warps_total()) {
        int i, j0, j1;
        march_item<H>(A, G, item, i, j0, j1);
        const bool col_ok = (i >= 0 && i < A.nx);
        FaceRow FR;
        FR.init(A, i, col_ok);
        // raw row loader: y_in, dir -> yn ; b, l, u kept for levels 2/emit
        auto yn_at = [&](int r, double& l_r, double& u_r, double& b_r) -> double {
            l_r = 0.0; u_r = 0.0; b_r = 0.0;
            if (!col_ok || r < 0 || r >= A.ny) return 0.0;
            const int v = i + A.nx * r;
            l_r = lo<SB>(Bd, v);
            u_r = hi<SB>(Bd, v);
            b_r = __ldg(b + v);
            const double yv = __ldg(y_in + v);
            return dir ? trial(yv, __ldg(dir + v), sgn, alpha, l_r, u_r) : mid(l_r, u_r, yv);
        };
        // windows
        double yn0 = 0.0, yn1 = 0.0;              // yn(j), yn(j+1)
        double l1 = 0.0, u1 = 0.0, b1 = 0.0;      // bounds/b of row j+1
        double l0 = 0.0, u0 = 0.0;                // bounds of row j
        double gn0 = 0.0;                          // gn(j)
        double dm = 0.0, d0 = 0.0;                 // d(j-1), d(j)
        // start 2 rows early to fill the windows (outputs begin at j0)
        int j = j0 - 2;
        {
            double lx, ux, bx;
            yn0 = yn_at(j, lx, ux, bx);
            (void)lx; (void)ux; (void)bx;
            yn1 = yn_at(j + 1, l1, u1, b1);
        }
        for (; j < j1; ++j) {
            double l2, u2, b2;
            const double yn2 = yn_at(j + 2, l2, u2, b2);
            // level 2 at row j+1
            const Faces f1 = FR.at(A, i, j + 1, col_ok);
            const bool ok1 = col_ok && (j + 1) >= 0 && (j + 1) < A.ny;
            const double sh1 = shift_at(A, i + A.nx * (j + 1), ok1);
            const double ay1 = apply5(f1, sh1, yn1, yn0, yn2);
            const double gn1 = ok1 ? ay1 - b1 : 0.0;
            const double d1 = ok1 ? pgrad(yn1, gn1, l1, u1) : 0.0;
            // level 3 at row j
            const Faces f0 = FR.at(A, i, j, col_ok);
            const bool ok0 = col_ok && j >= 0 && j < A.ny;
            const double sh0 = shift_at(A, i + A.nx * j, ok0);
            const double ad0 = apply5(f0, sh0, d0, dm, d1);
            if (out_lane && ok0 && j >= j0) {
                const int v = i + A.nx * j;
                y_out[v] = yn0;
                g_out[v] = gn0;
                const bool act = (yn0 == l0) || (yn0 == u0);
                const unsigned char m = act ? 0 : 1;
                mask_out[v] = m;
                acc[0] = fma(d0, d0, acc[0]);
                acc[1] = fma(gn0, gn0, acc[1]);
                acc[2] += act ? 1.0 : 0.0;
                if (mask_prev) acc[3] += (mask_prev[v] != m) ? 1.0 : 0.0;
                const bool binding = (yn0 == l0 && gn0 >= 0.0) || (yn0 == u0 && gn0 <= 0.0);
                acc[4] += (act && !binding) ? 1.0 : 0.0;
                acc[5] = fma(d0, ad0, acc[5]);
            }
            // shift windows
            yn0 = yn1; yn1 = yn2;
            l0 = l1; u0 = u1;
            l1 = l2; u1 = u2; b1 = b2;
            gn0 = gn1;
            dm = d0; d0 = d1;
        }
    }
    reduce_and_finish<6>(acc, R, [&](double* t) {
        S->pg2 = t[0];
        S->g2 = t[1];
        S->n_active = t[2];
        S->n_changed = t[3];
        S->n_nonbinding = t[4];
        S->dd = t[0];
        S->dAd = t[5];
        S->cauchy_ok = (t[5] > 0.0) ? 1 : 0;
        S->alpha0 = (t[5] > 0.0) ? t[0] / t[5] : 0.0;
    });
}

// ============================================================================
// a3: projected search, K step sizes per sweep.  H = 1.
//   level 1  s_h(r) = mid(l, u, y + alpha_h sgn dir) - y
//   level 2  sums <g, s_h>(j), <s_h, A s_h>(j)
// kDirIsG: the GP direction is -g, so dir and g are the same array (one load).
// ============================================================================
template <bool SB, int K, bool kDirIsG>
__global__ void __launch_bounds__(kThreads)
k2_search(StencilOp A, MarchGeom G, Bounds Bd, const double* __restrict__ y, const double* __restrict__ g,
          const double* __restrict__ dir, double sgn, int use_alpha0, int h0, double mu, Scal* S,
          RedScratch R) {
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
    const int nitems = G.nstrips * G.nchunks;
    for (int item = warp_global(); item < nitems; item += warps_total()) {
        int i, j0, j1;
        march_item<H>(A, G, item, i, j0, j1);
        const bool col_ok = (i >= 0 && i < A.nx);
        FaceRow FR;
        FR.init(A, i, col_ok);
        auto load_s = [&](int r, double (&s)[K], double& gr) {
            gr = 0.0;
#pragma unroll
            for (int h = 0; h < K; ++h) s[h] = 0.0;
            if (!col_ok || r < 0 || r >= A.ny) return;
            const int v = i + A.nx * r;
            const double yv = __ldg(y + v);
            const double dv = __ldg(dir + v);
            gr = kDirIsG ? dv : __ldg(g + v);
            const double l = lo<SB>(Bd, v), u = hi<SB>(Bd, v);
#pragma unroll
            for (int h = 0; h < K; ++h) s[h] = trial(yv, dv, sgn, al[h], l, u) - yv;
        };
        double sm[K], s0[K], s1[K];
        double g0, g1, gx;
        load_s(j0 - 1, sm, gx);
        load_s(j0, s0, g0);
        int j = j0;
        // loop invariant: sm = s(j-1), s0 = s(j), g0 = g(j)
        for (; j < j1; ++j) {
            load_s(j + 1, s1, g1);
            const Faces f = FR.at(A, i, j, col_ok);
            const bool ok = col_ok && j < A.ny;
            const double sh = shift_at(A, i + A.nx * j, ok);
#pragma unroll
            for (int h = 0; h < K; ++h) {
                const double as = apply5(f, sh, s0[h], sm[h], s1[h]);
                if (out_lane && ok) {
                    acc[2 * h] = fma(g0, s0[h], acc[2 * h]);
                    acc[2 * h + 1] = fma(s0[h], as, acc[2 * h + 1]);
                }
            }
#pragma unroll
            for (int h = 0; h < K; ++h) { sm[h] = s0[h]; s0[h] = s1[h]; }
            g0 = g1;
        }
    }
    reduce_and_finish<2 * K>(acc, R, [&](double* t) {
        S->s_h = -1;
        for (int h = 0; h < K; ++h) {
            const double gs = t[2 * h], sAs = t[2 * h + 1];
            const double dq = gs + 0.5 * sAs;
            if (dq <= mu * gs) {
                S->s_h = h0 + h;
                S->s_alpha = al[h];
                S->s_delta = dq;
                S->s_gs = gs;
                break;
            }
        }
    });
}

// ============================================================================
// a5 init: rho_0 = -[v in F] g_v, p_{-1} = 0, w_0 = 0; gamma_0, delta_0 = rho_0'A_F rho_0.
// Also copies the free mask into the fixed CG mask buffer.  H = 1.
// ============================================================================
__global__ void __launch_bounds__(kThreads)
k2_cg_init(StencilOp A, MarchGeom G, const double* __restrict__ g, const unsigned char* __restrict__ mask,
           unsigned char* __restrict__ mask_cg, double* __restrict__ rho, double* __restrict__ p,
           double* __restrict__ w, double eta2, long long cap, Scal* S, RedScratch R) {
    constexpr int H = 1;
    const int lane = threadIdx.x & 31;
    const bool out_lane = lane >= H && lane < 32 - H;
    double acc[2] = {0.0, 0.0};
    const int nitems = G.nstrips * G.nchunks;
    for (int item = warp_global(); item < nitems; item += warps_total()) {
        int i, j0, j1;
        march_item<H>(A, G, item, i, j0, j1);
        const bool col_ok = (i >= 0 && i < A.nx);
        FaceRow FR;
        FR.init(A, i, col_ok);
        auto rho_at = [&](int r, unsigned char& m) -> double {
            m = 0;
            if (!col_ok || r < 0 || r >= A.ny) return 0.0;
            const int v = i + A.nx * r;
            m = mask[v];
            return m ? -__ldg(g + v) : 0.0;
        };
        unsigned char m0, m1, mx;
        double rm = rho_at(j0 - 1, mx);
        double r0 = rho_at(j0, m0);
        for (int j = j0; j < j1; ++j) {
            const double r1 = rho_at(j + 1, m1);
            const Faces f = FR.at(A, i, j, col_ok);
            const bool ok = col_ok && j < A.ny;
            const double q = apply5(f, shift_at(A, i + A.nx * j, ok), r0, rm, r1);
            if (out_lane && ok) {
                const int v = i + A.nx * j;
                mask_cg[v] = m0;
                rho[v] = r0;
                p[v] = 0.0;
                w[v] = 0.0;
                if (m0) {
                    acc[0] = fma(r0, r0, acc[0]);
                    acc[1] = fma(r0, q, acc[1]);
                }
            }
            rm = r0; r0 = r1; m0 = m1;
        }
    }
    reduce_and_finish<2>(acc, R, [&](double* t) {
        S->cg_it = 0;
        S->cg_cap = cap;
        S->cg_eta2 = eta2;
        S->cg_maxdec = 0.0;
        S->cg_dec = 0.0;
        S->cg_gamma = t[0];
        S->cg_rnorm0 = sqrt(t[0]);
        S->cg_beta = 0.0;
        S->cg_done = 0;
        S->cg_reason = CG_RUNNING;
        if (t[0] == 0.0 || cap <= 0) {
            S->cg_done = 1; S->cg_reason = CG_EXACT; S->cg_alpha = 0.0;
        } else if (!(t[1] > 0.0)) {
            S->cg_done = 1; S->cg_reason = CG_NOTSPD; S->cg_alpha = 0.0;
        } else {
            S->cg_alpha = t[0] / t[1];
        }
    });
}

// ============================================================================
// a5 iteration, stencil form that stores only rho, p, w (49 B per free point
// instead of 81): the products s = A_F p and q = A_F rho are recomputed from
// neighbours instead of being carried as vectors.  H = 2.
//   level 1  pn(r)  = [r in F] (rho(r) + beta p(r))                 p_i
//   level 2  rn(r)  = [r in F] (rho(r) - alpha (A pn)(r))           rho_{i+1}
//   level 3  q(j)   = [j in F] (A rn)(j)                            A_F rho_{i+1}
//   emit     w(j) += alpha pn(j); rho'(j) = rn(j); p'(j) = pn(j); gamma += rn^2; delta += rn q
// Loads of rho, p, w are predicated on the mask (active regions cost 1 B/pt).
// Finaliser identical to the generic k_cg_iter (same recurrences).
// ============================================================================
__device__ __forceinline__ void cg_finalize(double gamma, double delta, Scal* S) {
    const double gamma_old = S->cg_gamma, alpha_old = S->cg_alpha;
    const double dec = 0.5 * alpha_old * gamma_old;
    const long long j = S->cg_it + 1;
    S->cg_it = j;
    S->cg_dec = dec;
    int reason = CG_RUNNING;
    if (j >= 2 && dec <= S->cg_eta2 * S->cg_maxdec) reason = CG_PROGRESS;
    else if (sqrt(gamma) <= 1e-14 * (1.0 + S->cg_rnorm0)) reason = CG_EXACT;
    else if (j >= S->cg_cap) reason = CG_CAP;
    if (dec > S->cg_maxdec) S->cg_maxdec = dec;
    S->cg_gamma = gamma;
    if (reason != CG_RUNNING) {
        S->cg_reason = reason;
        S->cg_done = 1;
        return;
    }
    const double beta = gamma / gamma_old;
    const double pap = delta - beta * gamma / alpha_old;
    S->cg_beta = beta;
    if (!(pap > 0.0)) {
        S->cg_reason = CG_NOTSPD;
        S->cg_done = 1;
        return;
    }
    S->cg_alpha = gamma / pap;
}

__global__ void __launch_bounds__(kThreads)
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
    const int nitems = G.nstrips * G.nchunks;
    for (int item = warp_global(); item < nitems; item += warps_total()) {
        int i, j0, j1;
        march_item<H>(A, G, item, i, j0, j1);
        const bool col_ok = (i >= 0 && i < A.nx);
        FaceRow FR;
        FR.init(A, i, col_ok);
        // raw row: mask, rho, p (w is read at emit only)
        auto raw_at = [&](int r, unsigned char& m, double& rr, double& pp) {
            m = 0; rr = 0.0; pp = 0.0;
            if (!col_ok || r < 0 || r >= A.ny) return;
            const int v = i + A.nx * r;
            m = mask[v];
            if (m) {
                rr = rho[v];
                pp = p[v];
            }
        };
        // windows: pn(j), pn(j+1); rn(j-1), rn(j); raw(j+1) (mask, rho); rows j..j+1 masks
        unsigned char m0 = 0, m1 = 0;
        double rho1 = 0.0, pr1 = 0.0;
        double pn0 = 0.0, pn1 = 0.0;
        double rnm = 0.0, rn0 = 0.0;
        int j = j0 - 2;
        {
            unsigned char mx;
            double rx, px;
            raw_at(j, mx, rx, px);
            pn0 = mx ? fma(beta, px, rx) : 0.0;         // pn(j0-2)
            raw_at(j + 1, m1, rho1, pr1);
            pn1 = m1 ? fma(beta, pr1, rho1) : 0.0;      // pn(j0-1)
            m0 = mx;
        }
        // loop invariant at top: pn0 = pn(j), pn1 = pn(j+1), (m1, rho1) raw of row j+1,
        //                        rnm = rn(j-1), rn0 = rn(j), m0 = mask(j)
        for (; j < j1; ++j) {
            unsigned char m2;
            double rho2, pr2;
            raw_at(j + 2, m2, rho2, pr2);
            const double pn2 = m2 ? fma(beta, pr2, rho2) : 0.0;
            // level 2 at row j+1
            const Faces f1 = FR.at(A, i, j + 1, col_ok);
            const bool ok1 = col_ok && (j + 1) >= 0 && (j + 1) < A.ny;
            const double ap1 = apply5(f1, shift_at(A, i + A.nx * (j + 1), ok1 && m1), pn1, pn0, pn2);
            const double rn1 = m1 ? fma(-alpha, ap1, rho1) : 0.0;
            // level 3 at row j
            const Faces f0 = FR.at(A, i, j, col_ok);
            const bool ok0 = col_ok && j >= 0 && j < A.ny;
            const double q0 = apply5(f0, shift_at(A, i + A.nx * j, ok0 && m0), rn0, rnm, rn1);
            if (out_lane && ok0 && j >= j0 && m0) {
                const int v = i + A.nx * j;
                w[v] = fma(alpha, pn0, w[v]);
                rho_n[v] = rn0;
                p_n[v] = pn0;
                acc[0] = fma(rn0, rn0, acc[0]);
                acc[1] = fma(rn0, q0, acc[1]);
            }
            pn0 = pn1; pn1 = pn2;
            rnm = rn0; rn0 = rn1;
            m0 = m1; m1 = m2;
            rho1 = rho2;
        }
    }
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_finalize(t[0], t[1], S); });
}

}  // namespace gpcg
