// fin.cuh -- the decision logic that follows each global reduction (SURVEY.md
// 8(a) a6/a7), as named device functions.  With one slab the last block of the
// reducing kernel calls them in place; with several slabs or ranks the kernel
// defers (RedScratch::out), the host sums the slab totals in a fixed order
// (k_combine), allreduces them across ranks (NCCL), and k_finalize applies the
// same function to the global totals -- so every rank holds bit-identical
// scalars and takes the same branch (one collective sequence on all ranks).
#pragma once

#include "common.cuh"

namespace gpcg {

// a1 (+ a2 fused): ||grad_Omega q||^2, ||g||^2, |A|, #changed, |A\B|, <d, A d>
// -> next GP step's Cauchy step alpha_0 = ||d||^2 / <d, A d> (Eq. bqpls).
__device__ __forceinline__ void fin_accept(const double* t, bool with_cauchy, Scal* S) {
    S->pg2 = t[0];
    S->g2 = t[1];
    S->n_active = t[2];
    S->n_changed = t[3];
    S->n_nonbinding = t[4];
    if (with_cauchy) {
        S->dd = t[0];
        S->dAd = t[5];
        S->cauchy_ok = (t[5] > 0.0) ? 1 : 0;
        S->alpha0 = (t[5] > 0.0) ? t[0] / t[5] : 0.0;
    }
}

// a2 (generic kernels): <d,d>, <d,Ad> -> alpha_0; <d,Ad> <= 0 -> ENOTSPD (R7).
__device__ __forceinline__ void fin_cauchy(const double* t, Scal* S) {
    S->dd = t[0];
    S->dAd = t[1];
    S->cauchy_ok = (t[1] > 0.0) ? 1 : 0;
    S->alpha0 = (t[1] > 0.0) ? t[0] / t[1] : 0.0;
    S->s_h = -1;                                   // no step accepted yet
}

// a3: first h in [h0, h0+K) with <g,s_h> + 1/2 <s_h,A s_h> <= mu <g,s_h>
// (Eqs. gplsstop P:346-361 / cglsstop2 P:473-481); s_h = -1 if none.
__device__ __forceinline__ void fin_search(const double* t, int K, int h0, double base, double mu, Scal* S) {
    S->s_h = -1;
    for (int h = 0; h < K; ++h) {
        const double gs = t[2 * h], sAs = t[2 * h + 1];
        const double dq = gs + 0.5 * sAs;
        if (dq <= mu * gs) {
            S->s_h = h0 + h;
            S->s_alpha = scalbn(base, -(h0 + h));
            S->s_delta = dq;
            S->s_gs = gs;
            break;
        }
    }
}

// a1 + a3 speculative (k_spec): t = <g,s>, <s,As> of h = 0 (step base), then the accept sums of
// the point it wrote.  Eq. gplsstop / cglsstop2 at h = 0 holds -> the step is taken (s_h = 0;
// the GP step's search / accept sweeps skip); else s_h = -1 and the search runs from h = 1.
__device__ __forceinline__ void fin_spec(const double* t, double base, double mu, Scal* S) {
    const double gs = t[0], sAs = t[1];
    const double dq = gs + 0.5 * sAs;
    if (dq <= mu * gs) {
        S->spec_ok = 1;
        S->s_h = 0;
        S->s_alpha = base;
        S->s_delta = dq;
        S->s_gs = gs;
        fin_accept(t + 2, false, S);
    } else {
        S->spec_ok = 0;
        S->s_h = -1;
    }
}

// k5_spec (2-D GP graph): t = ||d||^2, ||g||^2 (not formed), |A|, #changed, |A\B|, <d,Ad> of the
// speculative point, then <g,s>, <s,As> of h = 0.  Accepted -> the step is taken at the old
// alpha_0 and the accept sums (with the next Cauchy form) are applied; else s_h = -1.
__device__ __forceinline__ void fin_spec6(const double* t, double mu, Scal* S) {
    const double gs = t[6], sAs = t[7];
    const double dq = gs + 0.5 * sAs;
    if (dq <= mu * gs) {
        S->spec_ok = 1;
        S->s_h = 0;
        S->s_alpha = S->alpha0;
        S->s_delta = dq;
        S->s_gs = gs;
        fin_accept(t, true, S);
    } else {
        S->spec_ok = 0;
        S->s_h = -1;
    }
}

// a5 init: gamma_0 = rho_0'rho_0, delta_0 = rho_0'A_F rho_0.
__device__ __forceinline__ void cg_init_finalize(double gamma, double delta, double eta2, long long cap, Scal* S) {
    S->cg_it = 0;
    S->cg_cap = cap;
    S->cg_eta2 = eta2;
    S->cg_maxdec = 0.0;
    S->cg_dec = 0.0;
    S->cg_gamma = gamma;
    S->cg_rnorm0 = sqrt(gamma);
    S->cg_beta = 0.0;
    S->cg_done = 0;
    S->cg_reason = CG_RUNNING;
    if (gamma == 0.0 || cap <= 0) {            // r_k = 0: w = 0 is exact (R27)
        S->cg_done = 1; S->cg_reason = CG_EXACT; S->cg_alpha = 0.0;
    } else if (!(delta > 0.0)) {
        S->cg_done = 1; S->cg_reason = CG_NOTSPD; S->cg_alpha = 0.0;
    } else {
        S->cg_alpha = gamma / delta;
    }
}

// a5 iteration (Chronopoulos-Gear): decrease of step j = 1/2 alpha_{j-1} gamma_{j-1};
//   stop if j >= 2 and dec_j <= eta2 max_{l<j} dec_l (Eq. cgstop1, R10),
//   or ||rho_j|| <= 1e-14 (1 + ||r_k||) (S:371 guard), or j >= cap;
//   else beta = gamma_j / gamma_{j-1}, alpha = gamma_j / (delta_j - beta gamma_j / alpha_{j-1})
//   (= gamma_j / <p_j, A_k p_j>; <= 0 -> ENOTSPD).
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

// ---------------------------------------------------------------- textbook PCG (block-Jacobi ILU, bjilu.cuh)
__device__ __forceinline__ void pcg2_init_fin(double gamma, double eta2, long long cap, Scal* S) {
    S->cg_it = 0;
    S->cg_cap = cap;
    S->cg_eta2 = eta2;
    S->cg_maxdec = 0.0;
    S->cg_dec = 0.0;
    S->cg_gamma = gamma;
    S->cg_rnorm0 = sqrt(gamma);
    S->cg_beta = 0.0;
    S->cg_alpha = 0.0;
    S->cg_done = 0;
    S->cg_reason = CG_RUNNING;
    if (gamma == 0.0 || cap <= 0) { S->cg_done = 1; S->cg_reason = CG_EXACT; }
}
__device__ __forceinline__ void pcg2_alpha_fin(double pq, Scal* S) {
    if (S->cg_done) return;
    if (!(pq > 0.0)) { S->cg_done = 1; S->cg_reason = CG_NOTSPD; return; }
    S->cg_alpha = S->cg_gamma / pq;
}
// after w += alpha p, r -= alpha q, z = M^-1 r: same order of tests as the oracle
__device__ __forceinline__ void pcg2_beta_fin(double gamma_new, Scal* S) {
    if (S->cg_done) return;
    const double dec = 0.5 * S->cg_alpha * S->cg_gamma;
    const long long j = S->cg_it + 1;
    S->cg_it = j;
    S->cg_dec = dec;
    int reason = CG_RUNNING;
    if (j >= 2 && dec <= S->cg_eta2 * S->cg_maxdec) reason = CG_PROGRESS;
    else if (sqrt(gamma_new) <= 1e-14 * (1.0 + S->cg_rnorm0)) reason = CG_EXACT;
    else if (j >= S->cg_cap) reason = CG_CAP;
    if (dec > S->cg_maxdec) S->cg_maxdec = dec;
    if (reason != CG_RUNNING) { S->cg_reason = reason; S->cg_done = 1; return; }
    S->cg_beta = gamma_new / S->cg_gamma;
    S->cg_gamma = gamma_new;
}

// ---------------------------------------------------------------- deferred mode
enum FinKind : int {
    FIN_ACCEPT = 0,      // 6 sums (stencil kernels: + Cauchy form)
    FIN_ACCEPT5 = 1,     // 5 sums (generic kernels)
    FIN_CAUCHY = 2,
    FIN_SEARCH = 3,
    FIN_CG_INIT = 4,
    FIN_CG_ITER = 5,
    FIN_R2 = 6,          // plain sums -> r0, r1 (objective, validation)
    FIN_PCG2_INIT = 7,   // block-Jacobi ILU PCG (bjilu.cuh): gamma_0
    FIN_PCG2_ALPHA = 8,  //   p'A p -> alpha
    FIN_PCG2_BETA = 9,   //   r'z -> decrease, stop tests, beta
    FIN_SPEC = 10,       // k_spec: h = 0 search sums + accept sums
    FIN_SPEC6 = 11,      // k5_spec: accept sums + Cauchy form + h = 0 search sums
};

struct FinArgs {
    int kind;
    int K, h0, use_alpha0, has_dir, gp;
    double mu, eta2;
    long long cap;
};

// Sum per-slab totals in slab order (fixed: bitwise deterministic).
__global__ void k_combine(const double* __restrict__ per_slab, int nslabs, int ns, double* __restrict__ tot) {
    const int s = threadIdx.x;
    if (s >= ns) return;
    double acc = 0.0;
    for (int k = 0; k < nslabs; ++k) acc += per_slab[(long long)k * kMaxSums + s];
    tot[s] = acc;
}

// The same decisions as the in-place finalisers, on the global totals.  The
// early-exit conditions of the reducing kernels are mirrored so that a sweep
// that did no work leaves the scalars untouched.
__global__ void k_finalize(const double* __restrict__ t, Scal* S, FinArgs a) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (a.gp && S->gp_done) return;               // a sweep of a finished device-driven GP phase
    if (a.gp && S->spec_ok && (a.kind == FIN_SEARCH || a.kind == FIN_ACCEPT || a.kind == FIN_ACCEPT5))
        return;                                   // ... or of a step k_spec took
    switch (a.kind) {
        case FIN_ACCEPT:
        case FIN_ACCEPT5:
            if (a.has_dir && S->s_h < 0) return;
            fin_accept(t, a.kind == FIN_ACCEPT, S);
            break;
        case FIN_CAUCHY:
            fin_cauchy(t, S);
            break;
        case FIN_SEARCH:
            if (a.use_alpha0 && !S->cauchy_ok) { S->s_h = -1; return; }
            fin_search(t, a.K, a.h0, a.use_alpha0 ? S->alpha0 : 1.0, a.mu, S);
            break;
        case FIN_CG_INIT:
            cg_init_finalize(t[0], t[1], a.eta2, a.cap, S);
            break;
        case FIN_CG_ITER:
            if (S->cg_done) return;
            cg_finalize(t[0], t[1], S);
            break;
        case FIN_R2:
            S->r0 = t[0];
            S->r1 = t[1];
            break;
        case FIN_PCG2_INIT:
            pcg2_init_fin(t[0], a.eta2, a.cap, S);
            break;
        case FIN_PCG2_ALPHA:
            pcg2_alpha_fin(t[0], S);
            break;
        case FIN_PCG2_BETA:
            pcg2_beta_fin(t[0], S);
            break;
        case FIN_SPEC:
            if (a.use_alpha0 && !S->cauchy_ok) { S->spec_ok = 0; S->s_h = -1; return; }
            fin_spec(t, a.use_alpha0 ? S->alpha0 : 1.0, a.mu, S);
            break;
        case FIN_SPEC6:
            if (!S->cauchy_ok) { S->spec_ok = 0; S->s_h = -1; return; }
            fin_spec6(t, a.mu, S);
            break;
    }
}

// ---------------------------------------------------------------- a7 on the device: the GP phase
// as graph chunks of [search, accept, k_gp_step]; the host polls once per chunk.
__global__ void k_gp_begin(Scal* S, double tau, double eta1, long long gp_cap) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    S->gp_tau = tau;
    S->gp_eta1 = eta1;
    S->gp_cap = gp_cap;
    S->gp_j = 0;
    S->gp_maxdec = 0.0;
    S->gp_last_dec = 0.0;
    S->gp_done = 0;
    S->gp_reason = GP_RUNNING;
    S->spec_ok = 0;
    if (sqrt(S->pg2) <= tau) { S->gp_done = 1; S->gp_reason = GP_CONV; }
}

// After search + accept of GP step j (Eq. next-y / gplsstop): the stop rules of the phase,
// Eq. pgstop1 (no change of the active set, as index sets R9), Eq. pgstop2 (decrease <=
// eta1 * the largest earlier decrease, from j >= 2: R10), the cap; then the convergence test
// ||grad_Omega q|| <= tau (R13).  A first search batch without an acceptable step (or a
// Cauchy step with <d,Ad> <= 0) hands the step back to the host (GP_HOST).
__global__ void k_gp_step(Scal* S) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    S->spec_ok = 0;                                      // the next step's sweeps run
    if (S->gp_done) return;
    if (S->s_h < 0) { S->gp_done = 1; S->gp_reason = GP_HOST; return; }
    const long long j = ++S->gp_j;
    const double dec = -S->s_delta;                      // q(y_{j-1}) - q(y_j)
    S->gp_last_dec = dec;
    const bool stop = (S->n_changed == 0.0) || (j >= 2 && dec <= S->gp_eta1 * S->gp_maxdec) || (j >= S->gp_cap);
    if (dec > S->gp_maxdec) S->gp_maxdec = dec;
    if (stop) { S->gp_done = 1; S->gp_reason = GP_STOP; }
    else if (sqrt(S->pg2) <= S->gp_tau) { S->gp_done = 1; S->gp_reason = GP_CONV; }
}

// host-completed step: write back the phase state
__global__ void k_gp_set(Scal* S, long long j, double maxdec, int done, int reason) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    S->gp_j = j;
    S->gp_maxdec = maxdec;
    S->gp_done = done;
    S->gp_reason = reason;
}

}  // namespace gpcg
