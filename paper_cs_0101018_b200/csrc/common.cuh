// common.cuh -- operator policies, bounds policies, device scalars and the
// deterministic two-stage block reductions shared by every GPCG kernel.
//
// Layout: every vector is a dense fp64 array
// of the CSR rows, or, for stencils, of the grid rows at a pitch of nx rounded
// up to 32 points (256-byte aligned rows; linear index v = i + pitch*j; the
// padding is never read).  The free mask is one byte per point (1 = free),
// same pitch.  Vectors used by CG are
// zero off the free set, which makes A_F p = [v in F] (A p)_v.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gpcg {

constexpr int kThreads = 256;      // generic kernels: 256 threads = 8 warps
constexpr int kMarchThreads = 128; // column-march kernels: 4 warps (finer occupancy steps)
constexpr int kMaxSums = 34;       // reductions per kernel (search: 2*16 + 2)
constexpr int kMaxK = 16;          // projected-search step sizes per sweep

// ----------------------------------------------------------------------------
// point / neighbour iteration
// ----------------------------------------------------------------------------
struct Pt {
    int v, i, j, k;
};

// 5-point face-weight operator (gpcg.h, gpcg_create_stencil2d).  ld 0 means a
// broadcast row.  Iteration covers 32x8 point tiles: threadIdx.x&31 runs along
// i (coalesced), threadIdx.x>>5 along j.
//
// Slabs: a handle may own only grid rows [0, ny) of a larger
// grid (a row slab of one rank, or one of several slabs on one device).  Rows
// [rlo, 0) and [ny, rhi) are then GHOST rows holding the neighbouring slab's
// values (refreshed by the host's halo exchange); rows outside [rlo, rhi) are
// the Dirichlet boundary (zero).  Single slab: rlo = 0, rhi = ny.  Face arrays
// (ld != 0) carry the ghost rows too; outputs are only ever written for owned
// rows.
struct StencilOp {
    int nx, ny, pitch;                 // point (i, j) lives at i + pitch*j (pitch = nx rounded up to 32)
    const double* __restrict__ wx;
    const double* __restrict__ wy;
    const double* __restrict__ shift;
    long long wx_ld, wy_ld;
    int rlo, rhi;                      // readable rows (owned + ghost); outside: Dirichlet zero

    __device__ __forceinline__ int num_units() const { return ((nx + 31) >> 5) * ((ny + 7) >> 3); }
    __device__ __forceinline__ Pt point(int v) const { return Pt{v, v % pitch, v / pitch, 0}; }

    template <class Body>
    __device__ __forceinline__ void for_each_point(Body&& body) const {
        const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
        const int ntx = (nx + 31) >> 5;
        const int T = num_units();
        for (int t = blockIdx.x; t < T; t += gridDim.x) {
            const int bj = t / ntx, bi = t - bj * ntx;
            const int i = (bi << 5) + tx, j = (bj << 3) + ty;
            if (i < nx && j < ny) body(Pt{i + pitch * j, i, j, 0});
        }
    }

    // cb(column, coefficient) for every stored entry of row p.v; diagonal first.
    template <class CB>
    __device__ __forceinline__ void for_each_nbr(const Pt& p, CB&& cb) const {
        const double ww = __ldg(wx + (long long)p.j * wx_ld + p.i);
        const double we = __ldg(wx + (long long)p.j * wx_ld + p.i + 1);
        const double ws = __ldg(wy + (long long)p.j * wy_ld + p.i);
        const double wn = __ldg(wy + (long long)(p.j + 1) * wy_ld + p.i);
        double d = (ww + we) + (ws + wn);
        if (shift) d += __ldg(shift + p.v);
        cb(p.v, d);
        if (p.i > 0) cb(p.v - 1, -ww);
        if (p.i < nx - 1) cb(p.v + 1, -we);
        if (p.j - 1 >= rlo) cb(p.v - pitch, -ws);
        if (p.j + 1 < rhi) cb(p.v + pitch, -wn);
    }
};

// General CSR (both triangles, int64 row_ptr, int32 col).  One thread per row.
// Columns are LOCAL offsets from the slab's first owned row: a slab's vectors
// hold [lo ghost band | n owned rows | hi ghost band] and col may be negative
// (lower band) or >= n (upper band).
struct CsrOp {
    int n;
    const long long* __restrict__ rp;
    const int* __restrict__ ci;
    const double* __restrict__ val;

    __device__ __forceinline__ int num_units() const { return (n + kThreads - 1) / kThreads; }
    __device__ __forceinline__ Pt point(int v) const { return Pt{v, 0, 0, 0}; }

    template <class Body>
    __device__ __forceinline__ void for_each_point(Body&& body) const {
        for (int v = blockIdx.x * kThreads + threadIdx.x; v < n; v += gridDim.x * kThreads)
            body(Pt{v, 0, 0, 0});
    }

    template <class CB>
    __device__ __forceinline__ void for_each_nbr(const Pt& p, CB&& cb) const {
        const long long e = __ldg(rp + p.v + 1);
        for (long long k = __ldg(rp + p.v); k < e; ++k) cb(__ldg(ci + k), __ldg(val + k));
    }
};

// 3-D 7-point face-weight operator (gpcg_create_stencil3d), for the
// generic kernels.  Point (i, j, k) of the slab at v = i + nx j + plane k (plane = nx ny, no
// padding); k in [0, nz) owned, [klo, khi) readable (ghost planes of a slab), outside: zero.
// wx: (nx+1) per (j, k) line; wy: nx per face line, ny+1 face lines per plane; wz: one plane
// of nx ny per face plane (face plane k joins planes k-1, k).
struct Stencil3Op {
    int nx, ny, nz;
    long long plane;
    const double* __restrict__ wx;
    const double* __restrict__ wy;
    const double* __restrict__ wz;
    const double* __restrict__ shift;
    int klo, khi;

    __device__ __forceinline__ int num_units() const {
        return (int)((plane * nz + kThreads - 1) / kThreads);
    }
    __device__ __forceinline__ Pt point(int v) const {
        const int k = v / (int)plane, r = v - k * (int)plane;
        return Pt{v, r % nx, r / nx, k};
    }

    template <class Body>
    __device__ __forceinline__ void for_each_point(Body&& body) const {
        const int n = (int)(plane * nz);
        for (int v = blockIdx.x * kThreads + threadIdx.x; v < n; v += gridDim.x * kThreads) {
            const int k = v / (int)plane, r = v - k * (int)plane;
            const int j = r / nx, i = r - j * nx;
            body(Pt{v, i, j, k});
        }
    }

    template <class CB>
    __device__ __forceinline__ void for_each_nbr(const Pt& p, CB&& cb) const {
        const long long line = (long long)p.k * ny + p.j;
        const double ww = __ldg(wx + line * (nx + 1) + p.i);
        const double we = __ldg(wx + line * (nx + 1) + p.i + 1);
        const double ws = __ldg(wy + ((long long)p.k * (ny + 1) + p.j) * nx + p.i);
        const double wn = __ldg(wy + ((long long)p.k * (ny + 1) + p.j + 1) * nx + p.i);
        const long long ip = (long long)p.j * nx + p.i;
        const double wd = __ldg(wz + (long long)p.k * plane + ip);
        const double wu = __ldg(wz + (long long)(p.k + 1) * plane + ip);
        double d = ((ww + we) + (ws + wn)) + (wd + wu);
        if (shift) d += __ldg(shift + p.v);
        cb(p.v, d);
        if (p.i > 0) cb(p.v - 1, -ww);
        if (p.i < nx - 1) cb(p.v + 1, -we);
        if (p.j > 0) cb(p.v - nx, -ws);
        if (p.j < ny - 1) cb(p.v + nx, -wn);
        if (p.k - 1 >= klo) cb(p.v - (int)plane, -wd);
        if (p.k + 1 < khi) cb(p.v + (int)plane, -wu);
    }
};

// ----------------------------------------------------------------------------
// bounds: per-point arrays, or one scalar pair detected at create time
// ----------------------------------------------------------------------------
struct Bounds {
    const double* __restrict__ l;
    const double* __restrict__ u;
    double lc, uc;
};

template <bool kScalar>
__device__ __forceinline__ double lo(const Bounds& B, int v) {
    if constexpr (kScalar) return B.lc; else return __ldg(B.l + v);
}
template <bool kScalar>
__device__ __forceinline__ double hi(const Bounds& B, int v) {
    if constexpr (kScalar) return B.uc; else return __ldg(B.u + v);
}

// P[x] = mid(l, u, x).  Written so that the result is exactly l or
// u whenever x is outside, which keeps A(x) an exact-equality test (R15).
__device__ __forceinline__ double mid(double l, double u, double x) {
    return x < l ? l : (x > u ? u : x);
}

// Trial point of both projected searches: mid(l, u, y + alpha * (sgn * dir)).
// GP: sgn = -1, dir = g (Eq. next-y); CG: sgn = +1, dir = d_k (Eq. cglsstop2).
// Used verbatim by the search sweep and by the accept kernel so that the
// accepted iterate is bit-identical to the evaluated trial.
__device__ __forceinline__ double trial(double y, double dir, double sgn, double alpha,
                                        double l, double u) {
    return mid(l, u, fma(alpha, sgn * dir, y));
}

// Eq. proj-gradient; fixed variables give 0 (R16).
// Branch-free: the component is 0 at a lower bound unless g < 0, at an upper bound unless
// g > 0 (both at once for l = u: always 0), else g -- the same values as the case analysis.
__device__ __forceinline__ double pgrad(double x, double g, double l, double u) {
    const bool al = (x == l), au = (x == u);
    const bool zero = (al && !(g < 0.0)) || (au && !(g > 0.0));
    return zero ? 0.0 : g;
}

// ----------------------------------------------------------------------------
// device scalars (one block per handle; the host mirrors it in pinned memory)
// ----------------------------------------------------------------------------
enum CgReason : int { CG_RUNNING = 0, CG_PROGRESS = 1, CG_EXACT = 2, CG_CAP = 3, CG_NOTSPD = -5 };

struct Scal {
    // a1: project / accept / regrad
    double pg2, g2, n_active, n_changed, n_nonbinding;
    // a2: Cauchy step
    double dd, dAd, alpha0;
    int cauchy_ok, pad0;
    // a3: projected search
    double s_alpha, s_delta, s_gs;
    int s_h, s_pad;
    // a5: CG (Chronopoulos-Gear single-reduction form)
    double cg_alpha, cg_beta, cg_gamma, cg_rnorm0, cg_maxdec, cg_eta2, cg_dec;
    long long cg_it, cg_cap;
    int cg_done, cg_reason;
    // generic dot products (objective)
    double r0, r1;
    // a7: GP phase driven on the device (graph chunks of search + accept + k_gp_step)
    double gp_tau, gp_eta1, gp_maxdec, gp_last_dec;
    long long gp_j, gp_cap;
    int gp_done, gp_reason;
    int gp_fb, gp_pad;               // k6_gp_loop: steps whose speculative sweep was rejected (diagnostic)
    int spec_ok, spec_pad;           // k_spec accepted this GP step's h = 0 (its search / accept sweeps skip)
};
enum GpReason : int { GP_RUNNING = 0, GP_STOP = 1, GP_CONV = 2, GP_HOST = 3 };

// A device-driven GP-phase search / accept sweep with nothing to do: the phase is over, or this
// step's speculative sweep (k_spec) was accepted.
__device__ __forceinline__ bool gp_skip(const Scal* S) {
    return *(const volatile int*)&S->gp_done || *(const volatile int*)&S->spec_ok;
}


// ----------------------------------------------------------------------------
// deterministic two-stage reduction
// ----------------------------------------------------------------------------
struct RedScratch {
    double* partials;          // [kMaxSums][gridDim.x]
    unsigned int* counter;     // zero between launches
    double* out;               // non-null: DEFERRED mode (slabs / ranks) -- the last block writes the
                               // totals here and the decision logic runs in k_finalize after the
                               // cross-slab / cross-rank sum (fin.cuh); null: finalise in place
};

template <int NS>
__device__ __forceinline__ void warp_reduce(double (&v)[NS]) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[s] += __shfl_xor_sync(0xffffffffu, v[s], o);
    }
}

// Block-reduce v[NS] (all threads contribute); result valid in thread 0.
template <int NS>
__device__ __forceinline__ void block_reduce(double (&v)[NS], double* smem /* NS*32 */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    warp_reduce<NS>(v);
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) smem[s * 32 + wid] = v[s];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) v[s] = (lane < (int)(blockDim.x >> 5)) ? smem[s * 32 + lane] : 0.0;
        warp_reduce<NS>(v);
    }
    __syncthreads();
}

// Stage 1: per-block partials; stage 2: the last block to finish sums them in
// a fixed order and calls fin(total) on thread 0.  Bitwise deterministic for
// a fixed grid size (no float atomics; "Vec Red").
template <int NS, class Fin>
__device__ __forceinline__ void reduce_and_finish(double (&v)[NS], const RedScratch& R, Fin&& fin) {
    __shared__ double smem[NS * 32];
    __shared__ bool am_last;
    block_reduce<NS>(v, smem);
    const int G = gridDim.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) R.partials[s * G + blockIdx.x] = v[s];
        __threadfence();
        const unsigned t = atomicAdd(R.counter, 1u);
        am_last = (t == (unsigned)G - 1);
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    double t[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        double acc = 0.0;
        for (int b = threadIdx.x; b < G; b += blockDim.x) acc += __ldcg(R.partials + s * G + b);
        t[s] = acc;
    }
    block_reduce<NS>(t, smem);
    if (threadIdx.x == 0) {
        *R.counter = 0u;
        if (R.out) {
#pragma unroll
            for (int s = 0; s < NS; ++s) R.out[s] = t[s];
        } else {
            fin(t);
        }
    }
}

}  // namespace gpcg
