// extract.cuh -- explicit extraction of the reduced Hessian A_k = Z_k' A Z_k as a compact
// CSR matrix (the PETSc route the paper took, MatGetSubMatrix) for the
// extraction ablation of SURVEY.md 8(f) NEXT-4 (gpcg_params.cg_mode = 1).  The hot path
// applies A_F in place on full-length masked vectors (cg_mode = 0); this mode builds
//   idx[v]  compact index of free point v (exclusive prefix sum over the free mask, in the
//           owned-point order k = i + nx j (+ plane k) / CSR row order: deterministic),
//   A_F     m x m CSR (row_ptr by a second prefix sum over the free rows' in-set degrees),
//   r_F     the gradient on F (A y - b recomputed at the free points),
// runs the CSR CG kernels on the compact system and scatters w back (zero off F).
#pragma once

#include "common.cuh"

namespace gpcg {

constexpr int kScanBlock = 1024;          // owned points per scan block (256 threads x 4)

// owned-point order k -> storage index v (rowlen = points per stored row, pitch = stride)
__device__ __forceinline__ long long owned_v(long long k, int rowlen, int pitch) {
    return (k % rowlen) + (long long)pitch * (k / rowlen);
}

// per-block counts of set flags (flags: the free mask, or a per-free-row count array)
template <bool kMaskInput>
__global__ void __launch_bounds__(256)
k_scan_count(long long n, int rowlen, int pitch, const unsigned char* __restrict__ mask,
             const int* __restrict__ vals, long long* __restrict__ blocksum) {
    __shared__ long long sm[8];
    long long acc = 0;
    const long long base = (long long)blockIdx.x * kScanBlock;
    for (int e = threadIdx.x; e < kScanBlock; e += 256) {
        const long long k = base + e;
        if (k < n) acc += kMaskInput ? (mask[owned_v(k, rowlen, pitch)] ? 1 : 0) : vals[k];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < 8; ++w) t += sm[w];
        blocksum[blockIdx.x] = t;
    }
}

// exclusive scan of the block sums in place (one CTA; nb up to millions, sequential chunks)
__global__ void k_scan_blocks(long long nb, long long* __restrict__ blocksum, long long* __restrict__ total) {
    __shared__ long long carry;
    __shared__ long long sm[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long long c0 = 0; c0 < nb; c0 += blockDim.x) {
        const long long i = c0 + threadIdx.x;
        long long v = i < nb ? blocksum[i] : 0;
        // inclusive warp scan
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        long long x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) sm[w] = x;
        __syncthreads();
        if (w == 0) {
            long long s = lane < (int)(blockDim.x >> 5) ? sm[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            sm[lane] = s;                          // inclusive prefix of the warp totals
        }
        __syncthreads();
        const long long wbase = w > 0 ? sm[w - 1] : 0;
        if (i < nb) blocksum[i] = carry + wbase + x - v;   // exclusive
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += wbase + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

// idx[v] = compact index of free v (exclusive prefix within the block + the block offset),
// pos[i] = v.  Block-local order: e = 0 .. kScanBlock-1 (thread t handles e = 4t .. 4t+3).
__global__ void __launch_bounds__(256)
k_scan_assign(long long n, int rowlen, int pitch, const unsigned char* __restrict__ mask,
              const long long* __restrict__ blocksum, int* __restrict__ idx, int* __restrict__ pos) {
    __shared__ long long sm[8];
    const long long base = (long long)blockIdx.x * kScanBlock;
    int f[4];
    long long v[4];
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long k = base + 4 * threadIdx.x + q;
        v[q] = k < n ? owned_v(k, rowlen, pitch) : -1;
        f[q] = (k < n && mask[v[q]]) ? 1 : 0;
        cnt += f[q];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long x = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[w] = x;
    __syncthreads();
    long long wbase = 0;
    for (int u = 0; u < w; ++u) wbase += sm[u];
    long long run = blocksum[blockIdx.x] + wbase + x - cnt;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (f[q]) {
            if (idx) idx[v[q]] = (int)run;
            pos[run] = (int)v[q];
            ++run;
        }
    }
}

// rp[i] = exclusive prefix of vals (block-local order i = 4t .. 4t+3, plus the block offset)
__global__ void __launch_bounds__(256)
k_scan_assign_vals(long long n, const int* __restrict__ vals, const long long* __restrict__ blocksum,
                   long long* __restrict__ rp) {
    __shared__ long long sm[8];
    const long long base = (long long)blockIdx.x * kScanBlock;
    int f[4];
    long long cnt = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long k = base + 4 * threadIdx.x + q;
        f[q] = k < n ? vals[k] : 0;
        cnt += f[q];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long x = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[w] = x;
    __syncthreads();
    long long wbase = 0;
    for (int u = 0; u < w; ++u) wbase += sm[u];
    long long run = blocksum[blockIdx.x] + wbase + x - cnt;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long k = base + 4 * threadIdx.x + q;
        if (k < n) rp[k] = run;
        run += f[q];
    }
}

// in-set degree of every free row (compact order)
template <class Op>
__global__ void __launch_bounds__(kThreads)
k_extract_count(Op A, long long m, const int* __restrict__ pos, const unsigned char* __restrict__ mask,
                int* __restrict__ cnt) {
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < m; i += (long long)gridDim.x * kThreads) {
        const int v = pos[i];
        int c0 = 0;
        A.for_each_nbr(A.point(v), [&](int c, double) { c0 += mask[c] ? 1 : 0; });
        cnt[i] = c0;
    }
}

// A_F rows (columns as compact indices, in the operator's neighbour order), r_F = (A y - b)_F
template <class Op>
__global__ void __launch_bounds__(kThreads)
k_extract_fill(Op A, long long m, const int* __restrict__ pos, const unsigned char* __restrict__ mask,
               const int* __restrict__ idx, const long long* __restrict__ rp, int* __restrict__ col,
               double* __restrict__ val, const double* __restrict__ y, const double* __restrict__ b,
               const double* __restrict__ dinv, double* __restrict__ gF, double* __restrict__ dinvF) {
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < m; i += (long long)gridDim.x * kThreads) {
        const int v = pos[i];
        long long p = rp[i];
        double ay = 0.0;
        A.for_each_nbr(A.point(v), [&](int c, double a) {
            ay = fma(a, __ldg(y + c), ay);
            if (mask[c]) {
                col[p] = idx[c];
                val[p] = a;
                ++p;
            }
        });
        gF[i] = ay - __ldg(b + v);
        dinvF[i] = dinv[v];
    }
}

// w = Z w_F (zero off F)
__global__ void __launch_bounds__(kThreads)
k_scatter(long long n, int rowlen, int pitch, const unsigned char* __restrict__ mask, const int* __restrict__ idx,
          const double* __restrict__ wF, double* __restrict__ w) {
    for (long long k = blockIdx.x * (long long)kThreads + threadIdx.x; k < n; k += (long long)gridDim.x * kThreads) {
        const long long v = owned_v(k, rowlen, pitch);
        w[v] = mask[v] ? wF[idx[v]] : 0.0;
    }
}

}  // namespace gpcg
