// Microbenchmark: DRAM throughput of scattered reads -- the ceiling of the compact reduced
// product (gpcg_hessvec_free), whose free rows sit at scattered positions.  Every thread reads
// R independent chunks of B bytes (B = 8, 32, 64, 128; 8-byte loads, the chunk's loads issued
// back to back) at hashed positions of a 1 GiB buffer (>> the 126 MB L2), and the kernel is
// timed with CUDA events.  Reported: useful bytes / s (R * B per thread) and the same as a
// fraction of the streaming copy peak.  Also a contiguous streaming read of the same buffer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 gather.cu -o gather.bin
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

template <int W, int R>   // W doubles per chunk, R chunks per thread
__global__ void k_gather(const double* __restrict__ a, long long nchunks, long long threads, double* out) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= threads) return;
    double acc = 0.0;
    long long base[R];
#pragma unroll
    for (int r = 0; r < R; ++r) base[r] = (long long)(mix(t * R + r) % (unsigned long long)nchunks) * W;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int w = 0; w < W; ++w) acc += __ldg(a + base[r] + w);
    if (acc == 1.2345) out[0] = acc;
}

__global__ void k_stream(const double* __restrict__ a, long long n, double* out) {
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc += __ldg(a + i);
    if (acc == 1.2345) out[0] = acc;
}

template <int W, int R>
void run(const double* a, long long n, double* out, double peak) {
    const long long nchunks = n / W;
    const long long threads = 16ll << 20;     // 16M threads x R chunks
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 7; ++rep) {
        cudaEventRecord(e0);
        k_gather<W, R><<<(unsigned)(threads / 256), 256>>>(a, nchunks, threads, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    const double bytes = (double)threads * R * W * 8;
    printf("gather chunk=%4d B  R=%d: %8.1f us  %7.1f GB/s useful  (%.3f of %.0f GB/s)\n", W * 8, R, best * 1e3,
           bytes / (best * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9 / peak, peak);
}

int main(int argc, char** argv) {
    const double peak = argc > 1 ? atof(argv[1]) : 6546.2;
    const long long n = 1ll << 27;            // 1 GiB of doubles
    double *a, *out;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&out, 8);
    cudaMemset(a, 0, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 7; ++rep) {
        cudaEventRecord(e0);
        k_stream<<<148 * 8, 256>>>(a, n, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    printf("stream read 1 GiB: %8.1f us  %7.1f GB/s  (%.3f of %.0f GB/s)\n", best * 1e3, n * 8 / (best * 1e-3) / 1e9,
           n * 8 / (best * 1e-3) / 1e9 / peak, peak);
    run<1, 4>(a, n, out, peak);
    run<4, 4>(a, n, out, peak);
    run<8, 4>(a, n, out, peak);
    run<16, 4>(a, n, out, peak);
    run<4, 1>(a, n, out, peak);
    run<4, 8>(a, n, out, peak);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
