// Microbenchmark: cost of the software grid barrier used by the persistent kernels
// (march_tma.cuh grid_barrier) and of barrier + fixed-order partial-sum reduction, at the
// persistent kernels' grid shapes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks, unsigned int& gen) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int target = (gen + 1) * nblocks;
        atomicAdd(bar, 1u);
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
        ++gen;
    }
    __syncthreads();
}

__global__ void k_bar(unsigned int* bar, int iters, double* part, int reduce) {
    unsigned int gen = 0;
    __shared__ double red[32];
    double acc = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        if (reduce) {
            // block reduce + partial write
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
            __syncthreads();
            if (threadIdx.x == 0) {
                double t = 0; for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
                part[(it & 1) * gridDim.x + blockIdx.x] = t;
            }
        }
        grid_barrier(bar, gridDim.x, gen);
        if (reduce) {
            double t = 0.0;
            for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += __ldcg(part + (it & 1) * gridDim.x + b);
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
            __syncthreads();
            acc = red[0] * 1e-30 + threadIdx.x;
            __syncthreads();
        }
    }
    if (acc == 12345.0) part[0] = acc;
}

int main() {
    unsigned int* bar; double* part;
    cudaMalloc(&bar, 4); cudaMalloc(&part, 1 << 20);
    int grids[] = {148, 296, 592};
    for (int reduce = 0; reduce < 2; ++reduce)
        for (int g : grids) {
            const int iters = 2000;
            int threads = 160;
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(bar, 0, 4);
                void* args[] = {&bar, (void*)&iters, &part, &reduce};
                cudaEventRecord(a);
                cudaError_t e = cudaLaunchCooperativeKernel((void*)k_bar, dim3(g), dim3(threads), args, 0, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep == 1) printf("grid %d reduce %d: %.3f us per barrier (%s)\n", g, reduce, 1e3 * ms / iters,
                                     cudaGetErrorString(e));
            }
        }
    return 0;
}
