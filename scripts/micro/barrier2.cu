// Microbenchmark: grid-barrier variants for the persistent loops (cost per barrier, no work).
//  v0: one counter, arrive = threadfence + atomicAdd, spin on the counter (march_tma.cuh today)
//  v1: v0 but pollers spin on a separate generation flag written by the last arriver
//  v2: 16 sub-counters (one per 128-byte line), the last arriver of each bumps the top counter;
//      the last top arriver publishes the generation flag
//  v3: v1 with a release atomic instead of threadfence + relaxed atomic
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 barrier2.cu -o barrier2
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_rel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

template <int V>
__device__ __forceinline__ void barrier(unsigned* w, unsigned nb, unsigned& gen) {
    // w[0]: counter, w[32]: flag, w[64 + 32*s]: sub-counters
    __syncthreads();
    if (threadIdx.x == 0) {
        if (V == 0) {
            __threadfence();
            const unsigned target = (gen + 1) * nb;
            atomicAdd(w, 1u);
            while (ld_acq(w) < target) {}
        } else if (V == 1 || V == 3) {
            unsigned old;
            if (V == 1) { __threadfence(); old = atomicAdd(w, 1u); }
            else old = atom_add_rel(w, 1u);
            if (old == (gen + 1) * nb - 1) st_rel(w + 32, gen + 1);
            else while (ld_acq(w + 32) < gen + 1) {}
        } else {
            __threadfence();
            const unsigned s = blockIdx.x & 15;
            const unsigned per = (nb - s + 15) / 16;           // CTAs in sub-group s
            const unsigned old = atomicAdd(w + 64 + 32 * s, 1u);
            if (old == (gen + 1) * per - 1) {
                const unsigned o2 = atomicAdd(w, 1u);
                if (o2 == (gen + 1) * 16 - 1) st_rel(w + 32, gen + 1);
            }
            while (ld_acq(w + 32) < gen + 1) {}
        }
        ++gen;
    }
    __syncthreads();
}

template <int V>
__global__ void k_bar(unsigned* w, int iters) {
    unsigned gen = 0;
    for (int it = 0; it < iters; ++it) barrier<V>(w, gridDim.x, gen);
}

template <int V>
void run(int g, unsigned* w) {
    const int iters = 4000, threads = 160;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(w, 0, 4096);
        int it = iters;
        void* args[] = {&w, &it};
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k_bar<V>, dim3(g), dim3(threads), args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep == 1) printf("v%d grid %d: %.3f us per barrier (%s)\n", V, g, 1e3 * ms / iters, cudaGetErrorString(e));
    }
}

int main() {
    unsigned* w; cudaMalloc(&w, 4096);
    for (int g : {148, 296, 592}) { run<0>(g, w); run<1>(g, w); run<2>(g, w); run<3>(g, w); }
    return 0;
}
