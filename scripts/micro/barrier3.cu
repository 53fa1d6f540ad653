// Microbenchmark: grid barrier with thread-block clusters (hardware cluster barrier + one
// global arrival per cluster) vs the flat software barrier, cooperative launch, 160 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 barrier3.cu -o barrier3.bin
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int CL>
__global__ void k_bar(unsigned* w, int iters) {
    unsigned gen = 0;
    const unsigned nb = gridDim.x;
    for (int it = 0; it < iters; ++it) {
        if (CL == 1) {
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(w, 1u);
                const unsigned target = (gen + 1) * nb;
                while (ld_acq(w) < target) {}
            }
            __syncthreads();
        } else {
            cg::cluster_group cl = cg::this_cluster();
            cl.sync();                                    // the cluster's CTAs have arrived
            if (cl.block_rank() == 0 && threadIdx.x == 0) {
                __threadfence();
                atomicAdd(w, 1u);
                const unsigned target = (gen + 1) * (nb / CL);
                while (ld_acq(w) < target) {}
            }
            cl.sync();                                    // released by the leader
        }
        ++gen;
    }
}

template <int CL>
void run(int g, unsigned* w) {
    const int iters = 4000, threads = 160;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    int na = 1;
    if (CL > 1) {
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = CL; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
        na = 2;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    if (CL > 1) {
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, (void*)k_bar<CL>, &cfg);
        printf("cluster %d: max active clusters %d (CTAs %d)\n", CL, ncl, ncl * CL);
    }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(w, 0, 4096);
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_bar<CL>, w, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep == 1) printf("cluster %d grid %d: %.3f us per barrier (%s / %s)\n", CL, g, 1e3 * ms / iters,
                             cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
    }
}

int main() {
    unsigned* w; cudaMalloc(&w, 4096);
    for (int g : {296, 592}) { run<1>(g, w); run<2>(g, w); run<4>(g, w); }
    return 0;
}
