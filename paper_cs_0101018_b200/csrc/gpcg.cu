// gpcg.cu -- libgpcg.so: the C ABI of include/gpcg.h and the host state machine
// of Algorithm GPCG driving the sm_100a kernels of kernels.cuh.
//
// Control: the host runs the outer / GP logic from a few
// device scalars read once per GP sub-step (one pinned 200-byte readback); the
// CG inner solve runs as CUDA-graph chunks of `cg_chunk` single-reduction
// iterations whose device-side finaliser sets a done flag (later launches are
// no-ops), polled once per chunk.  The decisions below follow, step by step,
// the same algorithm as oracle/gpcg_oracle.c (written independently; the two
// share no code).
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "gpcg.h"
#include "kernels.cuh"
#include "march.cuh"
#include "tile.cuh"

#include <cudaTypedefs.h>

using namespace gpcg;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return set_err(e_ == cudaErrorMemoryAllocation ? GPCG_ENOMEM : GPCG_ECUDA,        \
                           "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define CKLAUNCH()                                                                            \
    do {                                                                                      \
        cudaError_t e_ = cudaGetLastError();                                                  \
        if (e_ != cudaSuccess)                                                                \
            return set_err(GPCG_ECUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_),   \
                           __FILE__, __LINE__);                                               \
    } while (0)

bool trace_on() {
    static const bool on = getenv("GPCG_TRACE") != nullptr;
    return on;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

struct gpcg_problem {
    int dev = 0, sms = 148;
    cudaStream_t user = nullptr;   // caller's stream
    cudaStream_t st = nullptr;     // private work stream (capturable)
    cudaEvent_t ev_sync = nullptr, ev_a = nullptr, ev_b = nullptr;
    bool is_csr = false;
    bool generic = false;          // GPCG_GENERIC=1: stencil problems use the flat generic kernels (A/B tests)
    StencilOp sop{};
    CsrOp cop{};
    int n = 0;                     // unknowns (nx*ny or CSR rows)
    int rows = 1, cols = 0, pitch = 0;   // vector layout: rows x cols at a pitch (stencil: nx rounded up to 32)
    long long nalloc = 0;          // doubles per internal vector = rows * pitch
    long long nnz = 0;
    // library-owned inputs
    double *wx = nullptr, *wy = nullptr, *shift = nullptr;
    long long* rp = nullptr;
    int* ci = nullptr;
    double* val = nullptr;
    double *b = nullptr, *l = nullptr, *u = nullptr;
    double c = 0.0;
    bool sb = false;               // scalar bounds detected
    bool bc = false;               // stencil with broadcast faces and no shift
    Bounds bounds{};
    // work vectors
    double *Y[2] = {nullptr, nullptr}, *G[2] = {nullptr, nullptr};
    unsigned char* M[2] = {nullptr, nullptr};
    unsigned char* Mcg = nullptr;  // free mask of the running CG call (fixed address for the graph)
    double *W = nullptr, *P = nullptr;
    double *Rho[2] = {nullptr, nullptr}, *Q[2] = {nullptr, nullptr}, *S2[2] = {nullptr, nullptr};
    double *stage_in = nullptr, *stage_out = nullptr;
    // scalars + reduction scratch
    Scal* dS = nullptr;
    Scal* hS = nullptr;            // pinned mirror
    double* partials = nullptr;
    unsigned int* counter = nullptr;
    int grid = 1;                  // generic kernels (CSR, hessvec, objective)
    MarchGeom mg1{}, mg2{};        // column-march geometry for halo 1 / halo 2 stencil kernels
    int grid_m1 = 1, grid_m2 = 1;
    // TMA tile path (broadcast-face stencils): tensor maps of every internal array
    bool tile = false;
    int tile_mask = 7;             // GPCG_TILE bits: 1 accept, 2 search, 4 CG iteration (A/B and debugging)
    TileGeom tg{};
    int grid_t_cg = 1, grid_t_acc = 1, grid_t_srch = 1;
    CUtensorMap tmY[2], tmG[2], tmW, tmWc, tmB, tmL, tmU, tmRho[2], tmP[2], tmM[2], tmMcg, tmStage;
    gpcg_params prm{};
    int free_mask = -1;            // index into M of the recorded free set, -1 none
    // CG graph chunk
    cudaGraphExec_t cg_exec = nullptr;
    int cg_exec_chunk = 0;
    long long launches = 0;
    cudaEvent_t ev_c0 = nullptr, ev_c1 = nullptr;
    long long cg_iters_timed = 0, cg_free_iters_timed = 0;
    double t_cg_timed_ms = 0.0;

    RedScratch red() const { return RedScratch{partials, counter}; }
};

namespace {

int sync_scal(gpcg_problem* h) {
    CK(cudaMemcpyAsync(h->hS, h->dS, sizeof(Scal), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return GPCG_OK;
}

// user stream -> work stream ordering at entry, work -> user at exit
int enter(gpcg_problem* h) {
    CK(cudaSetDevice(h->dev));
    CK(cudaEventRecord(h->ev_sync, h->user));
    CK(cudaStreamWaitEvent(h->st, h->ev_sync, 0));
    return GPCG_OK;
}
int leave(gpcg_problem* h) {
    CK(cudaEventRecord(h->ev_sync, h->st));
    CK(cudaStreamWaitEvent(h->user, h->ev_sync, 0));
    return GPCG_OK;
}

template <class F>
void with_op(gpcg_problem* h, F&& f) {
    if (h->is_csr) {
        if (h->sb) f(h->cop, std::true_type()); else f(h->cop, std::false_type());
    } else {
        if (h->sb) f(h->sop, std::true_type()); else f(h->sop, std::false_type());
    }
}

template <class F>
void with_op_only(gpcg_problem* h, F&& f) {
    if (h->is_csr) f(h->cop); else f(h->sop);
}

int units(const gpcg_problem* h) {
    if (h->is_csr) return (h->n + kThreads - 1) / kThreads;
    return ((h->sop.nx + 31) / 32) * ((h->sop.ny + 7) / 8);
}

// copy n doubles from a host-or-device pointer into a device buffer
int upload(gpcg_problem* h, double* dst, const double* src, size_t count) {
    const cudaMemcpyKind k = is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpyAsync(dst, src, count * sizeof(double), k, h->st));
    return GPCG_OK;
}
int upload_bytes(gpcg_problem* h, void* dst, const void* src, size_t bytes) {
    const cudaMemcpyKind k = is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpyAsync(dst, src, bytes, k, h->st));
    return GPCG_OK;
}

// user vector (contiguous n) <-> internal vector (rows x cols at pitch)
int upload_vec(gpcg_problem* h, double* dst, const double* src) {
    const cudaMemcpyKind k = is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpy2DAsync(dst, (size_t)h->pitch * sizeof(double), src, (size_t)h->cols * sizeof(double),
                         (size_t)h->cols * sizeof(double), h->rows, k, h->st));
    return GPCG_OK;
}
int download_vec(gpcg_problem* h, double* dst, const double* src) {
    const cudaMemcpyKind k = is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(cudaMemcpy2DAsync(dst, (size_t)h->cols * sizeof(double), src, (size_t)h->pitch * sizeof(double),
                         (size_t)h->cols * sizeof(double), h->rows, k, h->st));
    return GPCG_OK;
}

int count_nonfinite(gpcg_problem* h, const double* a, long long cnt, double* out) {
    const int g = (int)std::min<long long>((cnt + kThreads - 1) / kThreads, (long long)h->sms * 4);
    k_count_nonfinite<<<std::max(g, 1), kThreads, 0, h->st>>>(cnt, a, h->dS, h->red());
    CKLAUNCH();
    int rc = sync_scal(h);
    if (rc) return rc;
    *out = h->hS->r0;
    return GPCG_OK;
}

void free_all(gpcg_problem* h) {
    if (!h) return;
    cudaSetDevice(h->dev);
    if (h->st) cudaStreamSynchronize(h->st);
    void* ptrs[] = {h->wx, h->wy, h->shift, h->rp, h->ci, h->val, h->b, h->l, h->u,
                    h->Y[0], h->Y[1], h->G[0], h->G[1], h->M[0], h->M[1], h->Mcg, h->W, h->P,
                    h->Rho[0], h->Rho[1], h->Q[0], h->Q[1], h->S2[0], h->S2[1],
                    h->stage_in, h->stage_out, h->dS, h->partials, h->counter};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h->hS) cudaFreeHost(h->hS);
    if (h->cg_exec) cudaGraphExecDestroy(h->cg_exec);
    if (h->ev_sync) cudaEventDestroy(h->ev_sync);
    if (h->ev_a) cudaEventDestroy(h->ev_a);
    if (h->ev_b) cudaEventDestroy(h->ev_b);
    if (h->ev_c0) cudaEventDestroy(h->ev_c0);
    if (h->ev_c1) cudaEventDestroy(h->ev_c1);
    if (h->st) cudaStreamDestroy(h->st);
    delete h;
}

constexpr int kMarchTY = 16;

MarchGeom march_geom(int nx, int ny, int H) {
    MarchGeom g;
    g.nstrips = (nx + (32 - 2 * H) - 1) / (32 - 2 * H);
    g.TY = kMarchTY;
    g.nchunks = (ny + g.TY - 1) / g.TY;
    return g;
}
int march_grid(const MarchGeom& g) {     // one work item per warp
    const long long items = (long long)g.nstrips * g.nchunks;
    return (int)std::max<long long>(1, (items + kMarchThreads / 32 - 1) / (kMarchThreads / 32));
}
long long march_grid_bound(const gpcg_problem* h) {
    return std::max(march_grid(h->mg1), march_grid(h->mg2));
}

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D tensor map over an internal (pitched) stencil array; out-of-grid elements read as 0
int make_map(gpcg_problem* h, CUtensorMap* m, const void* ptr, bool u8, int bw, int bh) {
    auto enc = tma_encode_fn();
    if (!enc) return set_err(GPCG_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)h->cols, (cuuint64_t)h->rows};
    const cuuint64_t strides[1] = {(cuuint64_t)h->pitch * (u8 ? 1 : 8)};
    const cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                     const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(GPCG_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return GPCG_OK;
}

template <class K>
int set_smem(K kernel, int bytes) {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    return GPCG_OK;
}

// Build the TMA tile path for a broadcast-face stencil handle (C0/C2/C3 family).
int setup_tile(gpcg_problem* h) {
    int rc;
    for (int k = 0; k < 2; ++k) {
        if ((rc = make_map(h, &h->tmY[k], h->Y[k], false, TBW, TBH))) return rc;
        if ((rc = make_map(h, &h->tmG[k], h->G[k], false, TBW, TBH))) return rc;
        if ((rc = make_map(h, &h->tmRho[k], h->Rho[k], false, TBW, TBH))) return rc;
        if ((rc = make_map(h, &h->tmP[k], h->Q[k], false, TBW, TBH))) return rc;
        if ((rc = make_map(h, &h->tmM[k], h->M[k], true, MBW, TBH))) return rc;
    }
    if ((rc = make_map(h, &h->tmW, h->W, false, TBW, TBH))) return rc;
    if ((rc = make_map(h, &h->tmWc, h->W, false, TOX, TOY))) return rc;
    if ((rc = make_map(h, &h->tmB, h->b, false, TBW, TBH))) return rc;
    if ((rc = make_map(h, &h->tmL, h->l, false, TBW, TBH))) return rc;
    if ((rc = make_map(h, &h->tmU, h->u, false, TBW, TBH))) return rc;
    if ((rc = make_map(h, &h->tmMcg, h->Mcg, true, MBW, TBH))) return rc;
    if ((rc = make_map(h, &h->tmStage, h->stage_in, false, TBW, TBH))) return rc;
    h->tg = TileGeom{h->cols, h->rows, h->pitch, (h->cols + TOX - 1) / TOX, (h->rows + TOY - 1) / TOY};
    const int ntiles = h->tg.ntx * h->tg.nty;
    if ((rc = set_smem(k3_cg_iter<2>, CgStage<2>::kSmem))) return rc;
    if ((rc = set_smem(k3_accept<true>, AccStage<true>::kSmem))) return rc;
    if ((rc = set_smem(k3_accept<false>, AccStage<false>::kSmem))) return rc;
    if ((rc = set_smem(k3_search<true, true>, SrchStage<true, true>::kSmem))) return rc;
    if ((rc = set_smem(k3_search<true, false>, SrchStage<true, false>::kSmem))) return rc;
    if ((rc = set_smem(k3_search<false, true>, SrchStage<false, true>::kSmem))) return rc;
    if ((rc = set_smem(k3_search<false, false>, SrchStage<false, false>::kSmem))) return rc;
    auto resident = [&](auto kernel, int smem) {
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kTileThreads, smem);
        return std::max(1, nb) * h->sms;
    };
    h->grid_t_cg = std::min(ntiles, resident(k3_cg_iter<2>, CgStage<2>::kSmem));
    h->grid_t_acc = std::min(ntiles, h->sb ? resident(k3_accept<true>, AccStage<true>::kSmem)
                                            : resident(k3_accept<false>, AccStage<false>::kSmem));
    h->grid_t_srch = std::min(ntiles, h->sb ? resident(k3_search<true, true>, SrchStage<true, true>::kSmem)
                                             : resident(k3_search<false, true>, SrchStage<false, true>::kSmem));
    h->tile = true;
    return GPCG_OK;
}

const CUtensorMap* map_of(gpcg_problem* h, const void* p) {
    for (int k = 0; k < 2; ++k) {
        if (p == h->Y[k]) return &h->tmY[k];
        if (p == h->G[k]) return &h->tmG[k];
        if (p == h->M[k]) return &h->tmM[k];
    }
    if (p == h->W) return &h->tmW;
    if (p == h->stage_in) return &h->tmStage;
    return nullptr;
}

// common part of create: device, streams, vectors, bounds, validation
int create_common(gpcg_problem* h, void* stream, const double* b, const double* l, const double* u) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(GPCG_ECUDA, "no CUDA device (the library has no CPU fallback)");
    }
    CK(cudaGetDevice(&h->dev));
    CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->dev));
    h->user = (cudaStream_t)stream;
    CK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&h->ev_sync, cudaEventDisableTiming));
    CK(cudaEventCreate(&h->ev_a));
    CK(cudaEventCreate(&h->ev_b));
    CK(cudaEventCreate(&h->ev_c0));
    CK(cudaEventCreate(&h->ev_c1));
    CK(cudaEventRecord(h->ev_sync, h->user));
    CK(cudaStreamWaitEvent(h->st, h->ev_sync, 0));
    const size_t nb = (size_t)h->nalloc * sizeof(double);
    CK(cudaMalloc(&h->b, nb));
    CK(cudaMalloc(&h->l, nb));
    CK(cudaMalloc(&h->u, nb));
    for (int k = 0; k < 2; ++k) {
        CK(cudaMalloc(&h->Y[k], nb));
        CK(cudaMalloc(&h->G[k], nb));
        CK(cudaMalloc(&h->M[k], (size_t)h->nalloc));
        CK(cudaMemsetAsync(h->M[k], 0, (size_t)h->nalloc, h->st));
        if (k == 0) {
            CK(cudaMalloc(&h->Mcg, (size_t)h->nalloc));
            CK(cudaMemsetAsync(h->Mcg, 0, (size_t)h->nalloc, h->st));
        }
        CK(cudaMalloc(&h->Rho[k], nb));
        CK(cudaMalloc(&h->Q[k], nb));
        CK(cudaMalloc(&h->S2[k], nb));
    }
    CK(cudaMalloc(&h->W, nb));
    CK(cudaMalloc(&h->P, nb));
    CK(cudaMalloc(&h->stage_in, nb));
    CK(cudaMalloc(&h->stage_out, nb));
    CK(cudaMalloc(&h->dS, sizeof(Scal)));
    CK(cudaMemsetAsync(h->dS, 0, sizeof(Scal), h->st));
    CK(cudaMallocHost(&h->hS, sizeof(Scal)));
    // partial sums of the largest grid any kernel of this handle uses (grid-stride
    // generic kernels are capped at 16 blocks/SM; march grids are one warp per item)
    long long gmax = (long long)h->sms * 16;
    if (!h->is_csr) gmax = std::max<long long>(gmax, march_grid_bound(h));
    CK(cudaMalloc(&h->partials, (size_t)kMaxSums * gmax * sizeof(double)));
    CK(cudaMalloc(&h->counter, sizeof(unsigned int)));
    CK(cudaMemsetAsync(h->counter, 0, sizeof(unsigned int), h->st));
    int rc;
    for (double* v : {h->b, h->l, h->u, h->Y[0], h->Y[1], h->G[0], h->G[1], h->W, h->P, h->Rho[0], h->Rho[1],
                      h->Q[0], h->Q[1], h->S2[0], h->S2[1], h->stage_in, h->stage_out})
        CK(cudaMemsetAsync(v, 0, nb, h->st));        // padding columns stay 0
    if ((rc = upload_vec(h, h->b, b))) return rc;
    if ((rc = upload_vec(h, h->l, l))) return rc;
    if ((rc = upload_vec(h, h->u, u))) return rc;
    // validation: l <= u, no NaN / inf in b, l != +inf, u != -inf; constant bounds?
    const int g = std::max(1, std::min((h->n + kThreads - 1) / kThreads, h->sms * 4));
    k_check_inputs<<<g, kThreads, 0, h->st>>>(h->cols, h->rows, h->pitch, h->b, h->l, h->u, h->dS, h->red());
    CKLAUNCH();
    if ((rc = sync_scal(h))) return rc;
    if (h->hS->r0 != 0.0)
        return set_err(GPCG_EINVAL, "%.0f entries violate l <= u (or NaN/inf in b, l = +inf, u = -inf)",
                       h->hS->r0);
    h->sb = (h->hS->r1 == 0.0);
    double lu[2];
    CK(cudaMemcpy(&lu[0], h->l, sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&lu[1], h->u, sizeof(double), cudaMemcpyDeviceToHost));
    h->bounds = Bounds{h->l, h->u, lu[0], lu[1]};
    h->prm = gpcg_params_default();
    return GPCG_OK;
}

// ---------------------------------------------------------------- launches
int launch_accept(gpcg_problem* h, const double* y_in, const double* dir, double sgn,
                  const unsigned char* mask_prev, double* y_out, double* g_out, unsigned char* m_out) {
    if (h->tile && (h->tile_mask & 1)) {   // TMA tile path
        const CUtensorMap* my = map_of(h, y_in);
        const CUtensorMap* md = dir ? map_of(h, dir) : my;
        const CUtensorMap* mp = mask_prev ? map_of(h, mask_prev) : &h->tmM[0];
        if (!my || !md || !mp) return set_err(GPCG_ECUDA, "internal: no tensor map for an accept operand");
        if (h->sb)
            k3_accept<true><<<h->grid_t_acc, kTileThreads, AccStage<true>::kSmem, h->st>>>(
                h->sop, h->tg, h->bounds, *my, *md, h->tmB, h->tmL, h->tmU, *mp, dir ? 1 : 0, sgn,
                mask_prev ? 1 : 0, y_out, g_out, m_out, h->dS, h->red());
        else
            k3_accept<false><<<h->grid_t_acc, kTileThreads, AccStage<false>::kSmem, h->st>>>(
                h->sop, h->tg, h->bounds, *my, *md, h->tmB, h->tmL, h->tmU, *mp, dir ? 1 : 0, sgn,
                mask_prev ? 1 : 0, y_out, g_out, m_out, h->dS, h->red());
        h->launches++;
        CKLAUNCH();
        return GPCG_OK;
    }
    if (!h->is_csr && !h->generic) {   // stencil: accept + regrad + mask + counts + next Cauchy step in one sweep
        auto go = [&](auto sbt, auto bct) {
            constexpr bool SB = decltype(sbt)::value, BC = decltype(bct)::value;
            k2_accept<SB, BC><<<h->grid_m2, kMarchThreads, 0, h->st>>>(h->sop, h->mg2, h->bounds, y_in, dir, sgn,
                                                                       h->b, mask_prev, y_out, g_out, m_out, h->dS,
                                                                       h->red());
        };
        if (h->sb) { if (h->bc) go(std::true_type(), std::true_type()); else go(std::true_type(), std::false_type()); }
        else { if (h->bc) go(std::false_type(), std::true_type()); else go(std::false_type(), std::false_type()); }
        h->launches++;
        CKLAUNCH();
        return GPCG_OK;
    }
    with_op(h, [&](auto& op, auto sbt) {
        using Op = std::decay_t<decltype(op)>;
        constexpr bool SB = decltype(sbt)::value;
        k_accept<Op, SB><<<h->grid, kThreads, 0, h->st>>>(op, h->bounds, y_in, dir, sgn, h->b, mask_prev,
                                                          y_out, g_out, m_out, h->dS, h->red());
    });
    h->launches++;
    CKLAUNCH();
    return GPCG_OK;
}

int launch_cauchy(gpcg_problem* h, const double* y, const double* g) {
    if (!h->is_csr && !h->generic) return GPCG_OK;     // computed by the preceding k2_accept sweep
    with_op(h, [&](auto& op, auto sbt) {
        using Op = std::decay_t<decltype(op)>;
        constexpr bool SB = decltype(sbt)::value;
        k_cauchy<Op, SB><<<h->grid, kThreads, 0, h->st>>>(op, h->bounds, y, g, h->dS, h->red());
    });
    h->launches++;
    CKLAUNCH();
    return GPCG_OK;
}

// step sizes per projected-search sweep: the first sweep evaluates search_k
// (2 or 8 instantiated), later sweeps 8
int first_k(const gpcg_problem* h) { return h->prm.search_k <= 2 ? 2 : 8; }

int launch_search(gpcg_problem* h, const double* y, const double* g, const double* dir, double sgn,
                  int use_alpha0, int h0, int K) {
    const double mu = h->prm.mu;
    if (h->tile && (h->tile_mask & 2) && K == 2) {   // TMA tile path (first sweep); retries use the column march
        const CUtensorMap* my = map_of(h, y);
        const CUtensorMap* md = map_of(h, dir);
        const CUtensorMap* mg = map_of(h, g);
        if (!my || !md || !mg) return set_err(GPCG_ECUDA, "internal: no tensor map for a search operand");
        const bool dg = (dir == g);
        auto go = [&](auto sbt, auto dgt) {
            constexpr bool SB = decltype(sbt)::value, DG = decltype(dgt)::value;
            k3_search<SB, DG><<<h->grid_t_srch, kTileThreads, SrchStage<SB, DG>::kSmem, h->st>>>(
                h->sop, h->tg, h->bounds, *my, *md, *mg, h->tmL, h->tmU, sgn, use_alpha0, h0, mu, h->dS, h->red());
        };
        if (h->sb) { if (dg) go(std::true_type(), std::true_type()); else go(std::true_type(), std::false_type()); }
        else { if (dg) go(std::false_type(), std::true_type()); else go(std::false_type(), std::false_type()); }
        h->launches++;
        CKLAUNCH();
        return GPCG_OK;
    }
    if (!h->is_csr && !h->generic) {
        const bool dg = (dir == g);
        auto go = [&](auto sbt, auto bct, auto kt, auto dgt) {
            constexpr bool SB = decltype(sbt)::value, BC = decltype(bct)::value, DG = decltype(dgt)::value;
            constexpr int KK = decltype(kt)::value;
            k2_search<SB, BC, KK, DG><<<h->grid_m1, kMarchThreads, 0, h->st>>>(
                h->sop, h->mg1, h->bounds, y, g, dir, sgn, use_alpha0, h0, mu, h->dS, h->red());
        };
        auto byk = [&](auto sbt, auto bct, auto dgt) {
            if (K == 2) go(sbt, bct, std::integral_constant<int, 2>(), dgt);
            else go(sbt, bct, std::integral_constant<int, 8>(), dgt);
        };
        auto bydg = [&](auto sbt, auto bct) {
            if (dg) byk(sbt, bct, std::true_type()); else byk(sbt, bct, std::false_type());
        };
        auto bybc = [&](auto sbt) {
            if (h->bc) bydg(sbt, std::true_type()); else bydg(sbt, std::false_type());
        };
        if (h->sb) bybc(std::true_type()); else bybc(std::false_type());
        h->launches++;
        CKLAUNCH();
        return GPCG_OK;
    }
    with_op(h, [&](auto& op, auto sbt) {
        using Op = std::decay_t<decltype(op)>;
        constexpr bool SB = decltype(sbt)::value;
        if (K == 2)
            k_search<Op, SB, 2><<<h->grid, kThreads, 0, h->st>>>(op, h->bounds, y, g, dir, sgn, use_alpha0,
                                                                 h0, mu, h->dS, h->red());
        else
            k_search<Op, SB, 8><<<h->grid, kThreads, 0, h->st>>>(op, h->bounds, y, g, dir, sgn, use_alpha0,
                                                                 h0, mu, h->dS, h->red());
    });
    h->launches++;
    CKLAUNCH();
    return GPCG_OK;
}

// one projected search + accept:  y' = P[y + alpha sgn dir], g' = A y' - b.
// Host loops over batches of K step sizes until one is accepted.  Returns
// GPCG_OK with *accepted_h >= 0, or GPCG_ESEARCH.
int search_and_accept(gpcg_problem* h, int cur, const double* dir, double sgn, int use_alpha0,
                      int* accepted_h) {
    const int nxt = cur ^ 1;
    int rc;
    for (int h0 = 0, K = first_k(h); h0 < h->prm.max_halvings; h0 += K, K = 8) {
        if ((rc = launch_search(h, h->Y[cur], h->G[cur], dir, sgn, use_alpha0, h0, K))) return rc;
        if ((rc = launch_accept(h, h->Y[cur], dir, sgn, h->M[cur], h->Y[nxt], h->G[nxt], h->M[nxt])))
            return rc;
        if ((rc = sync_scal(h))) return rc;
        // the search is skipped (s_h = -1) when the Cauchy step of y has <d, A d> <= 0;
        // after an accepted step cauchy_ok already describes the NEW point (fused sweep)
        if (h->hS->s_h < 0 && use_alpha0 && !h->hS->cauchy_ok)
            return set_err(GPCG_ENOTSPD, "<d, A d> = %g <= 0 in the Cauchy step: A is not SPD", h->hS->dAd);
        if (h->hS->s_h >= 0) {
            if (h->hS->s_h >= h->prm.max_halvings) break;
            *accepted_h = h->hS->s_h;
            return GPCG_OK;
        }
    }
    return set_err(GPCG_ESEARCH, "projected search: no sufficient decrease within %lld halvings",
                   (long long)h->prm.max_halvings);
}

int build_cg_graph(gpcg_problem* h, int chunk) {
    if (h->cg_exec && h->cg_exec_chunk == chunk) return GPCG_OK;
    if (h->cg_exec) {
        cudaGraphExecDestroy(h->cg_exec);
        h->cg_exec = nullptr;
    }
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < chunk; ++i) {
        const int a = i & 1, bb = a ^ 1;
        if (h->tile && (h->tile_mask & 4)) {
            k3_cg_iter<2><<<h->grid_t_cg, kTileThreads, CgStage<2>::kSmem, h->st>>>(
                h->sop, h->tg, h->tmRho[a], h->tmP[a], h->tmWc, h->tmMcg, h->Rho[bb], h->Q[bb], h->W, h->dS,
                h->red());
            continue;
        }
        if (!h->is_csr && !h->generic) {   // stencil: rho, p ping-pong (p in Q[]), w in place
            if (h->bc)
                k2_cg_iter<true><<<h->grid_m2, kMarchThreads, 0, h->st>>>(h->sop, h->mg2, h->Mcg, h->Rho[a], h->Q[a],
                                                                          h->Rho[bb], h->Q[bb], h->W, h->dS, h->red());
            else
                k2_cg_iter<false><<<h->grid_m2, kMarchThreads, 0, h->st>>>(h->sop, h->mg2, h->Mcg, h->Rho[a], h->Q[a],
                                                                           h->Rho[bb], h->Q[bb], h->W, h->dS, h->red());
            continue;
        }
        with_op_only(h, [&](auto& op) {
            using Op = std::decay_t<decltype(op)>;
            k_cg_iter<Op><<<h->grid, kThreads, 0, h->st>>>(op, h->Mcg, h->Rho[a], h->Q[a], h->S2[a],
                                                           h->Rho[bb], h->Q[bb], h->S2[bb], h->P, h->W,
                                                           h->dS, h->red());
        });
    }
    cudaError_t e = cudaStreamEndCapture(h->st, &graph);
    if (e != cudaSuccess) return set_err(GPCG_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&h->cg_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return set_err(GPCG_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    h->cg_exec_chunk = chunk;
    return GPCG_OK;
}

// CG on the free set of M[cur].  On return W holds w_{j_k}.
int run_cg(gpcg_problem* h, int cur, long long m, double eta2, long long cap, long long* iters) {
    int rc;
    if (!h->is_csr && !h->generic) {
        if (h->bc)
            k2_cg_init<true><<<h->grid_m1, kMarchThreads, 0, h->st>>>(h->sop, h->mg1, h->G[cur], h->M[cur], h->Mcg,
                                                                      h->Rho[0], h->Q[0], h->W, eta2, cap, h->dS,
                                                                      h->red());
        else
            k2_cg_init<false><<<h->grid_m1, kMarchThreads, 0, h->st>>>(h->sop, h->mg1, h->G[cur], h->M[cur], h->Mcg,
                                                                       h->Rho[0], h->Q[0], h->W, eta2, cap, h->dS,
                                                                       h->red());
    } else with_op_only(h, [&](auto& op) {
        using Op = std::decay_t<decltype(op)>;
        k_cg_init<Op><<<h->grid, kThreads, 0, h->st>>>(op, h->G[cur], h->M[cur], h->Mcg, h->Rho[0], h->Q[0], h->S2[0],
                                                       h->Rho[1], h->Q[1], h->S2[1], h->P, h->W, eta2, cap,
                                                       h->dS, h->red());
    });
    h->launches++;
    CKLAUNCH();
    const int chunk = std::max(2, (h->prm.cg_chunk + 1) & ~1);
    if ((rc = build_cg_graph(h, chunk))) return rc;
    for (;;) {
        CK(cudaEventRecord(h->ev_c0, h->st));
        CK(cudaGraphLaunch(h->cg_exec, h->st));
        CK(cudaEventRecord(h->ev_c1, h->st));
        h->launches += chunk;
        if ((rc = sync_scal(h))) return rc;
        if (h->hS->cg_done) break;
        // every iteration of this chunk was real: steady-state timing sample
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev_c0, h->ev_c1));
        h->t_cg_timed_ms += ms;
        h->cg_iters_timed += chunk;
        h->cg_free_iters_timed += chunk * m;
    }
    *iters = h->hS->cg_it;
    if (h->hS->cg_reason == CG_NOTSPD)
        return set_err(GPCG_ENOTSPD, "CG breakdown: <p, A_k p> <= 0 at iteration %lld (A not SPD)",
                       (long long)h->hS->cg_it);
    return GPCG_OK;
}

}  // namespace

// ============================================================================
// ABI
// ============================================================================
extern "C" {

gpcg_params gpcg_params_default(void) {
    gpcg_params p;
    p.mu = 0.1;
    p.eta1 = 0.1;
    p.eta2 = 0.05;
    p.eta2_shrink = 0.1;
    p.eta2_floor = 1e-12;
    p.gp_cap = 100;
    p.refine_cap = 30;
    p.max_halvings = 50;
    p.cg_cap = 0;
    p.search_k = 2;
    p.cg_chunk = 32;
    return p;
}

const char* gpcg_last_error(void) { return g_err.c_str(); }

int64_t gpcg_size(const gpcg_problem* h) { return h ? h->n : -1; }

int gpcg_create_stencil2d(gpcg_problem** out, void* cuda_stream, int64_t nx, int64_t ny, const double* wx,
                          int64_t wx_ld, const double* wy, int64_t wy_ld, const double* shift,
                          const double* b, const double* l, const double* u, double c) {
    g_err.clear();
    if (!out) return set_err(GPCG_EINVAL, "out is NULL");
    *out = nullptr;
    if (nx <= 0 || ny <= 0 || nx * ny >= (1LL << 31))
        return set_err(GPCG_EINVAL, "grid %lld x %lld out of range (need 0 < n < 2^31)", (long long)nx,
                       (long long)ny);
    if (!wx || !wy || !b || !l || !u) return set_err(GPCG_EINVAL, "NULL array argument");
    if ((wx_ld != 0 && wx_ld < nx + 1) || (wy_ld != 0 && wy_ld < nx) || wx_ld < 0 || wy_ld < 0)
        return set_err(GPCG_EINVAL, "bad leading dimension (wx_ld %lld, wy_ld %lld)", (long long)wx_ld,
                       (long long)wy_ld);
    if (!std::isfinite(c)) return set_err(GPCG_EINVAL, "c is not finite");
    gpcg_problem* h = new gpcg_problem();
    h->n = (int)(nx * ny);
    h->rows = (int)ny;
    h->cols = (int)nx;
    h->pitch = (int)((nx + 31) / 32 * 32);
    h->nalloc = (long long)h->pitch * ny;
    if (h->nalloc >= (1LL << 31)) { delete h; return set_err(GPCG_EINVAL, "pitched grid too large"); }
    h->is_csr = false;
    h->generic = getenv("GPCG_GENERIC") != nullptr && getenv("GPCG_GENERIC")[0] == '1';
    h->mg1 = march_geom((int)nx, (int)ny, 1);
    h->mg2 = march_geom((int)nx, (int)ny, 2);
    h->grid_m1 = march_grid(h->mg1);
    h->grid_m2 = march_grid(h->mg2);
    int rc = create_common(h, cuda_stream, b, l, u);
    if (rc) { free_all(h); return rc; }
    h->c = c;
    const size_t wxn = (size_t)(wx_ld ? wx_ld * (ny - 1) + nx + 1 : nx + 1);
    const size_t wyn = (size_t)(wy_ld ? wy_ld * ny + nx : nx);
    auto fail = [&](int r) { free_all(h); return r; };
    if (cudaMalloc(&h->wx, wxn * sizeof(double)) != cudaSuccess) return fail(set_err(GPCG_ENOMEM, "wx"));
    if (cudaMalloc(&h->wy, wyn * sizeof(double)) != cudaSuccess) return fail(set_err(GPCG_ENOMEM, "wy"));
    if ((rc = upload(h, h->wx, wx, wxn))) return fail(rc);
    if ((rc = upload(h, h->wy, wy, wyn))) return fail(rc);
    double bad = 0.0, t = 0.0;
    if ((rc = count_nonfinite(h, h->wx, (long long)wxn, &t))) return fail(rc);
    bad += t;
    if ((rc = count_nonfinite(h, h->wy, (long long)wyn, &t))) return fail(rc);
    bad += t;
    if (shift) {
        if (cudaMalloc(&h->shift, (size_t)h->nalloc * sizeof(double)) != cudaSuccess)
            return fail(set_err(GPCG_ENOMEM, "shift"));
        if (cudaMemsetAsync(h->shift, 0, (size_t)h->nalloc * sizeof(double), h->st) != cudaSuccess)
            return fail(set_err(GPCG_ECUDA, "memset shift"));
        if ((rc = upload_vec(h, h->shift, shift))) return fail(rc);
        if ((rc = count_nonfinite(h, h->shift, h->nalloc, &t))) return fail(rc);
        bad += t;
    }
    if (bad != 0.0) return fail(set_err(GPCG_EINVAL, "%.0f non-finite stencil weights", bad));
    h->is_csr = false;
    h->sop = StencilOp{(int)nx, (int)ny, h->pitch, h->wx, h->wy, h->shift, (long long)wx_ld, (long long)wy_ld};
    h->bc = (wx_ld == 0 && wy_ld == 0 && shift == nullptr);
    {
        const char* e = getenv("GPCG_TILE");
        if (e && *e) h->tile_mask = atoi(e) & 7;
        const bool want_tile = h->bc && !h->generic && h->tile_mask != 0;
        if (want_tile && (rc = setup_tile(h))) return fail(rc);
    }
    h->nnz = 5 * (long long)h->n - 2 * nx - 2 * ny;
    h->grid = std::max(1, std::min(units(h), h->sms * 16));
    if ((rc = leave(h))) return fail(rc);
    *out = h;
    return GPCG_OK;
}

int gpcg_create_csr(gpcg_problem** out, void* cuda_stream, int64_t n, const int64_t* row_ptr,
                    const int32_t* col, const double* val, const double* b, const double* l, const double* u,
                    double c) {
    g_err.clear();
    if (!out) return set_err(GPCG_EINVAL, "out is NULL");
    *out = nullptr;
    if (n <= 0 || n >= (1LL << 31)) return set_err(GPCG_EINVAL, "n = %lld out of range", (long long)n);
    if (!row_ptr || !col || !val || !b || !l || !u) return set_err(GPCG_EINVAL, "NULL array argument");
    if (!std::isfinite(c)) return set_err(GPCG_EINVAL, "c is not finite");
    gpcg_problem* h = new gpcg_problem();
    h->n = (int)n;
    h->rows = 1;
    h->cols = (int)n;
    h->pitch = (int)n;
    h->nalloc = n;
    h->is_csr = true;
    auto fail = [&](int r) { free_all(h); return r; };
    int rc = create_common(h, cuda_stream, b, l, u);
    if (rc) return fail(rc);
    h->c = c;
    // row_ptr: need nnz on the host for the copies
    long long rp_end = 0, rp0 = 0;
    if (is_device_ptr(row_ptr)) {
        if (cudaMemcpy(&rp_end, row_ptr + n, sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(&rp0, row_ptr, sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(set_err(GPCG_ECUDA, "reading row_ptr"));
    } else {
        rp_end = row_ptr[n];
        rp0 = row_ptr[0];
    }
    if (rp0 != 0 || rp_end < n || rp_end >= (1LL << 40))
        return fail(set_err(GPCG_EINVAL, "row_ptr[0] = %lld, row_ptr[n] = %lld invalid", rp0, rp_end));
    h->nnz = rp_end;
    if (cudaMalloc(&h->rp, (size_t)(n + 1) * sizeof(long long)) != cudaSuccess ||
        cudaMalloc(&h->ci, (size_t)rp_end * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&h->val, (size_t)rp_end * sizeof(double)) != cudaSuccess)
        return fail(set_err(GPCG_ENOMEM, "CSR arrays (nnz = %lld)", rp_end));
    if ((rc = upload_bytes(h, h->rp, row_ptr, (size_t)(n + 1) * sizeof(long long)))) return fail(rc);
    if ((rc = upload_bytes(h, h->ci, col, (size_t)rp_end * sizeof(int)))) return fail(rc);
    if ((rc = upload(h, h->val, val, (size_t)rp_end))) return fail(rc);
    double t = 0.0;
    if ((rc = count_nonfinite(h, h->val, rp_end, &t))) return fail(rc);
    if (t != 0.0) return fail(set_err(GPCG_EINVAL, "%.0f non-finite CSR values", t));
    h->is_csr = true;
    h->cop = CsrOp{h->n, h->rp, h->ci, h->val};
    h->grid = std::max(1, std::min(units(h), h->sms * 16));
    if ((rc = leave(h))) return fail(rc);
    *out = h;
    return GPCG_OK;
}

int gpcg_set_params(gpcg_problem* h, const gpcg_params* p) {
    g_err.clear();
    if (!h || !p) return set_err(GPCG_EINVAL, "NULL argument");
    if (!(p->mu > 0.0 && p->mu < 0.5)) return set_err(GPCG_EINVAL, "mu must lie in (0, 1/2)");
    if (!(p->eta1 > 0.0 && p->eta1 < 1.0) || !(p->eta2 > 0.0 && p->eta2 < 1.0))
        return set_err(GPCG_EINVAL, "eta1, eta2 must lie in (0, 1)");
    if (!(p->eta2_shrink > 0.0 && p->eta2_shrink < 1.0) || !(p->eta2_floor > 0.0))
        return set_err(GPCG_EINVAL, "eta2_shrink in (0,1), eta2_floor > 0 required");
    if (p->gp_cap < 1 || p->refine_cap < 1 || p->max_halvings < 1 || p->max_halvings > 1000 ||
        p->cg_cap < 0 || p->search_k < 1 || p->search_k > kMaxK || p->cg_chunk < 1 || p->cg_chunk > 4096)
        return set_err(GPCG_EINVAL, "integer parameter out of range");
    const int old_chunk = h->prm.cg_chunk;
    h->prm = *p;
    if (old_chunk != p->cg_chunk && h->cg_exec) {
        cudaGraphExecDestroy(h->cg_exec);
        h->cg_exec = nullptr;
    }
    return GPCG_OK;
}

void gpcg_destroy(gpcg_problem* h) { free_all(h); }

int gpcg_project(gpcg_problem* h, const double* x, double* px, double* pg_norm2, int64_t* n_active,
                 int64_t* n_active_nonbinding) {
    g_err.clear();
    if (!h || !x || !px) return set_err(GPCG_EINVAL, "NULL argument");
    int rc;
    if ((rc = enter(h))) return rc;
    if ((rc = upload_vec(h, h->stage_in, x))) return rc;
    if ((rc = launch_accept(h, h->stage_in, nullptr, 0.0, nullptr, h->Y[0], h->G[0], h->M[0]))) return rc;
    if ((rc = download_vec(h, px, h->Y[0]))) return rc;
    if ((rc = sync_scal(h))) return rc;
    h->free_mask = 0;
    if (pg_norm2) *pg_norm2 = h->hS->pg2;
    if (n_active) *n_active = (int64_t)h->hS->n_active;
    if (n_active_nonbinding) *n_active_nonbinding = (int64_t)h->hS->n_nonbinding;
    return leave(h);
}

int gpcg_hessvec(gpcg_problem* h, const double* v, double* y, int reduced) {
    g_err.clear();
    if (!h || !v || !y) return set_err(GPCG_EINVAL, "NULL argument");
    if (v == y) return set_err(GPCG_EINVAL, "v and y must not alias");
    if (reduced && h->free_mask < 0)
        return set_err(GPCG_ESTATE, "reduced hessvec needs a free set: call gpcg_project or gpcg_solve first");
    int rc;
    if ((rc = enter(h))) return rc;
    // direct device access only when the layout is contiguous (CSR, or nx a multiple of 32)
    const bool contiguous = (h->pitch == h->cols);
    const bool vdev = is_device_ptr(v) && contiguous, ydev = is_device_ptr(y) && contiguous;
    const double* vin = v;
    if (!vdev) {
        if ((rc = upload_vec(h, h->stage_in, v))) return rc;
        vin = h->stage_in;
    }
    double* yout = ydev ? y : h->stage_out;
    const unsigned char* mask = reduced ? h->M[h->free_mask] : nullptr;
    with_op_only(h, [&](auto& op) {
        using Op = std::decay_t<decltype(op)>;
        if (reduced)
            k_hessvec<Op, true><<<h->grid, kThreads, 0, h->st>>>(op, vin, yout, mask);
        else
            k_hessvec<Op, false><<<h->grid, kThreads, 0, h->st>>>(op, vin, yout, mask);
    });
    h->launches++;
    CKLAUNCH();
    if (!ydev) {
        if ((rc = download_vec(h, y, h->stage_out))) return rc;
        if (!is_device_ptr(y)) CK(cudaStreamSynchronize(h->st));
    }
    return leave(h);
}

int gpcg_objective(gpcg_problem* h, const double* x, double* q) {
    g_err.clear();
    if (!h || !x || !q) return set_err(GPCG_EINVAL, "NULL argument");
    int rc;
    if ((rc = enter(h))) return rc;
    if ((rc = upload_vec(h, h->stage_in, x))) return rc;
    with_op_only(h, [&](auto& op) {
        using Op = std::decay_t<decltype(op)>;
        k_objective<Op><<<h->grid, kThreads, 0, h->st>>>(op, h->stage_in, h->b, h->dS, h->red());
    });
    h->launches++;
    CKLAUNCH();
    if ((rc = sync_scal(h))) return rc;
    *q = 0.5 * h->hS->r0 - h->hS->r1 + h->c;
    return leave(h);
}

// Algorithm GPCG, same steps as the oracle.
int gpcg_solve(gpcg_problem* h, const double* x0, double tol, int64_t max_it, double* x_out,
               gpcg_stats* stats) {
    g_err.clear();
    if (!h || !x0 || !x_out) return set_err(GPCG_EINVAL, "NULL argument");
    if (!(tol != 0.0) || !std::isfinite(tol)) return set_err(GPCG_EINVAL, "tol must be finite and nonzero");
    if (max_it < 0) return set_err(GPCG_EINVAL, "max_it < 0");
    const auto t_start = std::chrono::steady_clock::now();
    gpcg_stats st;
    memset(&st, 0, sizeof st);
    h->launches = 0;
    h->cg_iters_timed = h->cg_free_iters_timed = 0;
    h->t_cg_timed_ms = 0.0;
    int rc;
    if ((rc = enter(h))) return rc;
    const gpcg_params& prm = h->prm;
    float t_cg = 0.f, t_gp = 0.f, ms = 0.f;
    int status = GPCG_NOT_CONVERGED;
    int cur = 0;
    double tau = 0.0;
    const Scal& S = *h->hS;

    // Setup: x <- P[x0], g <- A x - b
    if ((rc = upload_vec(h, h->stage_in, x0))) return rc;
    if ((rc = launch_accept(h, h->stage_in, nullptr, 0.0, nullptr, h->Y[0], h->G[0], h->M[0]))) return rc;
    if ((rc = sync_scal(h))) return rc;
    st.full_spmvs++;
    st.g0_norm = std::sqrt(S.g2);
    tau = tol > 0.0 ? tol : -tol * st.g0_norm;
    st.tau = tau;
    if (std::sqrt(S.pg2) <= tau) {
        status = GPCG_OK;
    } else {
        for (int64_t k = 0; k < max_it && status == GPCG_NOT_CONVERGED; ++k) {
            st.outer_iters = k + 1;
            // ---- gradient projection phase, y_0 = x_k ------------
            CK(cudaEventRecord(h->ev_a, h->st));
            long long j = 0;
            double maxdec = 0.0;
            bool conv = false;
            for (;;) {
                if (std::sqrt(S.pg2) <= tau) { conv = true; break; }
                if ((rc = launch_cauchy(h, h->Y[cur], h->G[cur]))) goto fail;
                st.full_spmvs++;
                int hacc = -1;
                // direction -grad q (Eq. next-y); trial points equal those of the
                // -grad_Omega q reading for feasible y (reading R8)
                if ((rc = search_and_accept(h, cur, h->G[cur], -1.0, 1, &hacc))) goto fail;
                st.full_spmvs += 2;
                cur ^= 1;
                ++j;
                st.gp_iters++;
                const double dec = -S.s_delta;                      // q(y_{j-1}) - q(y_j)
                if (trace_on())
                    fprintf(stderr, "[gpcg] k=%lld GP j=%lld h=%d alpha=%.3e dec=%.3e |A|=%.0f changed=%.0f pg=%.3e t=%.2fms\n",
                            (long long)k, j, S.s_h, S.s_alpha, dec, S.n_active, S.n_changed, std::sqrt(S.pg2),
                            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
                const bool stop = (S.n_changed == 0.0) ||           // Eq. pgstop1 (index sets, R9)
                                  (j >= 2 && dec <= prm.eta1 * maxdec) ||   // Eq. pgstop2 (R10)
                                  (j >= prm.gp_cap);
                if (dec > maxdec) maxdec = dec;
                if (stop) break;
            }
            CK(cudaEventRecord(h->ev_b, h->st));
            CK(cudaEventSynchronize(h->ev_b));
            CK(cudaEventElapsedTime(&ms, h->ev_a, h->ev_b));
            t_gp += ms;
            if (conv || std::sqrt(S.pg2) <= tau) { status = GPCG_OK; break; }

            // ---- CG phase with eta2 refinement -------------------
            double eta2 = prm.eta2;
            for (int64_t rep = 0; rep < prm.refine_cap; ++rep) {
                const long long m = (long long)h->n - (long long)S.n_active;
                if (m == 0) break;                                  // reading R26
                const long long cap = prm.cg_cap > 0 ? prm.cg_cap : m;
                long long its = 0;
                CK(cudaEventRecord(h->ev_a, h->st));
                rc = run_cg(h, cur, m, eta2, cap, &its);
                st.cg_calls++;
                st.cg_iters += its;
                if (rc) goto fail;
                CK(cudaEventRecord(h->ev_b, h->st));
                CK(cudaEventSynchronize(h->ev_b));
                CK(cudaEventElapsedTime(&ms, h->ev_a, h->ev_b));
                t_cg += ms;
                // projected search along d_k = Z_k w (Eq. cglsstop2), alpha = 2^-h
                int hacc = -1;
                if ((rc = search_and_accept(h, cur, h->W, 1.0, 0, &hacc))) goto fail;
                st.full_spmvs += 2;
                cur ^= 1;
                if (trace_on())
                    fprintf(stderr, "[gpcg] k=%lld CG rep=%lld m=%lld its=%lld reason=%d cg_ms=%.2f search_h=%d "
                            "|A|=%.0f nonbinding=%.0f pg=%.3e t=%.2fms\n",
                            (long long)k, (long long)rep, m, its, S.cg_reason, ms, hacc, S.n_active, S.n_nonbinding,
                            std::sqrt(S.pg2),
                            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
                if (std::sqrt(S.pg2) <= tau) { status = GPCG_OK; break; }
                if (S.n_nonbinding != 0.0) break;                   // Eq. cgstop3 fails
                eta2 = std::max(eta2 * prm.eta2_shrink, prm.eta2_floor);
                st.refinements++;
            }
        }
    }
    // x_out, q, sets
    if ((rc = download_vec(h, x_out, h->Y[cur]))) return rc;
    with_op_only(h, [&](auto& op) {
        using Op = std::decay_t<decltype(op)>;
        k_objective<Op><<<h->grid, kThreads, 0, h->st>>>(op, h->Y[cur], h->b, h->dS, h->red());
    });
    h->launches++;
    CKLAUNCH();
    if ((rc = sync_scal(h))) return rc;
    h->free_mask = cur;
    st.q = 0.5 * S.r0 - S.r1 + h->c;
    st.pg_norm = std::sqrt(S.pg2);
    st.n_active = (int64_t)S.n_active;
    st.n_free = h->n - st.n_active;
    st.n_active_nonbinding = (int64_t)S.n_nonbinding;
    st.t_cg_ms = t_cg;
    st.t_gp_ms = t_gp;
    st.status = status;
    st.kernel_launches = (int32_t)(h->launches & 0x7fffffff);
    st.cg_iters_timed = h->cg_iters_timed;
    st.cg_free_iters_timed = h->cg_free_iters_timed;
    st.t_cg_timed_ms = h->t_cg_timed_ms;
    st.t_total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    if (stats) *stats = st;
    if ((rc = leave(h))) return rc;
    return status;

fail:
    // on ESEARCH / ENOTSPD return the last feasible iterate
    {
        const std::string msg = g_err;
        cudaGetLastError();
        download_vec(h, x_out, h->Y[cur]);
        cudaStreamSynchronize(h->st);
        h->free_mask = cur;
        st.status = rc;
        st.pg_norm = std::sqrt(S.pg2);
        st.kernel_launches = (int32_t)(h->launches & 0x7fffffff);
        if (stats) *stats = st;
        leave(h);
        g_err = msg;
        return rc;
    }
}

}  // extern "C"
