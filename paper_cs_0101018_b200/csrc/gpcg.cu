// gpcg.cu -- libgpcg.so: the C ABI of include/gpcg.h and the host state machine
// of Algorithm GPCG driving the sm_100a kernels.
//
// Control: the host runs the outer logic from a few device
// scalars (one pinned readback per phase).  One slab on one rank with a 2-D
// broadcast-face stencil: a whole GP phase and a whole CG call are one persistent
// cooperative kernel each (march_tma.cuh k6_*), deciding on the device.  Otherwise
// the GP phase and the CG solve run as CUDA-graph chunks whose device-side
// finalisers set done flags (later launches are no-ops), polled once per chunk.
// The decisions follow, step by step, the same algorithm as oracle/gpcg_oracle.c
// (written independently; no shared code).
//
// Slabs: a handle owns one or more contiguous row slabs of
// the problem.  Each slab stores its vectors with ghost rows (2-D stencil: 3 grid
// rows per side, 3-D: 1 plane, CSR: the band of neighbour rows its columns reach), refreshed
// after every sweep that writes a vector some neighbour reads -- by a device
// copy between slabs of this process, or by NCCL send/recv between ranks.
// With more than one slab (or rank) every reducing kernel DEFERS its decision
// (RedScratch::out): the per-slab totals are summed in slab order (k_combine),
// allreduced across ranks (one ncclAllReduce of <= 2K+2 doubles: one per CG
// iteration, one per GP sub-step) and k_finalize applies the decision to the
// global totals.  One slab on one rank: no ghosts, no copies, no collectives.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types only: the functions are resolved at run time (the process's own NCCL)

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "gpcg.h"
#include "fin.cuh"
#include "kernels.cuh"
#include "march.cuh"
#include "tma.cuh"
#include "march_tma.cuh"
#include "extract.cuh"
#include "compact.cuh"
#include "bjilu.cuh"
#include "bjilu2.cuh"
#include "march3.cuh"

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

#define RC(call)                    \
    do {                            \
        int rc_ = (call);           \
        if (rc_) return rc_;        \
    } while (0)

bool trace_on() {
    static const bool on = getenv("GPCG_TRACE") != nullptr && getenv("GPCG_TRACE")[0] == '1';
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

// ---------------------------------------------------------------- NCCL (run-time bound)
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi* nccl_api() {
    static NcclApi api;
    static bool tried = false, ok = false;
    if (!tried) {
        tried = true;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the process's NCCL (e.g. torch's)
        if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (lib) {
#define NSYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(lib, "nccl" #f))
            NSYM(GetUniqueId); NSYM(CommInitRank); NSYM(CommDestroy); NSYM(AllReduce); NSYM(Broadcast);
            NSYM(Send); NSYM(Recv); NSYM(GroupStart); NSYM(GroupEnd); NSYM(GetErrorString); NSYM(AllGather);
#undef NSYM
            ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Broadcast &&
                 api.Send && api.Recv && api.GroupStart && api.GroupEnd && api.GetErrorString;
        }
    }
    return ok ? &api : nullptr;
}

#define NK(call)                                                                                \
    do {                                                                                        \
        ncclResult_t r_ = (call);                                                               \
        if (r_ != ncclSuccess)                                                                  \
            return set_err(GPCG_ENCCL, "%s: %s (%s:%d)", #call, nccl_api()->GetErrorString(r_), \
                           __FILE__, __LINE__);                                                 \
    } while (0)

// ---------------------------------------------------------------- vectors of a slab
enum Vec : int { VY0, VY1, VG0, VG1, VW, VP, VRHO0, VRHO1, VQ0, VQ1, VS0, VS1, VIN, VOUT, VB, VL, VU, VD, NVEC };
// VD: 1 / diag(A) (point-Jacobi PCG, gpcg_params.precond = 1)
enum Msk : int { MK0, MK1, MKCG, NMSK };
constexpr int NO_VEC = -1;
constexpr int NB_NONE = -1, NB_REMOTE = -2;

inline Vec vy(int k) { return (Vec)(VY0 + k); }
inline Vec vg(int k) { return (Vec)(VG0 + k); }
inline Vec vrho(int k) { return (Vec)(VRHO0 + k); }
inline Vec vq(int k) { return (Vec)(VQ0 + k); }
inline Vec vs(int k) { return (Vec)(VS0 + k); }
inline Msk mk(int k) { return (Msk)(MK0 + k); }

struct Slab {
    int row0 = 0, rows = 0;         // owned rows [row0, row0+rows) of the rank's part (grid rows / CSR rows)
    int uoff = 0;                   // offset of row0 in the rank's user arrays (rows)
    int glo = 0, ghi = 0;           // ghost rows below / above
    int send_lo = 0, send_hi = 0;   // rows the lower / upper neighbour reads from this slab
    int nb_lo = NB_NONE, nb_hi = NB_NONE;
    long long nalloc = 0;           // elements per vector = (glo + rows + ghi) * pitch
    void* arena = nullptr;          // one allocation holding every vector and mask of the slab
    double* vb[NVEC] = {};          // allocation bases (inside the arena)
    double* v[NVEC] = {};           // origins (owned row 0)
    unsigned char* mb[NMSK] = {};
    unsigned char* m[NMSK] = {};
    double *wxb = nullptr, *wyb = nullptr, *shb = nullptr;   // face arrays / shift (bases)
    double* brow = nullptr;         // global grid row 0 of b (nx), for the row-broadcast test / k4_accept
    long long* rp = nullptr;
    int* ci = nullptr;
    double* val = nullptr;
    StencilOp sop{};
    CsrOp cop{};
    Stencil3Op s3op{};
    double* partials = nullptr;
    unsigned int* counter = nullptr;
    MarchGeom mg1{}, mg2{};
    int grid_m1 = 1, grid_m2 = 1, grid = 1;
    int grid7 = 1;                            // 3-D plane-march kernels (march3.cuh)
    // TMA-fed column march (k4_*): 116-column band boxes of the vectors, the 112-column
    // w box of the CG iteration, 144-byte mask boxes
    CUtensorMap t4[NVEC];
    CUtensorMap t4wo;
    CUtensorMap t4c[4];             // CG sweep per-warp boxes: rho0, rho1, p0 (Q0), p1 (Q1), 32 x 4
    CUtensorMap t4cw;               // CG sweep per-warp w box, 28 x 4
    CUtensorMap t4m[NMSK];
    BandGeom bg_cg{}, bg_acc{}, bg_srch{};   // band x segment items sized to each kernel's residency
    unsigned short* cgflags = nullptr;        // k_cg_block_flags of the running CG call (bg_cg geometry)
    // explicit extraction (cg_mode = 1): compact numbering, A_F in CSR, compact CG vectors
    void* xarena = nullptr;
    int *xidx = nullptr, *xpos = nullptr, *xcnt = nullptr, *xcol = nullptr;
    long long *xblk = nullptr, *xtot = nullptr, *xrp = nullptr;
    double* xval = nullptr;
    double* xv[12] = {};                      // gF, dinvF, rho x2, q x2, s x2, p, w, (spare)
    unsigned char *xmask = nullptr, *xmaskcg = nullptr;
    // compacted free-row list (compact.cuh; CSR / 3-D operators, one slab): rows of mask fmask
    int* flist = nullptr;
    unsigned* fbits = nullptr;      // the same set as bits (k_pack_bits: n / 8 bytes, L2-resident)
    int* fpos = nullptr;            // pos[v] = k for v = F[k] (stale elsewhere: read under a free bit)
    double* cv = nullptr;           // reduced-space CG vectors: rho0/1, q0/1, s0/1, p, w (cv_cap each)
    long long cv_cap = 0;
    long long *fblk = nullptr, *ftot = nullptr;
    long long fcount = -1;
    int fmask = -1;
    double* bjf = nullptr;                    // block-Jacobi ILU factor (precond 2 / 3): 5 x tiles x 32^2 doubles
                                              // + tiles x 32^2 code bytes
    CUtensorMap tbr;                          // r (RHO0) in 32 x 32 boxes for the BJ-ILU tile solves
    int grid4_cg = 1, grid4_acc = 1, grid4_srch = 1;
    // g-free sweeps (k5_*): 112-column boxes from x0 - 4, 128-byte mask boxes, 104-column bands
    CUtensorMap t5[NVEC];
    CUtensorMap t5m[NMSK];
    BandGeom bg5_acc{}, bg5_srch{}, bg5_init{};
    int grid5_acc = 1, grid5_srch = 1, grid5_init = 1;
};

}  // namespace

// A slab as the neighbour whose fused halo stores write into its ghost rows sees it: the origins
// of rho0/1, p0/1 (the CG loop's ping-pong; VQ* hold p) and y0/1, mask0/1 (the GP loop's), its rows
// and ghost depths.  From a slab of this process, or (GPCG_XRANK) the facing slab of the
// neighbouring rank through its IPC-mapped arena.
struct XrSide {
    double* v[6];                   // VRHO0, VRHO1, VQ0, VQ1, VY0, VY1
    unsigned char* m[2];            // MK0, MK1
    int rows, glo, ghi;
};
constexpr int kXrVec[6] = {VRHO0, VRHO1, VQ0, VQ1, VY0, VY1};

struct gpcg_problem {
    int dev = 0, sms = 148;
    cudaMemPool_t pool = nullptr;   // device allocations (mem_pool); null: cudaMalloc / cudaFree
    cudaStream_t user = nullptr;    // caller's stream
    cudaStream_t st = nullptr;      // private work stream (capturable)
    cudaEvent_t ev_sync = nullptr, ev_a = nullptr, ev_b = nullptr, ev_c0 = nullptr, ev_c1 = nullptr;
    bool is_csr = false;
    bool is3d = false;              // 3-D 7-point stencil (generic kernels; rows = z-planes)
    int rowlen = 1;                 // elements of one user row: 2-D nx, 3-D nx*ny, CSR 1
    bool generic = false;           // GPCG_GENERIC=1: stencil problems use the flat generic kernels (A/B tests)
    bool sb = false;                // scalar (constant) bounds
    bool bc = false;                // stencil with broadcast faces and no shift
    bool bb = false;                // stencil with b equal in every grid row (k4_accept reads brow)
    bool tile = false;              // TMA tile path built
    int tile_mask = 127;            // GPCG_TILE bits: TMA tile kernels (k3) 1 accept, 2 search, 4 CG
                                    // iteration; TMA-fed column march (k4, preferred) 8 CG, 16 accept,
                                    // 32 search; 64 g-free k5 accept / search / CG init (preferred,
                                    // g is never stored).  0 = column march (k2) only.
    bool gfree = false;             // k5 sweeps active: the G vectors are not maintained
    int nx = 0, pitch = 1;          // stencil: grid width and row pitch (nx rounded up to 32); CSR: 1
    long long wx_ld = 0, wy_ld = 0; // user face layout (0 = broadcast)
    long long n_local = 0;          // entries owned by this rank (the user's arrays)
    long long n_global = 0;
    long long rank_row0 = 0;        // this rank's first global row
    long long nnz = 0;
    double c = 0.0;
    double lc = 0.0, uc = 0.0;      // the scalar bounds when sb
    std::vector<Slab> slabs;
    int rank = 0, nranks = 1;
    ncclComm_t comm = nullptr;
    bool use_nccl = false;          // collectives go through NCCL (nranks > 1, or GPCG_FORCE_NCCL=1: a
                                    // 1-rank communicator, to exercise the NCCL path on one GPU)
    bool deferred = false;          // several slabs or ranks: reductions go through k_finalize
    double* red_all = nullptr;      // [nslabs][kMaxSums] per-slab totals
    double* red_tot = nullptr;      // [kMaxSums] global totals
    double* lu0 = nullptr;          // global (l_0, u_0)
    Scal* dS = nullptr;
    Scal* hS = nullptr;             // pinned mirror
    gpcg_params prm{};
    int free_mask = -1;             // index of the recorded free set, -1 none
    cudaGraphExec_t cg_exec = nullptr;
    int cg_exec_chunk = 0;
    cudaGraphExec_t gp_exec[2] = {nullptr, nullptr};   // GP chunk graphs starting from buffers 0 / 1
    cudaGraphExec_t gp_exec_s[2] = {nullptr, nullptr}; // ... of gp_exec_s_chunk (< gp_exec_chunk) steps: a phase's first launch
    int gp_exec_s_chunk = 0;
    cudaGraphExec_t bj_exec = nullptr;  // block-Jacobi ILU PCG chunk graph (precond = 2 / 3)
    int bj_exec_chunk = 0, bj_exec_pc = 0;
    int gp_exec_chunk = 0;
    bool gp_graph = true;           // GPCG_GP_GRAPH=0: host-driven GP steps (A/B)
    bool cg_persistent = true;      // GPCG_CG_PERSIST=0: CG as graph chunks instead of k6_cg_loop
    bool gp_persistent = true;      // GPCG_GP_PERSIST=0: GP phase as graph chunks instead of k6_gp_loop
    bool cg_skip = true;            // GPCG_CG_SKIP=0: the CG sweep loads every block (no active-block skip)
    bool cg_pw = false;             // CG sweep with per-warp boxes (large grids; GPCG_CG_PW=0/1 overrides)
    bool gp_spec = true;            // GPCG_GP_SPEC=0: no speculative h = 0 accept in k6_gp_loop
    int grid6_gp = 1;
    size_t smem6_gp = 0;
    unsigned int* gbar = nullptr;   // grid-barrier counter of the persistent kernels
    // cross-rank protocol of the multi-slab persistent loops (march_tma.cuh XRank):
    // GPCG_XRANK_EMU=1 runs it on one device with every slab a virtual rank (one launch)
    bool xr_emu = false;
    unsigned long long* xr_bar = nullptr;     // [kMaxRanks][local, go, cross][kXrLine] counters (never reset)
    unsigned long long* xr_base = nullptr;    // [kMaxRanks][kXrLine]: local, cross arrivals, barriers before a launch
    double* xr_part = nullptr;                // [kMaxRanks][2][kXrSums][xr_stride] mailboxes
    int* xr_err = nullptr;                    // spin-timeout flag
    int xr_stride = 0;
    // GPCG_XRANK=1 with several ranks: the loops span the ranks (setup_xrank_real)
    bool xr_real = false;
    void* xr_region = nullptr;                // this rank's counters / base / err / mailbox (cudaMalloc)
    void* xr_peer[kMaxRanks] = {};            // the other ranks' regions, IPC-mapped
    std::vector<void*> xr_mapped;             // every opened mapping (closed at destroy)
    XrSide xr_lo{}, xr_hi{};                  // the lower / upper rank's facing slab
    int xr_cta_cg[kMaxRanks] = {}, xr_cta_gp[kMaxRanks] = {};
    long long launches = 0;
    long long cg_iters_timed = 0, cg_free_iters_timed = 0;
    double t_cg_timed_ms = 0.0;
    double t_extract_ms = 0.0;

    int nslabs() const { return (int)slabs.size(); }
    RedScratch red(int s) const {
        double* out = nullptr;
        if (deferred) out = nslabs() > 1 ? red_all + (long long)s * kMaxSums : red_tot;
        return RedScratch{slabs[s].partials, slabs[s].counter, out};
    }
    Bounds bounds(const Slab& s) const { return Bounds{s.v[VL], s.v[VU], lc, uc}; }
};

namespace {

// Device memory of a handle comes from one stream-ordered pool per device and process that
// keeps freed blocks reserved (release threshold = max): a create / solve / destroy cycle
// per request then costs no cudaMalloc / cudaFree (page mapping, implicit device-wide
// synchronisation) after the first.  GPCG_POOL=0 at create: plain cudaMalloc / cudaFree.
cudaMemPool_t mem_pool(int dev) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!pools[dev]) {
        cudaMemPoolProps pp = {};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = dev;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &pp) != cudaSuccess) { cudaGetLastError(); return nullptr; }
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        pools[dev] = pool;
    }
    return pools[dev];
}

// (allocations happen at create and lazily at the first solve needing a buffer; the stream is
// synchronised so the block may be used from any stream or by synchronous copies at once)
template <class T>
cudaError_t dalloc(gpcg_problem* h, T** p, size_t bytes) {
    if (!h->pool) return cudaMalloc(reinterpret_cast<void**>(p), bytes);
    const cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, h->pool, h->st);
    return e != cudaSuccess ? e : cudaStreamSynchronize(h->st);
}

void dfree(gpcg_problem* h, void* p) {
    if (!p) return;
    if (h->pool) cudaFreeAsync(p, h->st);
    else cudaFree(p);
}

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

// ---------------------------------------------------------------- reductions (a6)
// After the reducing kernel of every slab: nothing (one slab, decided in place)
// or combine -> allreduce -> finalize.
int finish_reduce(gpcg_problem* h, const FinArgs& a, int ns) {
    if (!h->deferred) return GPCG_OK;
    if (h->nslabs() > 1) {
        k_combine<<<1, 64, 0, h->st>>>(h->red_all, h->nslabs(), ns, h->red_tot);
        h->launches++;
        CKLAUNCH();
    }
    if (h->use_nccl)
        NK(nccl_api()->AllReduce(h->red_tot, h->red_tot, (size_t)ns, ncclDouble, ncclSum, h->comm, h->st));
    k_finalize<<<1, 32, 0, h->st>>>(h->red_tot, h->dS, a);
    h->launches++;
    CKLAUNCH();
    return GPCG_OK;
}
FinArgs fin(int kind) {
    FinArgs a;
    memset(&a, 0, sizeof a);
    a.kind = kind;
    return a;
}

// ---------------------------------------------------------------- halo exchange (8(e))
// A row-structured per-slab array: row r of slab s starts at base(s) + r*row_elems
// (r may be negative: ghost rows).  Ghost rows [-glo, 0) come from the lower
// neighbour's rows [lo_end - glo, lo_end) (lo_end = its rows); ghost rows
// [top, top + ghi) (top = rows + top_extra) come from the upper neighbour's rows
// [hi_begin, hi_begin + ghi).  Vectors: top_extra = hi_begin = 0; y-face rows
// (rows + 1 per slab): 1.
struct RowArray {
    char* (*base)(gpcg_problem*, Slab&, int);   // origin (row 0) of slab s for array id
    int id;
    size_t row_elems, esize;
    ncclDataType_t ntype;
    int top_extra, hi_begin;
};

char* vec_base(gpcg_problem*, Slab& s, int id) { return reinterpret_cast<char*>(s.v[id]); }
char* msk_base(gpcg_problem*, Slab& s, int id) { return reinterpret_cast<char*>(s.m[id]); }

int exchange_arrays(gpcg_problem* h, const RowArray* arr, int na) {
    bool remote = false;
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        for (int k = 0; k < na; ++k) {
            const RowArray& A = arr[k];
            const size_t rb = A.row_elems * A.esize;
            char* me = A.base(h, S, A.id);
            if (S.nb_lo >= 0 && S.glo > 0) {
                Slab& N = h->slabs[S.nb_lo];
                const char* src = A.base(h, N, A.id) + (long long)(N.rows - S.glo) * (long long)rb;
                CK(cudaMemcpyAsync(me - (long long)S.glo * rb, src, S.glo * rb, cudaMemcpyDeviceToDevice, h->st));
            }
            if (S.nb_hi >= 0 && S.ghi > 0) {
                Slab& N = h->slabs[S.nb_hi];
                const char* src = A.base(h, N, A.id) + (long long)A.hi_begin * (long long)rb;
                CK(cudaMemcpyAsync(me + (long long)(S.rows + A.top_extra) * rb, src, S.ghi * rb,
                                   cudaMemcpyDeviceToDevice, h->st));
            }
            if (S.nb_lo == NB_REMOTE || S.nb_hi == NB_REMOTE) remote = true;
        }
    }
    if (!remote) return GPCG_OK;
    const NcclApi* N = nccl_api();
    NK(N->GroupStart());
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        for (int k = 0; k < na; ++k) {
            const RowArray& A = arr[k];
            const size_t rb = A.row_elems;      // elements
            char* me = A.base(h, S, A.id);
            const long long eb = (long long)A.esize;
            if (S.nb_lo == NB_REMOTE) {
                if (S.send_lo > 0)
                    NK(N->Send(me + (long long)A.hi_begin * rb * eb, S.send_lo * rb, A.ntype, h->rank - 1, h->comm, h->st));
                if (S.glo > 0)
                    NK(N->Recv(me - (long long)S.glo * rb * eb, S.glo * rb, A.ntype, h->rank - 1, h->comm, h->st));
            }
            if (S.nb_hi == NB_REMOTE) {
                if (S.send_hi > 0)
                    NK(N->Send(me + (long long)(S.rows - S.send_hi) * rb * eb, S.send_hi * rb, A.ntype, h->rank + 1,
                               h->comm, h->st));
                if (S.ghi > 0)
                    NK(N->Recv(me + (long long)(S.rows + A.top_extra) * rb * eb, S.ghi * rb, A.ntype, h->rank + 1,
                               h->comm, h->st));
            }
        }
    }
    NK(N->GroupEnd());
    return GPCG_OK;
}

bool has_ghosts(const gpcg_problem* h) { return h->nslabs() > 1 || h->nranks > 1; }

// several slabs of one device, one process: the persistent loops span all slabs (SlabLink)
// (GPCG_MS_ONE=1, diagnostic: one slab through the multi-slab kernels as well)
bool multi_slab_persistent(const gpcg_problem* h) {
    static const bool ms1 = getenv("GPCG_MS_ONE") && atoi(getenv("GPCG_MS_ONE")) != 0;
    if (h->xr_real) return h->nslabs() <= kMaxMs;
    return h->nranks == 1 && !h->use_nccl && (h->nslabs() > 1 || ms1) && h->nslabs() <= kMaxMs;
}

// 2-D stencil with its specialised sweeps (march / tile kernels); otherwise the generic kernels
bool spec2d(const gpcg_problem* h) { return !h->is_csr && !h->is3d && !h->generic; }

// f(op) with the slab's operator policy (generic kernels)
// 3-D stencils run the plane-march kernels (march3.cuh) unless GPCG_GENERIC=1
bool use_m3(const gpcg_problem* h) { return h->is3d && !h->generic; }

template <class F>
void with_gop(const gpcg_problem* h, Slab& S, F&& f) {
    if (h->is_csr) f(S.cop);
    else if (h->is3d) f(S.s3op);
    else f(S.sop);
}
template <class F>
void with_gop_sb(const gpcg_problem* h, Slab& S, F&& f) {
    if (h->sb) with_gop(h, S, [&](auto& op) { f(op, std::true_type()); });
    else with_gop(h, S, [&](auto& op) { f(op, std::false_type()); });
}

int exchange(gpcg_problem* h, std::initializer_list<int> vecs, std::initializer_list<int> msks = {}) {
    if (!has_ghosts(h)) return GPCG_OK;
    RowArray arr[8];
    int na = 0;
    for (int id : vecs)
        arr[na++] = RowArray{vec_base, id, (size_t)h->pitch, sizeof(double), ncclDouble, 0, 0};
    for (int id : msks)
        arr[na++] = RowArray{msk_base, id, (size_t)h->pitch, 1, ncclUint8, 0, 0};
    return exchange_arrays(h, arr, na);
}

// ---------------------------------------------------------------- user vectors <-> slabs
int copy_kind(const void* p, bool to_device) {
    const bool dev = is_device_ptr(p);
    return to_device ? (dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice)
                     : (dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
}

// the rank's contiguous user vector (n_local entries) -> vector id of every slab (owned rows)
int upload_vec(gpcg_problem* h, int id, const double* src) {
    const cudaMemcpyKind k = (cudaMemcpyKind)copy_kind(src, true);
    const size_t cols = (size_t)h->rowlen;
    for (Slab& S : h->slabs)
        CK(cudaMemcpy2DAsync(S.v[id], (size_t)h->pitch * sizeof(double), src + (long long)S.uoff * cols,
                             cols * sizeof(double), cols * sizeof(double), S.rows, k, h->st));
    return GPCG_OK;
}
int download_vec(gpcg_problem* h, double* dst, int id) {
    const cudaMemcpyKind k = (cudaMemcpyKind)copy_kind(dst, false);
    const size_t cols = (size_t)h->rowlen;
    for (Slab& S : h->slabs)
        CK(cudaMemcpy2DAsync(dst + (long long)S.uoff * cols, cols * sizeof(double), S.v[id],
                             (size_t)h->pitch * sizeof(double), cols * sizeof(double), S.rows, k, h->st));
    return GPCG_OK;
}

void free_all(gpcg_problem* h) {
    if (!h) return;
    cudaSetDevice(h->dev);
    if (h->st) cudaStreamSynchronize(h->st);
    for (Slab& S : h->slabs) {
        dfree(h, S.arena);
        for (void* p : {(void*)S.wxb, (void*)S.wyb, (void*)S.shb, (void*)S.brow, (void*)S.cgflags, S.xarena, (void*)S.bjf, (void*)S.rp,
                        (void*)S.flist, (void*)S.fbits, (void*)S.fpos, (void*)S.cv, (void*)S.fblk, (void*)S.ftot,
                        (void*)S.ci, (void*)S.val,
                        (void*)S.partials, (void*)S.counter})
            dfree(h, p);
    }
    for (void* p : {(void*)h->red_all, (void*)h->red_tot, (void*)h->lu0, (void*)h->dS, (void*)h->gbar,
                    (void*)h->xr_bar, (void*)h->xr_base, (void*)h->xr_part, (void*)h->xr_err})
        dfree(h, p);
    if (h->xr_real && h->comm && nccl_api()) {      // no rank frees what a peer still maps
        int* one = nullptr;
        if (cudaMalloc(&one, sizeof(int)) == cudaSuccess) {
            nccl_api()->AllReduce(one, one, 1, ncclInt32, ncclSum, h->comm, h->st);
            cudaStreamSynchronize(h->st);
            cudaFree(one);
        }
    }
    for (void* p : h->xr_mapped) cudaIpcCloseMemHandle(p);
    if (h->xr_region) cudaFree(h->xr_region);
    if (h->hS) cudaFreeHost(h->hS);
    if (h->cg_exec) cudaGraphExecDestroy(h->cg_exec);
    if (h->bj_exec) cudaGraphExecDestroy(h->bj_exec);
    for (cudaGraphExec_t g : h->gp_exec)
        if (g) cudaGraphExecDestroy(g);
    for (cudaGraphExec_t g : h->gp_exec_s)
        if (g) cudaGraphExecDestroy(g);
    if (h->comm && nccl_api()) nccl_api()->CommDestroy(h->comm);
    for (cudaEvent_t e : {h->ev_sync, h->ev_a, h->ev_b, h->ev_c0, h->ev_c1})
        if (e) cudaEventDestroy(e);
    if (h->st) cudaStreamDestroy(h->st);
    delete h;
}

// ---------------------------------------------------------------- geometry
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

// 2-D tensor map over a slab array: rows [-glo, rows+ghi) (owned + ghost); elements outside the
// tensor read as 0 (the Dirichlet boundary)
int make_map(gpcg_problem* h, const Slab& S, CUtensorMap* m, const void* origin, bool u8, int bw, int bh) {
    if (bw * (u8 ? 1 : 8) % 16 != 0) return set_err(GPCG_EINVAL, "internal: TMA box row not a multiple of 16 B");
    auto enc = tma_encode_fn();
    if (!enc) return set_err(GPCG_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const long long es = u8 ? 1 : 8;
    const char* base = static_cast<const char*>(origin) - (long long)S.glo * h->pitch * es;
    const cuuint64_t dims[2] = {(cuuint64_t)h->nx, (cuuint64_t)(S.glo + S.rows + S.ghi)};
    const cuuint64_t strides[1] = {(cuuint64_t)h->pitch * es};
    const cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                     const_cast<char*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(GPCG_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return GPCG_OK;
}

template <class K>
int set_smem(K kernel, int bytes) {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    return GPCG_OK;
}

// TMA tile path for a broadcast-face stencil (C0/C2/C3 family)
int setup_tile(gpcg_problem* h) {
    {
        // per-warp CG boxes pay off once the CG vectors (rho x2, p x2, w: 40 B per point) leave
        // the 126 MB L2 (C3: 64M points); below that the band boxes' 3 TMA operations a block win
        long long pts = 0;
        for (const Slab& S : h->slabs) pts += (long long)S.rows * h->nx;
        h->cg_pw = 40LL * pts > 256LL * 1024 * 1024;
        if (const char* e = getenv("GPCG_CG_PW")) h->cg_pw = atoi(e) != 0;
    }
    RC(set_smem(k4_hessvec<true>, m4hv::kSmem));
    RC(set_smem(k4_hessvec<false>, m4hv::kSmem));
    RC(set_smem(k4_cg_iter<false>, m4cg::kSmem));
    RC(set_smem(k4_cg_iter<true>, m4cg::kSmem));
    RC(set_smem(k6_cg_loop<false>, m4cg::kSmem));
    RC(set_smem(k6_cg_loop<true>, m4cg::kSmem));
    RC(set_smem(k6_cg_loop_ms<false, false>, m4cg::kSmem));
    RC(set_smem(k6_cg_loop_ms<true, false>, m4cg::kSmem));
    RC(set_smem(k6_cg_loop_ms<false, true>, m4cg::kSmem));
    RC(set_smem(k6_cg_loop_ms<true, true>, m4cg::kSmem));
    RC(set_smem(k4_accept<true, true, false>, AccLayout4<true, true, false>::kSmem));
    RC(set_smem(k4_accept<true, false, false>, AccLayout4<true, false, false>::kSmem));
    RC(set_smem(k4_accept<false, true, false>, AccLayout4<false, true, false>::kSmem));
    RC(set_smem(k4_accept<false, false, false>, AccLayout4<false, false, false>::kSmem));
    RC(set_smem(k4_accept<true, true, true>, AccLayout4<true, true, true>::kSmem));
    RC(set_smem(k4_accept<true, false, true>, AccLayout4<true, false, true>::kSmem));
    RC(set_smem(k4_accept<false, true, true>, AccLayout4<false, true, true>::kSmem));
    RC(set_smem(k4_accept<false, false, true>, AccLayout4<false, false, true>::kSmem));
#define K5ACC(SB, BB, M) RC(set_smem(k5_accept<SB, BB, M>, AccLayout5<SB, BB, M>::kSmem));
#define K5ACC2(SB, BB) K5ACC(SB, BB, m5::GP) K5ACC(SB, BB, m5::CG) K5ACC(SB, BB, m5::PROJ)
    K5ACC2(true, true) K5ACC2(true, false) K5ACC2(false, true) K5ACC2(false, false)
#define K5SP(SB, BB) RC(set_smem(k5_spec<SB, BB>, AccLayout5<SB, BB, m5::GP>::kSmem));
    K5SP(true, true) K5SP(true, false) K5SP(false, true) K5SP(false, false)
#define K5S(SB, BB, M, K) RC(set_smem(k5_search<SB, BB, M, K>, SrchLayout5<SB, BB, M, K>::kSmem));
#define K5S2(SB, BB) K5S(SB, BB, m5::GP, 2) K5S(SB, BB, m5::GP, 8) K5S(SB, BB, m5::CG, 2) K5S(SB, BB, m5::CG, 8)
    K5S2(true, true) K5S2(true, false) K5S2(false, true) K5S2(false, false)
    RC(set_smem(k5_cg_init<true, true>, CgInitLayout5<true>::kSmem));
    RC(set_smem(k5_cg_init<true, false>, CgInitLayout5<true>::kSmem));
    RC(set_smem(k5_cg_init<false, true>, CgInitLayout5<false>::kSmem));
    RC(set_smem(k5_cg_init<false, false>, CgInitLayout5<false>::kSmem));
#undef K5ACC
#undef K5ACC2
#undef K5S
#undef K5S2
    RC(set_smem(k4_search<true, true>, SrchLayout4<true, true>::kSmem));
    RC(set_smem(k4_search<true, false>, SrchLayout4<true, false>::kSmem));
    RC(set_smem(k4_search<false, true>, SrchLayout4<false, true>::kSmem));
    RC(set_smem(k4_search<false, false>, SrchLayout4<false, false>::kSmem));
    auto res4 = [&](auto kernel, int smem) {
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, m4::kThreads, smem);
        return std::max(1, nb) * h->sms;
    };
    int nbcg = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbcg, k4_cg_iter<false>, m4::kThreadsWS, m4cg::kSmem);
    const int r4cg = std::max(1, nbcg) * h->sms;
    const int r4acc = h->sb ? (h->bb ? res4(k4_accept<true, true, true>, AccLayout4<true, true, true>::kSmem)
                                     : res4(k4_accept<true, true, false>, AccLayout4<true, true, false>::kSmem))
                            : (h->bb ? res4(k4_accept<false, true, true>, AccLayout4<false, true, true>::kSmem)
                                     : res4(k4_accept<false, true, false>, AccLayout4<false, true, false>::kSmem));
    const int r4srch = h->sb ? res4(k4_search<true, true>, SrchLayout4<true, true>::kSmem)
                             : res4(k4_search<false, true>, SrchLayout4<false, true>::kSmem);
    // k5: residency of the GP-mode variants of this problem's (SB, BB)
    int r5acc, r5srch, r5init;
    {
        auto pick = [&](auto sbt, auto bbt) {
            constexpr bool SB = decltype(sbt)::value, BB = decltype(bbt)::value;
            r5acc = res4(k5_accept<SB, BB, m5::GP>, AccLayout5<SB, BB, m5::GP>::kSmem);
            r5srch = res4(k5_search<SB, BB, m5::GP, 2>, SrchLayout5<SB, BB, m5::GP, 2>::kSmem);
            r5init = res4(k5_cg_init<BB, false>, CgInitLayout5<BB>::kSmem);
        };
        if (h->sb) { if (h->bb) pick(std::true_type(), std::true_type()); else pick(std::true_type(), std::false_type()); }
        else { if (h->bb) pick(std::false_type(), std::true_type()); else pick(std::false_type(), std::false_type()); }
    }
    for (Slab& S : h->slabs) {
        // k4: bands of 112 columns, each split into nsegs row segments: one item per resident CTA
        for (int id : {VY0, VY1, VG0, VG1, VRHO0, VRHO1, VQ0, VQ1, VW, VB, VL, VU, VIN})
            RC(make_map(h, S, &S.t4[id], S.v[id], false, m4::kBW, m4::kBR));
        RC(make_map(h, S, &S.t4wo, S.v[VW], false, m4::kOut, m4::kBR));
        {
            const int ids[4] = {VRHO0, VRHO1, VQ0, VQ1};
            for (int i = 0; i < 4; ++i) RC(make_map(h, S, &S.t4c[i], S.v[ids[i]], false, m4cg::kPW, m4::kBR));
            RC(make_map(h, S, &S.t4cw, S.v[VW], false, m4cg::kWW, m4::kBR));
        }
        for (int k = 0; k < NMSK; ++k) RC(make_map(h, S, &S.t4m[k], S.m[k], true, m4::kMW, m4::kBR));
        for (int id : {VY0, VY1, VW, VB, VL, VU, VIN})
            RC(make_map(h, S, &S.t5[id], S.v[id], false, m5::kBW, m5::kBR5));
        for (int k = 0; k < NMSK; ++k) RC(make_map(h, S, &S.t5m[k], S.m[k], true, m5::kMW, m5::kBR5));
        // ipc: items per CTA (> 1 spreads each CTA's work over several shorter segments: the CG
        // sweep skips the loads of all-active blocks, so equal-area items are not equal work;
        // several items a CTA even out the grid barrier's wait for the slowest)
        auto band = [&](int resident, BandGeom& G, int& grid, int out = m4::kOut, int ipc = 1) {
            G.nbands = (h->nx + out - 1) / out;
            G.nsegs = std::max(1, std::min(resident * ipc / G.nbands, (S.rows + 15) / 16));
            G.seg = (S.rows + G.nsegs - 1) / G.nsegs;
            G.nsegs = (S.rows + G.seg - 1) / G.seg;
            G.rlo = -S.glo;
            grid = std::min(G.nbands * G.nsegs, resident);
        };
        // GPCG_CG_CTAS_PER_SM / GPCG_GP_CTAS_PER_SM (tuning): cap the CTAs per SM of the CG / GP bands
        auto cap_env = [&](const char* name, int r) {
            const char* e = getenv(name);
            return (e && atoi(e) > 0) ? std::min(r, atoi(e) * h->sms) : r;
        };
        // several slabs in one persistent CG launch: the resident CTAs are shared among the slabs
        {
            int ipc = h->cg_pw ? 16 : 1;                 // C3: 61-row items instead of 1000 (CG 420 -> 372 us)
            if (const char* e = getenv("GPCG_CG_ITEMS_PER_CTA")) ipc = std::max(1, atoi(e));
            band(cap_env("GPCG_CG_CTAS_PER_SM", r4cg) / (multi_slab_persistent(h) ? h->nslabs() : 1), S.bg_cg,
                 S.grid4_cg, m4::kOut, ipc);
        }
        {
            const long long nf = (long long)S.bg_cg.nbands * S.bg_cg.nsegs * ((S.bg_cg.seg + 4 + m4::kBR - 1) / m4::kBR);
            CK(dalloc(h, &S.cgflags, (size_t)std::max<long long>(nf, 1) * sizeof(unsigned short)));
        }
        band(r4acc, S.bg_acc, S.grid4_acc);
        band(r4srch, S.bg_srch, S.grid4_srch);
        const int gshare = multi_slab_persistent(h) ? h->nslabs() : 1;   // one persistent GP launch, all slabs
        // GP items per CTA: the count (1-4) that minimises the pipeline blocks of the most loaded
        // CTA -- 1 for one slab of C3 (429 items on 444 CTAs), 2 for each of two slabs (195 items
        // of 800 rows vs 429 of 364 on 222 CTAs)
        auto gp_ipc = [&](int resident) {
            int best = 1;
            long long best_cost = -1;
            for (int ipc = 1; ipc <= 4; ++ipc) {
                BandGeom T;
                int g = 0;
                band(resident, T, g, m5::kOut, ipc);
                const long long items = (long long)T.nbands * T.nsegs;
                // rows a CTA sweeps: its items' segments + 5 lag rows, in whole pipeline blocks, + one
                // block per item for the pipeline's restart
                const long long blk = (T.seg + 5 + m5::kBR5 - 1) / m5::kBR5 + 1;
                const long long cost = (items + g - 1) / g * blk;
                if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = ipc; }
            }
            return best;
        };
        const int r5a = cap_env("GPCG_GP_CTAS_PER_SM", r5acc) / gshare, r5s = cap_env("GPCG_GP_CTAS_PER_SM", r5srch) / gshare;
        const int gipc = getenv("GPCG_GP_ITEMS_PER_CTA") ? std::max(1, atoi(getenv("GPCG_GP_ITEMS_PER_CTA")))
                                                         : gp_ipc(std::min(r5a, r5s));
        band(r5a, S.bg5_acc, S.grid5_acc, m5::kOut, gipc);
        band(r5s, S.bg5_srch, S.grid5_srch, m5::kOut, gipc);
        band(r5init, S.bg5_init, S.grid5_init, m5::kOut);
    }
    h->tile = true;
    h->gfree = (h->tile_mask & 64) != 0;
    {
        // persistent GP phase: smem of the larger (accept) layout; grid within co-residency
        auto cfg = [&](auto sbt, auto bbt) {
            constexpr bool SB = decltype(sbt)::value, BB = decltype(bbt)::value;
            const size_t sm = std::max<size_t>(AccLayout5<SB, BB, m5::GP>::kSmem, SrchLayout5<SB, BB, m5::GP, 2>::kSmem);
            h->smem6_gp = sm;
            cudaFuncSetAttribute(k6_gp_loop<SB, BB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            cudaFuncSetAttribute(k6_gp_loop_ms<SB, BB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            cudaFuncSetAttribute(k6_gp_loop_ms<SB, BB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            int nb = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k6_gp_loop<SB, BB>, m4::kThreads, sm);
            return std::max(1, nb) * h->sms;
        };
        int r6;
        if (h->sb) r6 = h->bb ? cfg(std::true_type(), std::true_type()) : cfg(std::true_type(), std::false_type());
        else r6 = h->bb ? cfg(std::false_type(), std::true_type()) : cfg(std::false_type(), std::false_type());
        const Slab& S0 = h->slabs[0];
        h->grid6_gp = std::max(1, std::min({r6, S0.grid5_srch, S0.grid5_acc}));
    }
    return GPCG_OK;
}

// ---------------------------------------------------------------- create (common part)
// Slab layout of the rank's rows [0, rows_rank): nsl balanced contiguous slabs.
void partition(long long total, int parts, int k, long long* b, long long* e) {
    const long long q = total / parts, r = total % parts;
    *b = k * q + std::min<long long>(k, r);
    *e = *b + q + (k < r ? 1 : 0);
}

int setup_comm(gpcg_problem* h, const gpcg_dist* d) {
    h->rank = d ? d->rank : 0;
    h->nranks = d ? d->nranks : 1;
    if (h->nranks > 1) {
        const NcclApi* N = nccl_api();
        if (!N) return set_err(GPCG_ENCCL, "libnccl.so.2 not loadable: the multi-rank path needs NCCL");
        if (!d->nccl_id) return set_err(GPCG_EINVAL, "nccl_id is NULL with nranks > 1");
        ncclUniqueId id;
        memcpy(&id, d->nccl_id, sizeof id);
        NK(N->CommInitRank(&h->comm, h->nranks, id, h->rank));
        h->use_nccl = true;
    } else if (getenv("GPCG_FORCE_NCCL") && getenv("GPCG_FORCE_NCCL")[0] == '1') {
        const NcclApi* N = nccl_api();
        if (!N) return set_err(GPCG_ENCCL, "GPCG_FORCE_NCCL=1 but libnccl.so.2 is not loadable");
        ncclUniqueId id;
        NK(N->GetUniqueId(&id));
        NK(N->CommInitRank(&h->comm, 1, id, 0));
        h->use_nccl = true;
    }
    return GPCG_OK;
}

int create_streams(gpcg_problem* h, void* stream) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return set_err(GPCG_ECUDA, "no CUDA device (the library has no CPU fallback)");
    }
    CK(cudaGetDevice(&h->dev));
    CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->dev));
    h->user = (cudaStream_t)stream;
    {
        const char* e = getenv("GPCG_GP_GRAPH");
        h->gp_graph = !(e && e[0] == '0');
        const char* e2 = getenv("GPCG_CG_PERSIST");
        h->cg_persistent = !(e2 && e2[0] == '0');
        const char* e3 = getenv("GPCG_GP_PERSIST");
        h->gp_persistent = !(e3 && e3[0] == '0');
        const char* e4 = getenv("GPCG_CG_SKIP");
        h->cg_skip = !(e4 && e4[0] == '0');
        const char* e5 = getenv("GPCG_GP_SPEC");
        h->gp_spec = !(e5 && e5[0] == '0');
    }
    CK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    {
        const char* e6 = getenv("GPCG_POOL");
        const char* e8 = getenv("GPCG_XRANK");              // IPC-exported arenas need cudaMalloc memory
        h->pool = ((e6 && e6[0] == '0') || (e8 && atoi(e8) != 0)) ? nullptr : mem_pool(h->dev);
    }
    CK(dalloc(h, &h->gbar, sizeof(unsigned int)));
    {
        const char* e7 = getenv("GPCG_XRANK_EMU");
        h->xr_emu = e7 && atoi(e7) != 0;
    }
    CK(cudaEventCreateWithFlags(&h->ev_sync, cudaEventDisableTiming));
    CK(cudaEventCreate(&h->ev_a));
    CK(cudaEventCreate(&h->ev_b));
    CK(cudaEventCreate(&h->ev_c0));
    CK(cudaEventCreate(&h->ev_c1));
    CK(cudaEventRecord(h->ev_sync, h->user));
    CK(cudaStreamWaitEvent(h->st, h->ev_sync, 0));
    return GPCG_OK;
}

// slab vectors, masks, scratch; b, l, u uploaded; inputs validated (globally)
int create_vectors(gpcg_problem* h, const double* b, const double* l, const double* u) {
    for (Slab& S : h->slabs) {
        S.nalloc = (long long)(S.glo + S.rows + S.ghi) * h->pitch;
        const size_t nb = ((size_t)S.nalloc * sizeof(double) + 255) / 256 * 256;
        const size_t mbytes = ((size_t)S.nalloc + 255) / 256 * 256;
        const long long off = (long long)S.glo * h->pitch;
        // one arena per slab (few large allocations keep create / destroy cheap); 256-byte aligned
        // sub-arrays; zeroed: padding columns and boundary ghosts stay 0
        const size_t total = NVEC * nb + NMSK * mbytes;
        CK(dalloc(h, &S.arena, total));
        CK(cudaMemsetAsync(S.arena, 0, total, h->st));
        char* base = static_cast<char*>(S.arena);
        for (int k = 0; k < NVEC; ++k) {
            S.vb[k] = reinterpret_cast<double*>(base + k * nb);
            S.v[k] = S.vb[k] + off;
        }
        for (int k = 0; k < NMSK; ++k) {
            S.mb[k] = reinterpret_cast<unsigned char*>(base + NVEC * nb + k * mbytes);
            S.m[k] = S.mb[k] + off;
        }
        // partial sums of the largest grid any kernel of this slab uses (grid-stride generic kernels
        // are capped at 16 blocks/SM; march grids are one warp per item)
        long long gmax = (long long)h->sms * 16;
        if (!h->is_csr && !h->is3d) {
            S.mg1 = march_geom(h->nx, S.rows, 1);
            S.mg2 = march_geom(h->nx, S.rows, 2);
            S.grid_m1 = march_grid(S.mg1);
            S.grid_m2 = march_grid(S.mg2);
            gmax = std::max<long long>(gmax, std::max(S.grid_m1, S.grid_m2));
        }
        CK(dalloc(h, &S.partials, (size_t)kMaxSums * gmax * sizeof(double)));
        CK(dalloc(h, &S.counter, sizeof(unsigned int)));
        CK(cudaMemsetAsync(S.counter, 0, sizeof(unsigned int), h->st));
    }
    CK(dalloc(h, &h->red_all, (size_t)kMaxSums * h->nslabs() * sizeof(double)));
    CK(dalloc(h, &h->red_tot, (size_t)kMaxSums * sizeof(double)));
    CK(cudaMemsetAsync(h->red_tot, 0, (size_t)kMaxSums * sizeof(double), h->st));
    CK(dalloc(h, &h->lu0, 2 * sizeof(double)));
    CK(dalloc(h, &h->dS, sizeof(Scal)));
    CK(cudaMemsetAsync(h->dS, 0, sizeof(Scal), h->st));
    CK(cudaMallocHost(&h->hS, sizeof(Scal)));
    RC(upload_vec(h, VB, b));
    RC(upload_vec(h, VL, l));
    RC(upload_vec(h, VU, u));
    RC(exchange(h, {VB, VL, VU}));
    // validation: l <= u, no NaN / inf in b, l != +inf, u != -inf; constant bounds (vs the global
    // first pair, broadcast from rank 0)?
    CK(cudaMemcpyAsync(h->lu0, h->slabs[0].v[VL], sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(h->lu0 + 1, h->slabs[0].v[VU], sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    if (h->use_nccl) NK(nccl_api()->Broadcast(h->lu0, h->lu0, 2, ncclDouble, 0, h->comm, h->st));
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const int cols = h->is_csr ? S.rows : h->rowlen, rows = h->is_csr ? 1 : S.rows;
        const int g = std::max(1, (int)std::min<long long>(((long long)S.rows * h->rowlen + kThreads - 1) / kThreads,
                                                           (long long)h->sms * 4));
        k_check_inputs<<<g, kThreads, 0, h->st>>>(cols, rows, h->is_csr ? S.rows : h->pitch, S.v[VB], S.v[VL], S.v[VU],
                                                  h->lu0, h->dS, h->red(s));
        CKLAUNCH();
    }
    RC(finish_reduce(h, fin(FIN_R2), 2));
    RC(sync_scal(h));
    if (h->hS->r0 != 0.0)
        return set_err(GPCG_EINVAL, "%.0f entries violate l <= u (or NaN/inf in b, l = +inf, u = -inf)", h->hS->r0);
    h->sb = (h->hS->r1 == 0.0);
#ifdef GPCG_DIAG_FORCE_SB
    h->sb = true;                   // diagnostic builds only: time the sweeps without the l / u streams
#endif
    double lu[2];
    CK(cudaMemcpy(lu, h->lu0, sizeof lu, cudaMemcpyDeviceToHost));
    h->lc = lu[0];
    h->uc = lu[1];
    h->prm = gpcg_params_default();
    return GPCG_OK;
}

// count of non-finite values of a per-slab array (owned part), summed over slabs and ranks
int count_nonfinite(gpcg_problem* h, const double* const* arrs, const long long* cnts, double* out) {
    for (int s = 0; s < h->nslabs(); ++s) {
        const int g = (int)std::max<long long>(1, std::min<long long>((cnts[s] + kThreads - 1) / kThreads,
                                                                      (long long)h->sms * 4));
        k_count_nonfinite<<<g, kThreads, 0, h->st>>>(cnts[s], arrs[s], h->dS, h->red(s));
        CKLAUNCH();
    }
    RC(finish_reduce(h, fin(FIN_R2), 2));
    RC(sync_scal(h));
    *out = h->hS->r0;
    return GPCG_OK;
}

// slab rows of the rank's rows; neighbours; ghost widths (stencil: 2)
int layout_slabs(gpcg_problem* h, long long rows_rank, int nsl, int ghost) {
    if (nsl < 1 || nsl > 64) return set_err(GPCG_EINVAL, "local_slabs = %d out of range [1, 64]", nsl);
    h->slabs.resize(nsl);
    for (int s = 0; s < nsl; ++s) {
        Slab& S = h->slabs[s];
        long long b, e;
        partition(rows_rank, nsl, s, &b, &e);
        S.uoff = (int)b;
        S.row0 = (int)b;
        S.rows = (int)(e - b);
        S.nb_lo = s > 0 ? s - 1 : (h->rank > 0 ? NB_REMOTE : NB_NONE);
        S.nb_hi = s < nsl - 1 ? s + 1 : (h->rank < h->nranks - 1 ? NB_REMOTE : NB_NONE);
        S.glo = S.nb_lo != NB_NONE ? ghost : 0;
        S.ghi = S.nb_hi != NB_NONE ? ghost : 0;
        S.send_lo = S.glo;
        S.send_hi = S.ghi;
        const int need = (S.nb_lo != NB_NONE || S.nb_hi != NB_NONE) ? std::max(ghost, 1) : 1;
        if (S.rows < need) return set_err(GPCG_EINVAL, "slab %d has %d rows (need >= %d)", s, S.rows, need);
    }
    h->deferred = has_ghosts(h) || h->use_nccl;
    return GPCG_OK;
}

// ---------------------------------------------------------------- launches (every slab)
int launch_accept(gpcg_problem* h, int y_in, int dir, double sgn, int mask_prev, int y_out, int g_out, int m_out,
                  int gp = 0) {
    const bool use_k5 = h->gfree;
    const bool use_k4 = h->tile && (h->tile_mask & 16);
    const int mode = dir < 0 ? m5::PROJ : ((dir == VG0 || dir == VG1) ? m5::GP : m5::CG);
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const Bounds B = h->bounds(S);
        const RedScratch R = h->red(s);
        if (use_k5) {
            const CUtensorMap& md = S.t5[dir >= 0 && mode == m5::CG ? dir : y_in];
            const CUtensorMap& mp = S.t5m[mask_prev >= 0 ? mask_prev : MK0];
            const int has_mp = mask_prev >= 0 ? 1 : 0;
            auto go = [&](auto sbt, auto bbt, auto mt) {
                constexpr bool SB = decltype(sbt)::value, BB = decltype(bbt)::value;
                constexpr int M = decltype(mt)::value;
                k5_accept<SB, BB, M><<<S.grid5_acc, m4::kThreads, AccLayout5<SB, BB, M>::kSmem, h->st>>>(
                    S.sop, S.bg5_acc, B, S.brow, S.t5[y_in], md, S.t5[VB], S.t5[VL], S.t5[VU], mp, has_mp,
                    S.v[y_out], S.m[m_out], h->dS, R, gp);
            };
            auto bymode = [&](auto sbt, auto bbt) {
                if (mode == m5::GP) go(sbt, bbt, std::integral_constant<int, m5::GP>());
                else if (mode == m5::CG) go(sbt, bbt, std::integral_constant<int, m5::CG>());
                else go(sbt, bbt, std::integral_constant<int, m5::PROJ>());
            };
            auto bybb = [&](auto sbt) {
                if (h->bb) bymode(sbt, std::true_type()); else bymode(sbt, std::false_type());
            };
            if (h->sb) bybb(std::true_type()); else bybb(std::false_type());
        } else if (use_k4) {
            const CUtensorMap& md = S.t4[dir >= 0 ? dir : y_in];
            const CUtensorMap& mp = S.t4m[mask_prev >= 0 ? mask_prev : MK0];
            const int has_mp = mask_prev >= 0 ? 1 : 0;
            auto go = [&](auto sbt, auto hdt, auto bbt) {
                constexpr bool SB = decltype(sbt)::value, HD = decltype(hdt)::value, BB = decltype(bbt)::value;
                k4_accept<SB, HD, BB><<<S.grid4_acc, m4::kThreads, AccLayout4<SB, HD, BB>::kSmem, h->st>>>(
                    S.sop, S.bg_acc, B, S.brow, S.t4[y_in], md, S.t4[VB], S.t4[VL], S.t4[VU], mp, has_mp, sgn,
                    S.v[y_out], S.v[g_out], S.m[m_out], h->dS, R, gp);
            };
            auto bydir = [&](auto sbt, auto bbt) {
                if (dir >= 0) go(sbt, std::true_type(), bbt); else go(sbt, std::false_type(), bbt);
            };
            auto bybb = [&](auto sbt) {
                if (h->bb) bydir(sbt, std::true_type()); else bydir(sbt, std::false_type());
            };
            if (h->sb) bybb(std::true_type()); else bybb(std::false_type());
        } else if (spec2d(h)) {   // accept + regrad + mask + counts + next Cauchy step, one sweep
            const double* dp = dir >= 0 ? S.v[dir] : nullptr;
            const unsigned char* mp = mask_prev >= 0 ? S.m[mask_prev] : nullptr;
            auto go = [&](auto sbt, auto bct) {
                constexpr bool SB = decltype(sbt)::value, BC = decltype(bct)::value;
                k2_accept<SB, BC><<<S.grid_m2, kMarchThreads, 0, h->st>>>(S.sop, S.mg2, B, S.v[y_in], dp, sgn, S.v[VB],
                                                                          mp, S.v[y_out], S.v[g_out], S.m[m_out], h->dS, R,
                                                                          gp);
            };
            if (h->sb) { if (h->bc) go(std::true_type(), std::true_type()); else go(std::true_type(), std::false_type()); }
            else { if (h->bc) go(std::false_type(), std::true_type()); else go(std::false_type(), std::false_type()); }
        } else {
            const double* dp = dir >= 0 ? S.v[dir] : nullptr;
            const unsigned char* mp = mask_prev >= 0 ? S.m[mask_prev] : nullptr;
            if (use_m3(h)) {
                if (h->sb)
                    k7_accept<true><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, B, S.v[y_in], dp, sgn, S.v[VB], mp,
                                                                         S.v[y_out], S.v[g_out], S.m[m_out], h->dS, R, gp);
                else
                    k7_accept<false><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, B, S.v[y_in], dp, sgn, S.v[VB], mp,
                                                                          S.v[y_out], S.v[g_out], S.m[m_out], h->dS, R, gp);
            } else
            with_gop_sb(h, S, [&](auto& op, auto sbt) {
                using Op = std::decay_t<decltype(op)>;
                constexpr bool SB = decltype(sbt)::value;
                k_accept<Op, SB><<<S.grid, kThreads, 0, h->st>>>(op, B, S.v[y_in], dp, sgn, S.v[VB], mp, S.v[y_out],
                                                                S.v[g_out], S.m[m_out], h->dS, R, gp);
            });
        }
        h->launches++;
        CKLAUNCH();
    }
    FinArgs a = fin(spec2d(h) ? FIN_ACCEPT : FIN_ACCEPT5);
    a.has_dir = dir >= 0 ? 1 : 0;
    a.gp = gp;
    RC(finish_reduce(h, a, a.kind == FIN_ACCEPT ? 6 : 5));
    if (use_k5) return exchange(h, {y_out}, {m_out});      // g is not stored
    return exchange(h, {y_out, g_out}, {m_out});
}

bool fused_cauchy(const gpcg_problem* h) { return spec2d(h); }

int launch_cauchy(gpcg_problem* h, int y, int g, int gp = 0) {
    if (fused_cauchy(h)) return GPCG_OK;     // computed by the preceding accept sweep
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const Bounds B = h->bounds(S);
        if (use_m3(h)) {
            if (h->sb) k7_cauchy<true><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, B, S.v[y], S.v[g], h->dS, h->red(s), gp);
            else k7_cauchy<false><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, B, S.v[y], S.v[g], h->dS, h->red(s), gp);
        } else
        with_gop_sb(h, S, [&](auto& op, auto sbt) {
            using Op = std::decay_t<decltype(op)>;
            constexpr bool SB = decltype(sbt)::value;
            k_cauchy<Op, SB><<<S.grid, kThreads, 0, h->st>>>(op, B, S.v[y], S.v[g], h->dS, h->red(s), gp);
        });
        h->launches++;
        CKLAUNCH();
    }
    FinArgs a = fin(FIN_CAUCHY);
    a.gp = gp;
    return finish_reduce(h, a, 2);
}

// The generic operators (CSR, 3-D) take each GP step and the CG phase's step speculatively at
// h = 0 (k_spec: search sums + accept in one sweep; GPCG_GP_SPEC=0: off); the 2-D stencils fuse
// the GP step into their own sweeps (k6_gp_loop, spec_sweep6).
bool graph_spec(const gpcg_problem* h) { return h->gp_spec && !spec2d(h); }
// the 2-D GP graph (slabs / ranks off the persistent loop) takes its steps with k5_spec
bool graph_spec5(const gpcg_problem* h) { return h->gp_spec && spec2d(h) && h->gfree; }

int launch_spec5(gpcg_problem* h, int cur) {
    const int nxt = cur ^ 1;
    const double mu = h->prm.mu;
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const Bounds B = h->bounds(S);
        auto go = [&](auto sbt, auto bbt) {
            constexpr bool SB = decltype(sbt)::value, BB = decltype(bbt)::value;
            k5_spec<SB, BB><<<S.grid5_acc, m4::kThreads, AccLayout5<SB, BB, m5::GP>::kSmem, h->st>>>(
                S.sop, S.bg5_acc, B, S.brow, S.t5[vy(cur)], S.t5[VB], S.t5[VL], S.t5[VU], S.t5m[mk(cur)],
                S.v[vy(nxt)], S.m[mk(nxt)], mu, h->dS, h->red(s));
        };
        auto bybb = [&](auto sbt) {
            if (h->bb) go(sbt, std::true_type()); else go(sbt, std::false_type());
        };
        if (h->sb) bybb(std::true_type()); else bybb(std::false_type());
        h->launches++;
        CKLAUNCH();
    }
    FinArgs a = fin(FIN_SPEC6);
    a.mu = mu;
    a.gp = 1;
    RC(finish_reduce(h, a, 8));
    return exchange(h, {vy(nxt)}, {mk(nxt)});    // g is not stored
}

// y(nxt), g(nxt), mask(nxt) = the step at h = 0 from y(cur) along sgn * dir (base alpha_0 or 1)
int launch_spec(gpcg_problem* h, int cur, int dir, double sgn, int use_alpha0, int gp) {
    const double mu = h->prm.mu;
    const int nxt = cur ^ 1;
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const Bounds B = h->bounds(S);
        with_gop_sb(h, S, [&](auto& op, auto sbt) {
            using Op = std::decay_t<decltype(op)>;
            constexpr bool SB = decltype(sbt)::value;
            k_spec<Op, SB><<<S.grid, kThreads, 0, h->st>>>(op, B, S.v[vy(cur)], S.v[dir], sgn, use_alpha0, S.v[vg(cur)],
                                                          S.v[VB], S.v[vy(nxt)], S.v[vg(nxt)], S.m[mk(nxt)], mu, h->dS,
                                                          h->red(s), gp);
        });
        h->launches++;
        CKLAUNCH();
    }
    FinArgs a = fin(FIN_SPEC);
    a.mu = mu;
    a.gp = gp;
    a.use_alpha0 = use_alpha0;
    RC(finish_reduce(h, a, 7));
    return exchange(h, {vy(nxt), vg(nxt)}, {mk(nxt)});
}

// step sizes per projected-search sweep: the first sweep evaluates search_k
// (2 or 8 instantiated), later sweeps 8
int first_k(const gpcg_problem* h) { return h->prm.search_k <= 2 ? 2 : 8; }

int launch_search(gpcg_problem* h, int y, int g, int dir, double sgn, int use_alpha0, int h0, int K, int gp = 0) {
    const double mu = h->prm.mu;
    const bool dg = (dir == g);
    const bool use_k5 = h->gfree;                                  // K = 2 and the K = 8 retries
    const bool use_k4 = h->tile && (h->tile_mask & 32) && K == 2;  // retries use the column march
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const Bounds B = h->bounds(S);
        const RedScratch R = h->red(s);
        if (use_k5) {
            // GP: direction -g (recomputed from y); CG: direction w
            auto go = [&](auto sbt, auto bbt, auto mt, auto kt) {
                constexpr bool SB = decltype(sbt)::value, BB = decltype(bbt)::value;
                constexpr int M = decltype(mt)::value, KK = decltype(kt)::value;
                k5_search<SB, BB, M, KK><<<S.grid5_srch, m4::kThreads, SrchLayout5<SB, BB, M, KK>::kSmem, h->st>>>(
                    S.sop, S.bg5_srch, B, S.brow, S.t5[y], S.t5[dg ? y : dir], S.t5[VB], S.t5[VL], S.t5[VU], h0, mu,
                    h->dS, R, gp);
            };
            auto byk = [&](auto sbt, auto bbt, auto mt) {
                if (K == 2) go(sbt, bbt, mt, std::integral_constant<int, 2>());
                else go(sbt, bbt, mt, std::integral_constant<int, 8>());
            };
            auto bymode = [&](auto sbt, auto bbt) {
                if (dg) byk(sbt, bbt, std::integral_constant<int, m5::GP>());
                else byk(sbt, bbt, std::integral_constant<int, m5::CG>());
            };
            auto bybb = [&](auto sbt) {
                if (h->bb) bymode(sbt, std::true_type()); else bymode(sbt, std::false_type());
            };
            if (h->sb) bybb(std::true_type()); else bybb(std::false_type());
        } else if (use_k4) {
            auto go = [&](auto sbt, auto dgt) {
                constexpr bool SB = decltype(sbt)::value, DG = decltype(dgt)::value;
                k4_search<SB, DG><<<S.grid4_srch, m4::kThreads, SrchLayout4<SB, DG>::kSmem, h->st>>>(
                    S.sop, S.bg_srch, B, S.t4[y], S.t4[dir], S.t4[g], S.t4[VL], S.t4[VU], sgn, use_alpha0, h0, mu, h->dS, R, gp);
            };
            if (h->sb) { if (dg) go(std::true_type(), std::true_type()); else go(std::true_type(), std::false_type()); }
            else { if (dg) go(std::false_type(), std::true_type()); else go(std::false_type(), std::false_type()); }
        } else if (spec2d(h)) {
            auto go = [&](auto sbt, auto bct, auto kt, auto dgt) {
                constexpr bool SB = decltype(sbt)::value, BC = decltype(bct)::value, DG = decltype(dgt)::value;
                constexpr int KK = decltype(kt)::value;
                k2_search<SB, BC, KK, DG><<<S.grid_m1, kMarchThreads, 0, h->st>>>(
                    S.sop, S.mg1, B, S.v[y], S.v[g], S.v[dir], sgn, use_alpha0, h0, mu, h->dS, R, gp);
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
        } else if (use_m3(h) && K == 2) {
            if (h->sb)
                k7_search<true, 2><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, B, S.v[y], S.v[g], S.v[dir], sgn,
                                                                        use_alpha0, h0, mu, h->dS, R, gp);
            else
                k7_search<false, 2><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, B, S.v[y], S.v[g], S.v[dir], sgn,
                                                                         use_alpha0, h0, mu, h->dS, R, gp);
        } else {
            with_gop_sb(h, S, [&](auto& op, auto sbt) {
                using Op = std::decay_t<decltype(op)>;
                constexpr bool SB = decltype(sbt)::value;
                if (K == 2)
                    k_search<Op, SB, 2><<<S.grid, kThreads, 0, h->st>>>(op, B, S.v[y], S.v[g], S.v[dir], sgn, use_alpha0,
                                                                        h0, mu, h->dS, R, gp);
                else
                    k_search<Op, SB, 8><<<S.grid, kThreads, 0, h->st>>>(op, B, S.v[y], S.v[g], S.v[dir], sgn, use_alpha0,
                                                                        h0, mu, h->dS, R, gp);
            });
        }
        h->launches++;
        CKLAUNCH();
    }
    FinArgs a = fin(FIN_SEARCH);
    a.K = K;
    a.h0 = h0;
    a.use_alpha0 = use_alpha0;
    a.mu = mu;
    a.gp = gp;
    return finish_reduce(h, a, 2 * K);
}

// one projected search + accept:  y' = P[y + alpha sgn dir], g' = A y' - b.
// Host loops over batches of K step sizes until one is accepted.  Returns
// GPCG_OK with *accepted_h >= 0, or GPCG_ESEARCH.
int search_and_accept(gpcg_problem* h, int cur, int dir, double sgn, int use_alpha0, int* accepted_h, int h_start = 0) {
    const int nxt = cur ^ 1;
    for (int h0 = h_start, K = h_start ? 8 : first_k(h); h0 < h->prm.max_halvings; h0 += K, K = 8) {
        RC(launch_search(h, vy(cur), vg(cur), dir, sgn, use_alpha0, h0, K));
        RC(launch_accept(h, vy(cur), dir, sgn, mk(cur), vy(nxt), vg(nxt), mk(nxt)));
        RC(sync_scal(h));
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

// one CG iteration on every slab (+ exchange + deferred finalize): captured into the graph
int enqueue_cg_iter(gpcg_problem* h, int a) {
    const int bb = a ^ 1;
    const bool pc = h->prm.precond == 1;
    const bool use_k4 = h->tile && (h->tile_mask & 8);
    const bool skip = h->cg_skip;
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const RedScratch R = h->red(s);
        if (use_k4) {
            if (pc)
                k4_cg_iter<true><<<S.grid4_cg, m4::kThreadsWS, m4cg::kSmem, h->st>>>(
                    S.sop, S.bg_cg, h->cg_pw ? S.t4c[a] : S.t4[vrho(a)], h->cg_pw ? S.t4c[2 + a] : S.t4[vq(a)],
                    h->cg_pw ? S.t4cw : S.t4wo, S.t4m[MKCG], S.v[vrho(bb)], S.v[vq(bb)], S.v[VW],
                    h->dS, R, skip ? S.cgflags : nullptr, h->cg_pw ? 1 : 0);
            else
                k4_cg_iter<false><<<S.grid4_cg, m4::kThreadsWS, m4cg::kSmem, h->st>>>(
                    S.sop, S.bg_cg, h->cg_pw ? S.t4c[a] : S.t4[vrho(a)], h->cg_pw ? S.t4c[2 + a] : S.t4[vq(a)],
                    h->cg_pw ? S.t4cw : S.t4wo, S.t4m[MKCG], S.v[vrho(bb)], S.v[vq(bb)], S.v[VW],
                    h->dS, R, skip ? S.cgflags : nullptr, h->cg_pw ? 1 : 0);
        } else if (spec2d(h)) {   // stencil: rho, p ping-pong (p in Q[]), w in place
            auto go = [&](auto bct, auto pct) {
                constexpr bool BC = decltype(bct)::value, PC = decltype(pct)::value;
                k2_cg_iter<BC, PC><<<S.grid_m2, kMarchThreads, 0, h->st>>>(S.sop, S.mg2, S.m[MKCG], S.v[vrho(a)],
                                                                           S.v[vq(a)], S.v[vrho(bb)], S.v[vq(bb)],
                                                                           S.v[VW], h->dS, R);
            };
            if (h->bc) { if (pc) go(std::true_type(), std::true_type()); else go(std::true_type(), std::false_type()); }
            else { if (pc) go(std::false_type(), std::true_type()); else go(std::false_type(), std::false_type()); }
        } else if (use_m3(h)) {
            auto go = [&](auto pct) {
                constexpr bool PC = decltype(pct)::value;
                k7_cg_iter<PC><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, S.m[MKCG], S.v[vrho(a)], S.v[vq(a)],
                                                                    S.v[vs(a)], S.v[vrho(bb)], S.v[vq(bb)], S.v[vs(bb)],
                                                                    S.v[VP], S.v[VW], S.v[VD], h->dS, R);
            };
            if (pc) go(std::true_type()); else go(std::false_type());
        } else {
            with_gop(h, S, [&](auto& op) {
                using Op = std::decay_t<decltype(op)>;
                auto go = [&](auto pct) {
                    constexpr bool PC = decltype(pct)::value;
                    k_cg_iter<Op, PC><<<S.grid, kThreads, 0, h->st>>>(op, S.m[MKCG], S.v[vrho(a)], S.v[vq(a)],
                                                                      S.v[vs(a)], S.v[vrho(bb)], S.v[vq(bb)],
                                                                      S.v[vs(bb)], S.v[VP], S.v[VW], S.v[VD], h->dS, R);
                };
                if (pc) go(std::true_type()); else go(std::false_type());
            });
        }
        h->launches++;
        CKLAUNCH();
    }
    if (!spec2d(h)) RC(exchange(h, {vrho(bb), vq(bb), vs(bb)}));
    else RC(exchange(h, {vrho(bb), vq(bb)}));
    return finish_reduce(h, fin(FIN_CG_ITER), 2);
}

int build_cg_graph(gpcg_problem* h, int chunk) {
    if (h->cg_exec && h->cg_exec_chunk == chunk) return GPCG_OK;
    if (h->cg_exec) {
        cudaGraphExecDestroy(h->cg_exec);
        h->cg_exec = nullptr;
    }
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
    const long long l0 = h->launches;
    int rc = GPCG_OK;
    for (int i = 0; i < chunk && !rc; ++i) rc = enqueue_cg_iter(h, i & 1);
    h->launches = l0;
    cudaError_t e = cudaStreamEndCapture(h->st, &graph);
    if (rc) {
        if (e == cudaSuccess) cudaGraphDestroy(graph);
        return rc;
    }
    if (e != cudaSuccess) return set_err(GPCG_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&h->cg_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return set_err(GPCG_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    h->cg_exec_chunk = chunk;
    return GPCG_OK;
}

// GP chunk: `chunk` steps of [Cauchy (generic kernels), first search batch, accept, k_gp_step]
// starting from buffers c0, the buffers alternating per step (a finished phase makes the rest no-ops)
int build_gp_graph_into(gpcg_problem* h, int chunk, cudaGraphExec_t (&out)[2]) {
    for (int c0 = 0; c0 < 2; ++c0) {
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
        const long long l0 = h->launches;
        int rc = GPCG_OK;
        for (int i = 0; i < chunk && !rc; ++i) {
            const int cur = (c0 + i) & 1, nxt = cur ^ 1;
            rc = launch_cauchy(h, vy(cur), vg(cur), 1);
            if (!rc && graph_spec(h)) rc = launch_spec(h, cur, vg(cur), -1.0, 1, 1);
            if (!rc && graph_spec5(h)) rc = launch_spec5(h, cur);
            const int h0 = (graph_spec(h) || graph_spec5(h)) ? 1 : 0;
            if (!rc) rc = launch_search(h, vy(cur), vg(cur), vg(cur), -1.0, 1, h0, first_k(h), 1);
            if (!rc) rc = launch_accept(h, vy(cur), vg(cur), -1.0, mk(cur), vy(nxt), vg(nxt), mk(nxt), 1);
            if (!rc) {
                k_gp_step<<<1, 32, 0, h->st>>>(h->dS);
                cudaError_t e = cudaGetLastError();
                if (e != cudaSuccess) rc = set_err(GPCG_ECUDA, "k_gp_step launch: %s", cudaGetErrorString(e));
            }
        }
        h->launches = l0;
        cudaError_t e = cudaStreamEndCapture(h->st, &graph);
        if (rc) {
            if (e == cudaSuccess) cudaGraphDestroy(graph);
            return rc;
        }
        if (e != cudaSuccess) return set_err(GPCG_ECUDA, "graph capture: %s", cudaGetErrorString(e));
        e = cudaGraphInstantiate(&out[c0], graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return set_err(GPCG_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
    }
    return GPCG_OK;
}

// the chunk graphs, and a 2-step pair for the first launch of each phase (short phases -- C4's
// are 2-3 steps -- then launch no no-op steps)
int build_gp_graph(gpcg_problem* h, int chunk) {
    if (h->gp_exec[0] && h->gp_exec_chunk == chunk) return GPCG_OK;
    for (cudaGraphExec_t& g : h->gp_exec)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    for (cudaGraphExec_t& g : h->gp_exec_s)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    RC(build_gp_graph_into(h, chunk, h->gp_exec));
    h->gp_exec_chunk = chunk;
    h->gp_exec_s_chunk = 0;
    if (chunk > 2) {
        RC(build_gp_graph_into(h, 2, h->gp_exec_s));
        h->gp_exec_s_chunk = 2;
    }
    return GPCG_OK;
}

int launches_per_gp_step(const gpcg_problem* h) {
    const int fins = h->deferred ? (1 + (h->nslabs() > 1 ? 1 : 0)) : 0;
    return (fused_cauchy(h) ? 0 : h->nslabs() + fins) +
           ((graph_spec(h) || graph_spec5(h)) ? 3 : 2) * (h->nslabs() + fins) + 1;
}

// The whole GP phase (until it stops or hands a step back) as one cooperative launch.
// the persistent GP phase runs: one slab and rank, or several slabs of one device (k6_gp_loop_ms)
bool gp_persist(const gpcg_problem* h) {
    return h->gp_persistent && h->gfree && (!h->deferred || multi_slab_persistent(h));
}

XrSide side_of(const Slab& N) {
    XrSide x;
    for (int k = 0; k < 6; ++k) x.v[k] = N.v[kXrVec[k]];
    x.m[0] = N.m[MK0];
    x.m[1] = N.m[MK1];
    x.rows = N.rows;
    x.glo = N.glo;
    x.ghi = N.ghi;
    return x;
}

// the slab whose ghost rows slab S's fused halo stores write into, below (lo) or above it
bool neighbour_side(const gpcg_problem* h, const Slab& S, bool lo, XrSide* out) {
    const int nb = lo ? S.nb_lo : S.nb_hi;
    if (nb >= 0) { *out = side_of(h->slabs[nb]); return true; }
    if (nb == NB_REMOTE && h->xr_real) { *out = lo ? h->xr_lo : h->xr_hi; return true; }
    return false;
}

// GPCG_XRANK=1, several ranks, 2-D broadcast-face stencil on the persistent loops: export this
// rank's counter / mailbox region and the arenas of its two boundary slabs (CUDA IPC), all-gather
// them with the CTA counts of its launches over the handle's NCCL communicator, open the other
// ranks' regions and the neighbours' facing arenas.  Not run here: one GPU per
// machine (the one-launch emulation runs the same kernels and neighbour tables).
struct XrRecord {
    cudaIpcMemHandle_t region, arena_lo, arena_hi;
    long long off_lo[8], off_hi[8];           // kXrVec origins, then MK0, MK1: bytes from the arena base
    int rows_lo, glo_lo, ghi_lo, rows_hi, glo_hi, ghi_hi;
    int ctas_cg, ctas_gp;
};

int setup_xrank_real(gpcg_problem* h) {
    const NcclApi* N = nccl_api();
    if (!N || !N->AllGather) return set_err(GPCG_ENCCL, "GPCG_XRANK: ncclAllGather not available");
    if (h->nranks > kMaxRanks) return set_err(GPCG_EINVAL, "GPCG_XRANK: at most %d ranks", kMaxRanks);
    if (h->pool) return set_err(GPCG_EINVAL, "GPCG_XRANK: the arenas must come from cudaMalloc");
    constexpr size_t L = kXrLine * sizeof(unsigned long long);
    h->xr_stride = h->nranks * h->sms * 8;
    const size_t bytes = 5 * L + (size_t)2 * kXrSums * h->xr_stride * sizeof(double);
    CK(cudaMalloc(&h->xr_region, bytes));
    CK(cudaMemset(h->xr_region, 0, bytes));
    XrRecord me;
    memset(&me, 0, sizeof me);
    CK(cudaIpcGetMemHandle(&me.region, h->xr_region));
    const Slab& F = h->slabs.front();
    const Slab& B = h->slabs.back();
    CK(cudaIpcGetMemHandle(&me.arena_lo, F.arena));
    CK(cudaIpcGetMemHandle(&me.arena_hi, B.arena));
    auto offs = [](const Slab& S, long long* o) {
        const XrSide x = side_of(S);
        const char* a = static_cast<const char*>(S.arena);
        for (int k = 0; k < 6; ++k) o[k] = reinterpret_cast<const char*>(x.v[k]) - a;
        o[6] = reinterpret_cast<const char*>(x.m[0]) - a;
        o[7] = reinterpret_cast<const char*>(x.m[1]) - a;
    };
    offs(F, me.off_lo);
    offs(B, me.off_hi);
    me.rows_lo = F.rows; me.glo_lo = F.glo; me.ghi_lo = F.ghi;
    me.rows_hi = B.rows; me.glo_hi = B.glo; me.ghi_hi = B.ghi;
    for (const Slab& S : h->slabs) {
        me.ctas_cg += S.grid4_cg;
        me.ctas_gp += std::max(1, std::min(S.grid5_srch, S.grid5_acc));
    }
    std::vector<XrRecord> all(h->nranks);
    char* dbuf = nullptr;
    CK(cudaMalloc(&dbuf, (size_t)(h->nranks + 1) * sizeof(XrRecord)));
    CK(cudaMemcpy(dbuf, &me, sizeof me, cudaMemcpyHostToDevice));
    const ncclResult_t nr = N->AllGather(dbuf, dbuf + sizeof(XrRecord), sizeof(XrRecord), ncclChar, h->comm, h->st);
    cudaError_t ce = cudaStreamSynchronize(h->st);
    if (ce == cudaSuccess)
        ce = cudaMemcpy(all.data(), dbuf + sizeof(XrRecord), (size_t)h->nranks * sizeof(XrRecord), cudaMemcpyDeviceToHost);
    cudaFree(dbuf);
    if (nr != ncclSuccess) return set_err(GPCG_ENCCL, "GPCG_XRANK: record all-gather failed");
    CK(ce);
    auto open = [&](const cudaIpcMemHandle_t& hd, void** p) {
        const cudaError_t e = cudaIpcOpenMemHandle(p, hd, cudaIpcMemLazyEnablePeerAccess);
        if (e == cudaSuccess) h->xr_mapped.push_back(*p);
        return e;
    };
    for (int r = 0; r < h->nranks; ++r) {
        h->xr_cta_cg[r] = all[r].ctas_cg;
        h->xr_cta_gp[r] = all[r].ctas_gp;
        if (r != h->rank) CK(open(all[r].region, &h->xr_peer[r]));
    }
    auto side = [](char* base, const long long* o, int rows, int glo, int ghi) {
        XrSide x;
        for (int k = 0; k < 6; ++k) x.v[k] = reinterpret_cast<double*>(base + o[k]);
        x.m[0] = reinterpret_cast<unsigned char*>(base + o[6]);
        x.m[1] = reinterpret_cast<unsigned char*>(base + o[7]);
        x.rows = rows; x.glo = glo; x.ghi = ghi;
        return x;
    };
    if (h->rank > 0) {                        // the lower rank's top slab
        const XrRecord& R = all[h->rank - 1];
        void* p = nullptr;
        CK(open(R.arena_hi, &p));
        h->xr_lo = side(static_cast<char*>(p), R.off_hi, R.rows_hi, R.glo_hi, R.ghi_hi);
    }
    if (h->rank < h->nranks - 1) {            // the upper rank's bottom slab
        const XrRecord& R = all[h->rank + 1];
        void* p = nullptr;
        CK(open(R.arena_lo, &p));
        h->xr_hi = side(static_cast<char*>(p), R.off_lo, R.rows_lo, R.glo_lo, R.ghi_lo);
    }
    h->xr_err = reinterpret_cast<int*>(static_cast<char*>(h->xr_region) + 4 * L);
    h->xr_real = true;
    return GPCG_OK;
}

// The XRank of a multi-slab persistent launch: nr = 0 (one device, the plain grid barrier), or
// under GPCG_XRANK_EMU every slab a virtual rank with its own counter and mailbox (the cross-rank
// protocol run inside one cooperative launch; same sums in the same order -> same bits).
int make_xrank(gpcg_problem* h, const int* cta0, int nslabs, int total, XRank* X, bool cg) {
    memset(X, 0, sizeof *X);
    if (h->xr_real) {
        const int* ctas = cg ? h->xr_cta_cg : h->xr_cta_gp;
        X->nr = h->nranks;
        int acc = 0;
        for (int r = 0; r < h->nranks; ++r) {
            X->cta0[r] = acc;
            acc += ctas[r];
        }
        X->cta0[h->nranks] = acc;
        X->cta_total = acc;
        X->cta_base = X->cta0[h->rank];
        X->cta_stride = h->xr_stride;
        if (total != ctas[h->rank] || acc > h->xr_stride)
            return set_err(GPCG_EINVAL, "cross-rank launch of %d CTAs (exported %d, all ranks %d, mailbox %d)", total,
                           ctas[h->rank], acc, h->xr_stride);
        char* R = static_cast<char*>(h->xr_region);
        constexpr size_t L = kXrLine * sizeof(unsigned long long);
        X->lbar[h->rank] = reinterpret_cast<unsigned long long*>(R);               // line 0; line 1: go flag
        X->base[h->rank] = reinterpret_cast<unsigned long long*>(R + 3 * L);
        X->err = reinterpret_cast<int*>(R + 4 * L);
        for (int r = 0; r < h->nranks; ++r) {
            char* Q = r == h->rank ? R : static_cast<char*>(h->xr_peer[r]);
            X->bar[r] = reinterpret_cast<unsigned long long*>(Q + 2 * L);
            X->part[r] = reinterpret_cast<double*>(Q + 5 * L);
        }
        X->sys = 1;
        return GPCG_OK;
    }
    (void)cg;
    if (!h->xr_emu) return GPCG_OK;
    if (nslabs > kMaxRanks) return set_err(GPCG_EINVAL, "GPCG_XRANK_EMU: at most %d slabs", kMaxRanks);
    if (!h->xr_bar) {
        h->xr_stride = std::max(total, h->sms * 16);
        const size_t nbar = (size_t)kMaxRanks * 3 * kXrLine, nbase = (size_t)kMaxRanks * kXrLine;
        CK(dalloc(h, &h->xr_bar, nbar * sizeof(unsigned long long)));
        CK(dalloc(h, &h->xr_base, nbase * sizeof(unsigned long long)));
        CK(dalloc(h, &h->xr_part, (size_t)kMaxRanks * 2 * kXrSums * h->xr_stride * sizeof(double)));
        CK(dalloc(h, &h->xr_err, sizeof(int)));
        CK(cudaMemsetAsync(h->xr_bar, 0, nbar * sizeof(unsigned long long), h->st));
        CK(cudaMemsetAsync(h->xr_base, 0, nbase * sizeof(unsigned long long), h->st));
        CK(cudaMemsetAsync(h->xr_err, 0, sizeof(int), h->st));
    }
    if (total > h->xr_stride)
        return set_err(GPCG_EINVAL, "GPCG_XRANK_EMU: launch of %d CTAs > mailbox %d", total, h->xr_stride);
    X->nr = nslabs;
    X->cta_base = 0;
    X->cta_total = total;
    X->cta_stride = h->xr_stride;
    for (int r = 0; r < nslabs; ++r) {
        X->cta0[r] = cta0[r];
        X->lbar[r] = h->xr_bar + (size_t)(3 * r) * kXrLine;       // + kXrLine: the rank's go flag
        X->bar[r] = h->xr_bar + (size_t)(3 * r + 2) * kXrLine;
        X->base[r] = h->xr_base + (size_t)r * kXrLine;
        X->part[r] = h->xr_part + (size_t)r * 2 * kXrSums * h->xr_stride;
    }
    X->cta0[nslabs] = total;
    X->err = h->xr_err;
    X->sys = getenv("GPCG_XRANK_SYS") && atoi(getenv("GPCG_XRANK_SYS")) != 0;   // A/B: system scope on one device
    return GPCG_OK;
}

// after a launch with XRank: a spin that timed out (a rank that never arrived) is an error
int check_xrank(gpcg_problem* h) {
    if (!h->xr_err) return GPCG_OK;
    int e = 0;
    CK(cudaMemcpyAsync(&e, h->xr_err, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (e) return set_err(GPCG_ECUDA, "cross-rank barrier: a rank did not arrive within %llu s",
                          kXrSpinNs / 1000000000ull);
    return GPCG_OK;
}

int launch_gp_loop_ms(gpcg_problem* h, int cur) {
    GpMsArgs P;
    memset(&P, 0, sizeof P);
    P.nslabs = h->nslabs();
    int cta = 0;
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        GpMsSlab& X = P.s[s];
        X.m_y0 = S.t5[VY0]; X.m_y1 = S.t5[VY1]; X.m_b = S.t5[VB]; X.m_l = S.t5[VL]; X.m_u = S.t5[VU];
        X.m_m0 = S.t5m[MK0]; X.m_m1 = S.t5m[MK1];
        X.A = S.sop;
        X.Gs = S.bg5_srch;
        X.Ga = S.bg5_acc;
        X.Bd = h->bounds(S);
        X.brow = S.brow;
        X.y0p = S.v[VY0]; X.y1p = S.v[VY1]; X.mk0 = S.m[MK0]; X.mk1 = S.m[MK1];
        const int g = std::max(1, std::min(S.grid5_srch, S.grid5_acc));
        X.Ls = SlabLink{0, g, 0, 0, 0};
        XrSide N;
        if (neighbour_side(h, S, true, &N)) {
            X.lo_y0 = N.v[4]; X.lo_y1 = N.v[5]; X.lo_m0 = N.m[0]; X.lo_m1 = N.m[1];
            X.Ls.lo_rows = N.rows;
            X.Ls.lo_ghost = N.ghi;
        }
        if (neighbour_side(h, S, false, &N)) {
            X.hi_y0 = N.v[4]; X.hi_y1 = N.v[5]; X.hi_m0 = N.m[0]; X.hi_m1 = N.m[1];
            X.Ls.hi_ghost = N.glo;
        }
        X.La = X.Ls;
        X.cta0 = cta;
        cta += g;
    }
    int c0[kMaxMs];
    for (int s = 0; s < h->nslabs(); ++s) c0[s] = P.s[s].cta0;
    XRank XR;
    RC(make_xrank(h, c0, h->nslabs(), cta, &XR, false));
    CK(cudaMemsetAsync(h->gbar, 0, sizeof(unsigned int), h->st));
    double mu = h->prm.mu;
    int spec = h->gp_spec ? 1 : 0;
    void* args[] = {(void*)&P, (void*)&cur, (void*)&mu, (void*)&h->dS, (void*)&h->slabs[0].partials,
                    (void*)&h->gbar, (void*)&spec, (void*)&XR};
    const void* fn;
    if (h->xr_emu || h->xr_real) {
        if (h->sb) fn = h->bb ? (const void*)k6_gp_loop_ms<true, true, true> : (const void*)k6_gp_loop_ms<true, false, true>;
        else fn = h->bb ? (const void*)k6_gp_loop_ms<false, true, true> : (const void*)k6_gp_loop_ms<false, false, true>;
    } else {
        if (h->sb) fn = h->bb ? (const void*)k6_gp_loop_ms<true, true, false> : (const void*)k6_gp_loop_ms<true, false, false>;
        else fn = h->bb ? (const void*)k6_gp_loop_ms<false, true, false> : (const void*)k6_gp_loop_ms<false, false, false>;
    }
    CK(cudaLaunchCooperativeKernel(fn, dim3(cta), dim3(m4::kThreads), args, h->smem6_gp, h->st));
    h->launches++;
    return GPCG_OK;
}

int launch_gp_loop(gpcg_problem* h, int cur) {
    if (h->nslabs() > 1 || h->xr_real) return launch_gp_loop_ms(h, cur);
    Slab& S = h->slabs[0];
    CK(cudaMemsetAsync(h->gbar, 0, sizeof(unsigned int), h->st));
    Bounds B = h->bounds(S);
    double mu = h->prm.mu;
    int spec = h->gp_spec ? 1 : 0;
    void* args[] = {(void*)&S.sop, (void*)&S.bg5_srch, (void*)&S.bg5_acc, (void*)&B, (void*)&S.brow,
                    (void*)&S.t5[VY0], (void*)&S.t5[VY1], (void*)&S.t5[VB], (void*)&S.t5[VL], (void*)&S.t5[VU],
                    (void*)&S.t5m[MK0], (void*)&S.t5m[MK1], (void*)&S.v[VY0], (void*)&S.v[VY1], (void*)&S.m[MK0],
                    (void*)&S.m[MK1], (void*)&cur, (void*)&mu, (void*)&h->dS, (void*)&S.partials, (void*)&h->gbar,
                    (void*)&spec};
    const void* fn;
    if (h->sb) fn = h->bb ? (const void*)k6_gp_loop<true, true> : (const void*)k6_gp_loop<true, false>;
    else fn = h->bb ? (const void*)k6_gp_loop<false, true> : (const void*)k6_gp_loop<false, false>;
    CK(cudaLaunchCooperativeKernel(fn, dim3(h->grid6_gp), dim3(m4::kThreads), args, h->smem6_gp, h->st));
    h->launches++;
    return GPCG_OK;
}

// kernels per CG iteration (for the launch count)
int launches_per_cg_iter(const gpcg_problem* h) {
    int n = h->nslabs();
    if (h->deferred) n += 1 + (h->nslabs() > 1 ? 1 : 0);
    return n;
}

// ---------------------------------------------------------------- explicit extraction (cg_mode = 1)
// The extraction ablation (the paper's MatGetSubMatrix route):
// build A_F = Z'AZ as an m x m CSR and r_F, run CG on the compact system with the CSR kernels,
// scatter w back.  One slab, one rank.
int ensure_extract_buffers(gpcg_problem* h, Slab& S) {
    if (S.xarena) return GPCG_OK;
    const long long n = S.rows * (long long)h->rowlen;
    long long nnzmax = 0;                     // stored entries of the operator bound those of A_F
    if (h->is_csr) {
        long long last = 0;
        CK(cudaMemcpy(&last, S.rp + S.rows, sizeof(long long), cudaMemcpyDeviceToHost));
        nnzmax = last;
    } else {
        nnzmax = (h->is3d ? 7 : 5) * n;
    }
    const long long nblk = (n + kScanBlock - 1) / kScanBlock;
    auto r256 = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t b_idx = r256((size_t)S.nalloc * 4), b_pos = r256((size_t)n * 4), b_cnt = r256((size_t)n * 4);
    const size_t b_col = r256((size_t)nnzmax * 4), b_blk = r256((size_t)(nblk + 1) * 8), b_tot = 256;
    const size_t b_rp = r256((size_t)(n + 1) * 8), b_val = r256((size_t)nnzmax * 8), b_vec = r256((size_t)n * 8);
    const size_t b_msk = r256((size_t)n);
    const size_t total = b_idx + b_pos + b_cnt + b_col + b_blk + b_tot + b_rp + b_val + 12 * b_vec + 2 * b_msk;
    CK(dalloc(h, &S.xarena, total));
    CK(cudaMemsetAsync(S.xarena, 0, total, h->st));
    char* p = static_cast<char*>(S.xarena);
    S.xidx = reinterpret_cast<int*>(p) + (long long)S.glo * h->pitch; p += b_idx;   // indexed by v (ghosts incl.)
    S.xpos = reinterpret_cast<int*>(p); p += b_pos;
    S.xcnt = reinterpret_cast<int*>(p); p += b_cnt;
    S.xcol = reinterpret_cast<int*>(p); p += b_col;
    S.xblk = reinterpret_cast<long long*>(p); p += b_blk;
    S.xtot = reinterpret_cast<long long*>(p); p += b_tot;
    S.xrp = reinterpret_cast<long long*>(p); p += b_rp;
    S.xval = reinterpret_cast<double*>(p); p += b_val;
    for (int k = 0; k < 12; ++k) { S.xv[k] = reinterpret_cast<double*>(p); p += b_vec; }
    S.xmask = reinterpret_cast<unsigned char*>(p); p += b_msk;
    S.xmaskcg = reinterpret_cast<unsigned char*>(p);
    CK(cudaMemsetAsync(S.xmask, 1, (size_t)n, h->st));                     // every compact row is free
    return GPCG_OK;
}

// ---------------------------------------------------------------- compacted free-row list (a4 (iii))
// F of mask mk, in owned-point order, by the deterministic scans of extract.cuh; S.fcount = |F|
// (read back: the callers synchronise anyway).
int build_free_list(gpcg_problem* h, Slab& S, int mk) {
    const long long n = S.rows * (long long)h->rowlen;
    const long long nblk = (n + kScanBlock - 1) / kScanBlock;
    if (!S.flist) {
        CK(dalloc(h, &S.flist, (size_t)std::max<long long>(n, 1) * sizeof(int)));
        CK(dalloc(h, &S.fblk, (size_t)(nblk + 1) * sizeof(long long)));
        CK(dalloc(h, &S.ftot, sizeof(long long)));
        CK(dalloc(h, &S.fbits, (size_t)((n + 31) / 32 + 1) * sizeof(unsigned)));
        if (h->pitch == h->rowlen) CK(dalloc(h, &S.fpos, (size_t)std::max<long long>(n, 1) * sizeof(int)));
    }
    k_scan_count<true><<<(unsigned)nblk, 256, 0, h->st>>>(n, h->rowlen, h->pitch, S.m[mk], nullptr, S.fblk);
    k_scan_blocks<<<1, 1024, 0, h->st>>>(nblk, S.fblk, S.ftot);
    k_scan_assign<<<(unsigned)nblk, 256, 0, h->st>>>(n, h->rowlen, h->pitch, S.m[mk], S.fblk, S.fpos, S.flist);
    if (h->pitch == h->rowlen)      // contiguous owned points (CSR, 3-D): the free bits for the reduced products
        k_pack_bits<<<(unsigned)((n + kThreads - 1) / kThreads), kThreads, 0, h->st>>>(n, S.m[mk], S.fbits);
    CKLAUNCH();
    h->launches += 4;
    long long m = 0;
    CK(cudaMemcpyAsync(&m, S.ftot, sizeof(long long), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    S.fcount = m;
    S.fmask = mk;
    return GPCG_OK;
}

// the compact (free-row list) regime: CSR / 3-D operator, one slab on one rank, |F| < 0.3 n
bool compact_ok(const gpcg_problem* h) { return !spec2d(h) && h->nslabs() == 1 && h->nranks == 1 && !h->deferred; }

// CG on A_F applied in place over the free-row list (cg_mode 3, and cg_mode 2 for small free
// sets): the C-G recurrences of k_cg_init / k_cg_iter on the free rows only, the vectors in the
// reduced space (m entries), no copy of A's values.  On return W holds w (zero off F).
int run_cg_compact(gpcg_problem* h, int cur, double eta2, long long cap, long long* iters) {
    if (!compact_ok(h))
        return set_err(GPCG_EINVAL, "cg_mode = 3 (free-row list) supports CSR / 3-D operators on one slab and rank");
    Slab& S = h->slabs[0];
    CK(cudaEventRecord(h->ev_c0, h->st));
    RC(build_free_list(h, S, cur));
    const long long n = S.rows * (long long)h->rowlen;
    const long long mm = S.fcount;
    if (mm > S.cv_cap) {                           // reduced-space vectors, grown on demand
        dfree(h, S.cv);
        S.cv = nullptr;
        S.cv_cap = std::min<long long>(n, mm + mm / 4 + 1024);
        CK(dalloc(h, &S.cv, (size_t)8 * S.cv_cap * sizeof(double)));
    }
    double* cvv[8];
    for (int k = 0; k < 8; ++k) cvv[k] = S.cv + (size_t)k * S.cv_cap;
    double *rho2[2] = {cvv[0], cvv[1]}, *q2[2] = {cvv[2], cvv[3]}, *s2[2] = {cvv[4], cvv[5]};
    double *pc_ = cvv[6], *wc = cvv[7];
    CK(cudaMemsetAsync(S.v[VW], 0, (size_t)n * sizeof(double), h->st));       // w = 0 off F
    CK(cudaEventRecord(h->ev_c1, h->st));
    CK(cudaEventSynchronize(h->ev_c1));
    float ms_x = 0.f;
    CK(cudaEventElapsedTime(&ms_x, h->ev_c0, h->ev_c1));
    h->t_extract_ms += ms_x;
    if (mm <= 0) { *iters = 0; return GPCG_OK; }
    const int g = (int)std::max<long long>(1, std::min<long long>((mm + kThreads - 1) / kThreads, (long long)h->sms * 16));
    const bool pc = h->prm.precond == 1;
    const RedScratch R = h->red(0);
    with_gop(h, S, [&](auto& op) {
        using Op = std::decay_t<decltype(op)>;
        if (pc)
            k_cg_init_c<Op, true><<<g, kThreads, 0, h->st>>>(op, mm, S.flist, S.fbits, S.v[vg(cur)], rho2[0], q2[0],
                                                             s2[0], pc_, wc, S.v[VD], eta2, cap, h->dS, R);
        else
            k_cg_init_c<Op, false><<<g, kThreads, 0, h->st>>>(op, mm, S.flist, S.fbits, S.v[vg(cur)], rho2[0], q2[0],
                                                              s2[0], pc_, wc, S.v[VD], eta2, cap, h->dS, R);
    });
    CKLAUNCH();
    h->launches++;
    // chunks of 4, 8, 16, ... iterations up to cg_chunk: short CG calls (C4: 3-4 iterations) launch
    // few no-op iterations, long ones poll as rarely as before
    const int chunk_max = std::max(2, (h->prm.cg_chunk + 1) & ~1);
    int chunk = std::min(4, chunk_max);
    long long it_prev = 0;                      // k_cg_init_c set cg_it = 0
    for (;; chunk = std::min(2 * chunk, chunk_max)) {
        CK(cudaEventRecord(h->ev_c0, h->st));
        for (int i = 0; i < chunk; ++i) {
            const int a = i & 1, bb = a ^ 1;
            with_gop(h, S, [&](auto& op) {
                using Op = std::decay_t<decltype(op)>;
                if (pc)
                    k_cg_iter_c<Op, true><<<g, kThreads, 0, h->st>>>(op, mm, S.flist, S.fbits, S.fpos, rho2[a], q2[a],
                                                                     s2[a], rho2[bb], q2[bb], s2[bb], pc_, wc,
                                                                     S.v[VD], h->dS, R);
                else
                    k_cg_iter_c<Op, false><<<g, kThreads, 0, h->st>>>(op, mm, S.flist, S.fbits, S.fpos, rho2[a],
                                                                      q2[a], s2[a], rho2[bb], q2[bb], s2[bb], pc_, wc,
                                                                      S.v[VD], h->dS, R);
            });
        }
        CKLAUNCH();
        CK(cudaEventRecord(h->ev_c1, h->st));
        h->launches += chunk;
        RC(sync_scal(h));
        // per-iteration timing over every chunk (C4's calls end inside their first chunk): the
        // iterations the chunk ran, its no-op launches included
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev_c0, h->ev_c1));
        const long long ran = h->hS->cg_it - it_prev;
        it_prev = h->hS->cg_it;
        if (ran > 0) {
            h->t_cg_timed_ms += ms;
            h->cg_iters_timed += ran;
            h->cg_free_iters_timed += ran * mm;
        }
        if (h->hS->cg_done) break;
    }
    k_scatter_free<<<(unsigned)((mm + kThreads - 1) / kThreads), kThreads, 0, h->st>>>(mm, S.flist, wc, S.v[VW]);
    CKLAUNCH();
    h->launches++;
    *iters = h->hS->cg_it;
    if (h->hS->cg_reason == CG_NOTSPD)
        return set_err(GPCG_ENOTSPD, "CG breakdown: <p, A_k p> <= 0 at iteration %lld (A not SPD)",
                       (long long)h->hS->cg_it);
    return GPCG_OK;
}

int run_cg_extract(gpcg_problem* h, int cur, double eta2, long long cap, long long* iters) {
    if (h->nslabs() != 1 || h->nranks != 1 || h->deferred)
        return set_err(GPCG_EINVAL, "cg_mode = 1 (explicit extraction) supports one slab on one rank");
    Slab& S = h->slabs[0];
    RC(ensure_extract_buffers(h, S));
    const long long n = S.rows * (long long)h->rowlen;
    const long long nblk = (n + kScanBlock - 1) / kScanBlock;
    const unsigned char* mask = S.m[cur];
    CK(cudaEventRecord(h->ev_c0, h->st));
    // compact numbering of F
    k_scan_count<true><<<(unsigned)nblk, 256, 0, h->st>>>(n, h->rowlen, h->pitch, mask, nullptr, S.xblk);
    k_scan_blocks<<<1, 1024, 0, h->st>>>(nblk, S.xblk, S.xtot);
    k_scan_assign<<<(unsigned)nblk, 256, 0, h->st>>>(n, h->rowlen, h->pitch, mask, S.xblk, S.xidx, S.xpos);
    CKLAUNCH();
    long long mm = 0;
    CK(cudaMemcpyAsync(&mm, S.xtot, sizeof(long long), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (mm <= 0) { *iters = 0; return GPCG_OK; }
    const int g = (int)std::min<long long>((mm + kThreads - 1) / kThreads, (long long)h->sms * 16);
    // row pointers of A_F
    with_gop(h, S, [&](auto& op) {
        using Op = std::decay_t<decltype(op)>;
        k_extract_count<Op><<<g, kThreads, 0, h->st>>>(op, mm, S.xpos, mask, S.xcnt);
    });
    const long long mblk = (mm + kScanBlock - 1) / kScanBlock;
    k_scan_count<false><<<(unsigned)mblk, 256, 0, h->st>>>(mm, 1, 1, nullptr, S.xcnt, S.xblk);
    k_scan_blocks<<<1, 1024, 0, h->st>>>(mblk, S.xblk, S.xtot);
    k_scan_assign_vals<<<(unsigned)mblk, 256, 0, h->st>>>(mm, S.xcnt, S.xblk, S.xrp);
    CK(cudaMemcpyAsync(S.xrp + mm, S.xtot, sizeof(long long), cudaMemcpyDeviceToDevice, h->st));
    // A_F, r_F (recomputed from y: works with or without stored g), 1/diag on F
    with_gop(h, S, [&](auto& op) {
        using Op = std::decay_t<decltype(op)>;
        k_extract_fill<Op><<<g, kThreads, 0, h->st>>>(op, mm, S.xpos, mask, S.xidx, S.xrp, S.xcol, S.xval,
                                                      S.v[vy(cur)], S.v[VB], S.v[VD], S.xv[0], S.xv[1]);
    });
    CKLAUNCH();
    CK(cudaEventRecord(h->ev_c1, h->st));
    h->launches += 8;
    // CG on the compact system (CSR kernels, all rows free)
    const CsrOp cop{(int)mm, S.xrp, S.xcol, S.xval};
    const bool pc = h->prm.precond == 1;
    const RedScratch R = h->red(0);
    double* rho[2] = {S.xv[2], S.xv[3]};
    double* q[2] = {S.xv[4], S.xv[5]};
    double* sv[2] = {S.xv[6], S.xv[7]};
    double* pv = S.xv[8];
    double* wv = S.xv[9];
    if (pc)
        k_cg_init<CsrOp, true><<<g, kThreads, 0, h->st>>>(cop, S.xv[0], S.xmask, S.xmaskcg, rho[0], q[0], sv[0], rho[1],
                                                          q[1], sv[1], pv, wv, S.xv[1], eta2, cap, h->dS, R);
    else
        k_cg_init<CsrOp, false><<<g, kThreads, 0, h->st>>>(cop, S.xv[0], S.xmask, S.xmaskcg, rho[0], q[0], sv[0], rho[1],
                                                           q[1], sv[1], pv, wv, S.xv[1], eta2, cap, h->dS, R);
    CKLAUNCH();
    h->launches++;
    const int chunk = std::max(2, (h->prm.cg_chunk + 1) & ~1);
    float ms_x = 0.f;
    CK(cudaEventSynchronize(h->ev_c1));
    CK(cudaEventElapsedTime(&ms_x, h->ev_c0, h->ev_c1));
    h->t_extract_ms += ms_x;
    for (;;) {
        CK(cudaEventRecord(h->ev_c0, h->st));
        for (int i = 0; i < chunk; ++i) {
            const int a = i & 1, bb = a ^ 1;
            if (pc)
                k_cg_iter<CsrOp, true><<<g, kThreads, 0, h->st>>>(cop, S.xmaskcg, rho[a], q[a], sv[a], rho[bb], q[bb],
                                                                  sv[bb], pv, wv, S.xv[1], h->dS, R);
            else
                k_cg_iter<CsrOp, false><<<g, kThreads, 0, h->st>>>(cop, S.xmaskcg, rho[a], q[a], sv[a], rho[bb], q[bb],
                                                                   sv[bb], pv, wv, S.xv[1], h->dS, R);
        }
        CKLAUNCH();
        CK(cudaEventRecord(h->ev_c1, h->st));
        h->launches += chunk;
        RC(sync_scal(h));
        if (h->hS->cg_done) break;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev_c0, h->ev_c1));
        h->t_cg_timed_ms += ms;
        h->cg_iters_timed += chunk;
        h->cg_free_iters_timed += chunk * mm;
    }
    *iters = h->hS->cg_it;
    if (h->hS->cg_reason == CG_NOTSPD)
        return set_err(GPCG_ENOTSPD, "CG breakdown: <p, A_k p> <= 0 at iteration %lld (A not SPD)",
                       (long long)h->hS->cg_it);
    // w = Z w_F
    const int gs = (int)std::min<long long>((n + kThreads - 1) / kThreads, (long long)h->sms * 16);
    k_scatter<<<gs, kThreads, 0, h->st>>>(n, h->rowlen, h->pitch, mask, S.xidx, wv, S.v[VW]);
    CKLAUNCH();
    h->launches++;
    return GPCG_OK;
}

// ---------------------------------------------------------------- block-Jacobi ILU(0) PCG (precond = 2)
// Vectors: r = RHO0, z = RHO1, p = Q0 / Q1 (ping-pong), q = S0, w = W; the factor in Slab::bjf.
long long bj_tiles(const gpcg_problem* h, const Slab& S) {
    return (long long)((h->nx + kTile - 1) / kTile) * ((S.rows + kTile - 1) / kTile);
}

int bj_grid_tiles(const gpcg_problem* h, const Slab& S) {
    const int wpc = kBjThreads / 32;
    return (int)std::max<long long>(1, std::min<long long>((bj_tiles(h, S) + wpc - 1) / wpc, (long long)h->sms * 16));
}

int bj_grid_mv(const gpcg_problem* h, const Slab& S) {
    return (int)std::max<long long>(1, std::min<long long>(bj_tiles(h, S), (long long)h->sms * 8));
}

// broadcast faces: dinv + code bytes (the cs / cw arrays unused); else dinv, cs, cw
BjFactor bj_factor(const gpcg_problem* h, const Slab& S, long long nt) {
    const long long e = nt * kTile * kTile;
    unsigned char* code = h->bc ? reinterpret_cast<unsigned char*>(S.bjf + 5 * e) : nullptr;
    return BjFactor{S.bjf, S.bjf + e, S.bjf + 2 * e, code};
}

// ILU(2): l_S, l_SE, l_SEE, l_W, 1/d in the same storage
Bj2Factor bj2_factor(const Slab& S, long long nt) {
    const long long e = nt * kTile * kTile;
    return Bj2Factor{S.bjf, S.bjf + e, S.bjf + 2 * e, S.bjf + 3 * e, S.bjf + 4 * e};
}

int enqueue_bj_iter(gpcg_problem* h, int a) {
    const int bb = a ^ 1;
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        if (h->generic)
            k_pcg2_matvec<<<S.grid, kThreads, 0, h->st>>>(S.sop, S.m[MKCG], S.v[VRHO1], S.v[vq(a)], S.v[vq(bb)],
                                                          S.v[VS0], S.v[VW], h->dS, h->red(s));
        else
            k_pcg2_matvec_tile<<<bj_grid_mv(h, S), kMvThreads, 0, h->st>>>(S.sop, S.m[MKCG], S.v[VRHO1], S.v[vq(a)],
                                                                          S.v[vq(bb)], S.v[VS0], S.v[VW], h->dS,
                                                                          h->red(s));
        CKLAUNCH();
    }
    RC(finish_reduce(h, fin(FIN_PCG2_ALPHA), 1));
    RC(exchange(h, {vq(bb)}));
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        if (h->prm.precond == 3)
            k_pcg3_solve<1><<<bj_grid_tiles(h, S), kBjThreads, kSolveSmem, h->st>>>(S.sop, bj2_factor(S, bj_tiles(h, S)), S.tbr,
                                                                                 S.glo, S.v[VRHO0], S.v[VS0], S.v[VRHO1],
                                                                                 0.0, 0, h->dS, h->red(s));
        else if (h->bc)
            k_pcg2_solve<1, true><<<bj_grid_tiles(h, S), kBjThreads, kSolveSmem, h->st>>>(S.sop, bj_factor(h, S, bj_tiles(h, S)), S.tbr,
                                                                              S.glo, S.v[VRHO0], S.v[VS0], S.v[VRHO1],
                                                                              0.0, 0, h->dS, h->red(s));
        else
            k_pcg2_solve<1, false><<<bj_grid_tiles(h, S), kBjThreads, kSolveSmem, h->st>>>(S.sop, bj_factor(h, S, bj_tiles(h, S)), S.tbr,
                                                                              S.glo, S.v[VRHO0], S.v[VS0], S.v[VRHO1],
                                                                              0.0, 0, h->dS, h->red(s));
        CKLAUNCH();
    }
    RC(finish_reduce(h, fin(FIN_PCG2_BETA), 1));
    return exchange(h, {VRHO1});
}

int run_cg_bjilu(gpcg_problem* h, int cur, long long m, double eta2, long long cap, long long* iters) {
    if (h->is_csr || h->is3d)
        return set_err(GPCG_EINVAL, "precond = 2 / 3 (block-Jacobi ILU(0) / ILU(2)) is implemented for 2-D stencils");
    const bool ilu2 = h->prm.precond == 3;
    RC(set_smem(k_bjilu_factor, kFactorSmem));
    RC(set_smem(k_bjilu2_factor, kBj2FactorSmem));
    RC(set_smem(k_pcg3_solve<0>, kSolveSmem));
    RC(set_smem(k_pcg3_solve<1>, kSolveSmem));
    RC(set_smem(k_pcg2_solve<0, false>, kSolveSmem));
    RC(set_smem(k_pcg2_solve<1, false>, kSolveSmem));
    RC(set_smem(k_pcg2_solve<0, true>, kSolveSmem));
    RC(set_smem(k_pcg2_solve<1, true>, kSolveSmem));
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const long long nt = bj_tiles(h, S);
        if (!S.bjf) {
            CK(dalloc(h, &S.bjf, (size_t)5 * nt * kTile * kTile * sizeof(double) + (size_t)nt * kTile * kTile));
            RC(make_map(h, S, &S.tbr, S.v[VRHO0], false, kTile, kTile));
        }
        k_pcg2_init<<<S.grid, kThreads, 0, h->st>>>(S.sop, S.v[vy(cur)], S.v[VB], S.m[cur], S.m[MKCG], S.v[VRHO0],
                                                    S.v[VQ0], S.v[VQ1], S.v[VW]);
        CKLAUNCH();
        if (ilu2) {
            const int gw = (int)std::max<long long>(1, std::min<long long>((nt + kBj2FactorWarps - 1) / kBj2FactorWarps,
                                                                           (long long)h->sms * 8));
            k_bjilu2_factor<<<gw, 32 * kBj2FactorWarps, kBj2FactorSmem, h->st>>>(S.sop, S.m[MKCG], bj2_factor(S, nt));
            CKLAUNCH();
            k_pcg3_solve<0><<<bj_grid_tiles(h, S), kBjThreads, kSolveSmem, h->st>>>(S.sop, bj2_factor(S, nt), S.tbr, S.glo,
                                                                                 S.v[VRHO0], S.v[VS0], S.v[VRHO1], eta2,
                                                                                 cap, h->dS, h->red(s));
        } else {
        k_bjilu_factor<<<bj_grid_tiles(h, S), kBjThreads, kFactorSmem, h->st>>>(S.sop, S.m[MKCG], bj_factor(h, S, nt));
        CKLAUNCH();
        if (h->bc)
            k_pcg2_solve<0, true><<<bj_grid_tiles(h, S), kBjThreads, kSolveSmem, h->st>>>(S.sop, bj_factor(h, S, nt), S.tbr, S.glo,
                                                                              S.v[VRHO0], S.v[VS0], S.v[VRHO1], eta2,
                                                                              cap, h->dS, h->red(s));
        else
            k_pcg2_solve<0, false><<<bj_grid_tiles(h, S), kBjThreads, kSolveSmem, h->st>>>(S.sop, bj_factor(h, S, nt), S.tbr, S.glo,
                                                                              S.v[VRHO0], S.v[VS0], S.v[VRHO1], eta2,
                                                                              cap, h->dS, h->red(s));
        }
        CKLAUNCH();
        h->launches += 3;
    }
    FinArgs a = fin(FIN_PCG2_INIT);
    a.eta2 = eta2;
    a.cap = cap;
    RC(finish_reduce(h, a, 1));
    RC(exchange(h, {VRHO1, VQ0, VQ1}, {MKCG}));
    const int chunk = std::max(2, (h->prm.cg_chunk + 1) & ~1);
    if (!h->bj_exec || h->bj_exec_chunk != chunk || h->bj_exec_pc != h->prm.precond) {
        if (h->bj_exec) { cudaGraphExecDestroy(h->bj_exec); h->bj_exec = nullptr; }
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
        const long long l0 = h->launches;
        int rc = GPCG_OK;
        for (int i = 0; i < chunk && !rc; ++i) rc = enqueue_bj_iter(h, i & 1);
        h->launches = l0;
        cudaError_t e = cudaStreamEndCapture(h->st, &graph);
        if (rc) { if (e == cudaSuccess) cudaGraphDestroy(graph); return rc; }
        if (e != cudaSuccess) return set_err(GPCG_ECUDA, "graph capture: %s", cudaGetErrorString(e));
        e = cudaGraphInstantiate(&h->bj_exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return set_err(GPCG_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
        h->bj_exec_chunk = chunk;
        h->bj_exec_pc = h->prm.precond;
    }
    const int per_iter = 2 * h->nslabs() + (h->deferred ? 2 * (1 + (h->nslabs() > 1 ? 1 : 0)) : 0);
    for (;;) {
        CK(cudaEventRecord(h->ev_c0, h->st));
        CK(cudaGraphLaunch(h->bj_exec, h->st));
        CK(cudaEventRecord(h->ev_c1, h->st));
        h->launches += (long long)chunk * per_iter;
        RC(sync_scal(h));
        if (h->hS->cg_done) break;
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
    // the last iteration's w += alpha p (iteration j wrote p_j into Q[j & 1]; chunks are even)
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        k_pcg2_wlast<<<S.grid, kThreads, 0, h->st>>>(S.sop, S.v[vq((int)(h->hS->cg_it & 1))], S.v[VW], h->dS);
        CKLAUNCH();
        h->launches++;
    }
    return exchange(h, {VW});
}

// CG on the free set of M[cur].  On return W holds w_{j_k}.
int run_cg(gpcg_problem* h, int cur, long long m, double eta2, long long cap, long long* iters) {
    if (h->prm.precond >= 2) return run_cg_bjilu(h, cur, m, eta2, cap, iters);
    // cg_mode 1: always extract; 2 (auto): extract for the generic kernels (CSR, 3-D) when the
    // free set is small (m < 0.3 n), where the compact system wins
    if (h->prm.cg_mode == 1) return run_cg_extract(h, cur, eta2, cap, iters);
    if (h->prm.cg_mode == 3 || (h->prm.cg_mode == 2 && compact_ok(h) && 10 * m < 3 * h->n_global))
        return run_cg_compact(h, cur, eta2, cap, iters);
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const RedScratch R = h->red(s);
        const bool pc = h->prm.precond == 1;
        if (h->gfree) {
            auto go = [&](auto bbt, auto pct) {
                constexpr bool BB = decltype(bbt)::value, PC = decltype(pct)::value;
                k5_cg_init<BB, PC><<<S.grid5_init, m4::kThreads, CgInitLayout5<BB>::kSmem, h->st>>>(
                    S.sop, S.bg5_init, S.brow, S.t5[vy(cur)], S.t5[VB], S.t5m[cur], S.m[MKCG], S.v[VRHO0], S.v[VQ0],
                    S.v[VW], eta2, cap, h->dS, R);
            };
            if (h->bb) { if (pc) go(std::true_type(), std::true_type()); else go(std::true_type(), std::false_type()); }
            else { if (pc) go(std::false_type(), std::true_type()); else go(std::false_type(), std::false_type()); }
        } else if (spec2d(h)) {
            auto go = [&](auto bct, auto pct) {
                constexpr bool BC = decltype(bct)::value, PC = decltype(pct)::value;
                k2_cg_init<BC, PC><<<S.grid_m1, kMarchThreads, 0, h->st>>>(S.sop, S.mg1, S.v[vg(cur)], S.m[cur],
                                                                           S.m[MKCG], S.v[VRHO0], S.v[VQ0], S.v[VW],
                                                                           eta2, cap, h->dS, R);
            };
            if (h->bc) { if (pc) go(std::true_type(), std::true_type()); else go(std::true_type(), std::false_type()); }
            else { if (pc) go(std::false_type(), std::true_type()); else go(std::false_type(), std::false_type()); }
        } else if (use_m3(h)) {
            auto go = [&](auto pct) {
                constexpr bool PC = decltype(pct)::value;
                k7_cg_init<PC><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, S.v[vg(cur)], S.m[cur], S.m[MKCG], S.v[VRHO0],
                                                                    S.v[VQ0], S.v[VS0], S.v[VRHO1], S.v[VQ1], S.v[VS1],
                                                                    S.v[VP], S.v[VW], S.v[VD], eta2, cap, h->dS, R);
            };
            if (pc) go(std::true_type()); else go(std::false_type());
        } else {
            with_gop(h, S, [&](auto& op) {
                using Op = std::decay_t<decltype(op)>;
                auto go = [&](auto pct) {
                    constexpr bool PC = decltype(pct)::value;
                    k_cg_init<Op, PC><<<S.grid, kThreads, 0, h->st>>>(op, S.v[vg(cur)], S.m[cur], S.m[MKCG],
                                                                      S.v[VRHO0], S.v[VQ0], S.v[VS0], S.v[VRHO1],
                                                                      S.v[VQ1], S.v[VS1], S.v[VP], S.v[VW], S.v[VD],
                                                                      eta2, cap, h->dS, R);
                };
                if (pc) go(std::true_type()); else go(std::false_type());
            });
        }
        h->launches++;
        CKLAUNCH();
    }
    FinArgs a = fin(FIN_CG_INIT);
    a.eta2 = eta2;
    a.cap = cap;
    RC(finish_reduce(h, a, 2));
    if (!spec2d(h)) RC(exchange(h, {VRHO0, VQ0, VS0}, {MKCG}));
    else RC(exchange(h, {VRHO0, VQ0}, {MKCG}));
    if (h->tile && (h->tile_mask & 8) && h->cg_skip) {
        for (Slab& S : h->slabs) {
            const long long nf = (long long)S.bg_cg.nbands * S.bg_cg.nsegs * ((S.bg_cg.seg + 4 + m4::kBR - 1) / m4::kBR);
            const int g = (int)std::min<long long>((nf * 32 + 255) / 256, (long long)h->sms * 8);
            k_cg_block_flags<<<std::max(g, 1), 256, 0, h->st>>>(h->nx, h->pitch, S.bg_cg, S.m[MKCG], S.rows + S.ghi,
                                                                S.cgflags);
            h->launches++;
            CKLAUNCH();
        }
    }
    if (h->cg_persistent && h->tile && (h->tile_mask & 8) && !h->deferred) {
        // one cooperative launch runs the whole CG call (k6_cg_loop)
        Slab& S = h->slabs[0];
        const unsigned short* flags = h->cg_skip ? S.cgflags : nullptr;
        CK(cudaMemsetAsync(h->gbar, 0, sizeof(unsigned int), h->st));
        CK(cudaEventRecord(h->ev_c0, h->st));
        const bool pw = h->cg_pw;
        int pwi = pw ? 1 : 0;
        void* args[] = {(void*)&S.sop, (void*)&S.bg_cg, (void*)(pw ? &S.t4c[0] : &S.t4[VRHO0]),
                        (void*)(pw ? &S.t4c[1] : &S.t4[VRHO1]), (void*)(pw ? &S.t4c[2] : &S.t4[VQ0]),
                        (void*)(pw ? &S.t4c[3] : &S.t4[VQ1]), (void*)(pw ? &S.t4cw : &S.t4wo), (void*)&S.t4m[MKCG],
                        (void*)&S.v[VRHO0],
                        (void*)&S.v[VRHO1], (void*)&S.v[VQ0], (void*)&S.v[VQ1], (void*)&S.v[VW], (void*)&h->dS,
                        (void*)&S.partials, (void*)&h->gbar, (void*)&flags, (void*)&pwi};
        const void* fn = h->prm.precond == 1 ? (const void*)k6_cg_loop<true> : (const void*)k6_cg_loop<false>;
        CK(cudaLaunchCooperativeKernel(fn, dim3(S.grid4_cg), dim3(m4::kThreadsWS), args, (size_t)m4cg::kSmem, h->st));
        CK(cudaEventRecord(h->ev_c1, h->st));
        h->launches++;
        RC(sync_scal(h));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev_c0, h->ev_c1));
        h->t_cg_timed_ms += ms;
        h->cg_iters_timed += h->hS->cg_it;
        h->cg_free_iters_timed += h->hS->cg_it * m;
        *iters = h->hS->cg_it;
        if (h->hS->cg_reason == CG_NOTSPD)
            return set_err(GPCG_ENOTSPD, "CG breakdown: <p, A_k p> <= 0 at iteration %lld (A not SPD)",
                           (long long)h->hS->cg_it);
        return GPCG_OK;    // one slab: no ghosts of w to refresh
    }
    if (h->cg_persistent && h->tile && (h->tile_mask & 8) && multi_slab_persistent(h)) {
        // one cooperative launch over every slab (k6_cg_loop_ms, fused halo writes)
        CgMsArgs P;
        memset(&P, 0, sizeof P);
        P.nslabs = h->nslabs();
        P.pw = h->cg_pw ? 1 : 0;
        int cta = 0;
        for (int s = 0; s < h->nslabs(); ++s) {
            Slab& S = h->slabs[s];
            CgMsSlab& X = P.s[s];
            if (h->cg_pw) {
                X.m_rho0 = S.t4c[0]; X.m_rho1 = S.t4c[1]; X.m_p0 = S.t4c[2]; X.m_p1 = S.t4c[3];
                X.m_w = S.t4cw;
            } else {
                X.m_rho0 = S.t4[VRHO0]; X.m_rho1 = S.t4[VRHO1]; X.m_p0 = S.t4[VQ0]; X.m_p1 = S.t4[VQ1];
                X.m_w = S.t4wo;
            }
            X.m_mask = S.t4m[MKCG];
            X.A = S.sop;
            X.G = S.bg_cg;
            X.rho0 = S.v[VRHO0]; X.rho1 = S.v[VRHO1]; X.p0 = S.v[VQ0]; X.p1 = S.v[VQ1]; X.w = S.v[VW];
            X.flags = h->cg_skip ? S.cgflags : nullptr;
            X.L = SlabLink{0, S.grid4_cg, 0, 0, 0};
            XrSide N;
            if (neighbour_side(h, S, true, &N)) {
                X.lo_rho0 = N.v[0]; X.lo_rho1 = N.v[1]; X.lo_p0 = N.v[2]; X.lo_p1 = N.v[3];
                X.L.lo_rows = N.rows;
                X.L.lo_ghost = N.ghi;
            }
            if (neighbour_side(h, S, false, &N)) {
                X.hi_rho0 = N.v[0]; X.hi_rho1 = N.v[1]; X.hi_p0 = N.v[2]; X.hi_p1 = N.v[3];
                X.L.hi_ghost = N.glo;
            }
            X.cta0 = cta;
            cta += S.grid4_cg;
        }
        int c0[kMaxMs];
        for (int s = 0; s < h->nslabs(); ++s) c0[s] = P.s[s].cta0;
        XRank XR;
        RC(make_xrank(h, c0, h->nslabs(), cta, &XR, true));
        CK(cudaMemsetAsync(h->gbar, 0, sizeof(unsigned int), h->st));
        CK(cudaEventRecord(h->ev_c0, h->st));
        void* args[] = {(void*)&P, (void*)&h->dS, (void*)&h->slabs[0].partials, (void*)&h->gbar, (void*)&XR};
        const void* fn = (h->xr_emu || h->xr_real) ? (h->prm.precond == 1 ? (const void*)k6_cg_loop_ms<true, true>
                                                            : (const void*)k6_cg_loop_ms<false, true>)
                                   : (h->prm.precond == 1 ? (const void*)k6_cg_loop_ms<true, false>
                                                            : (const void*)k6_cg_loop_ms<false, false>);
        CK(cudaLaunchCooperativeKernel(fn, dim3(cta), dim3(m4::kThreadsWS), args, (size_t)m4cg::kSmem, h->st));
        CK(cudaEventRecord(h->ev_c1, h->st));
        h->launches++;
        RC(sync_scal(h));
        RC(check_xrank(h));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, h->ev_c0, h->ev_c1));
        h->t_cg_timed_ms += ms;
        h->cg_iters_timed += h->hS->cg_it;
        h->cg_free_iters_timed += h->hS->cg_it * m;
        *iters = h->hS->cg_it;
        if (h->hS->cg_reason == CG_NOTSPD)
            return set_err(GPCG_ENOTSPD, "CG breakdown: <p, A_k p> <= 0 at iteration %lld (A not SPD)",
                           (long long)h->hS->cg_it);
        // the search along d = w reads w at the neighbours
        return exchange(h, {VW});
    }
    const int chunk = std::max(2, (h->prm.cg_chunk + 1) & ~1);
    RC(build_cg_graph(h, chunk));
    for (;;) {
        CK(cudaEventRecord(h->ev_c0, h->st));
        CK(cudaGraphLaunch(h->cg_exec, h->st));
        CK(cudaEventRecord(h->ev_c1, h->st));
        h->launches += (long long)chunk * launches_per_cg_iter(h);
        RC(sync_scal(h));
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
    // the search along d = w reads w at the neighbours
    return exchange(h, {VW});
}

int launch_objective(gpcg_problem* h, int x) {
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        with_gop(h, S, [&](auto& op) {
            using Op = std::decay_t<decltype(op)>;
            k_objective<Op><<<S.grid, kThreads, 0, h->st>>>(op, S.v[x], S.v[VB], h->dS, h->red(s));
        });
        h->launches++;
        CKLAUNCH();
    }
    return finish_reduce(h, fin(FIN_R2), 2);
}

// Is b the same in every grid row?  (global row 0 from slab 0 / rank 0, compared everywhere)
int detect_b_rows(gpcg_problem* h) {
    for (Slab& S : h->slabs) {
        CK(dalloc(h, &S.brow, (size_t)h->nx * sizeof(double)));
        CK(cudaMemcpyAsync(S.brow, h->slabs[0].v[VB], (size_t)h->nx * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    }
    if (h->use_nccl)
        NK(nccl_api()->Broadcast(h->slabs[0].brow, h->slabs[0].brow, (size_t)h->nx, ncclDouble, 0, h->comm, h->st));
    for (int s = 1; s < h->nslabs(); ++s)
        CK(cudaMemcpyAsync(h->slabs[s].brow, h->slabs[0].brow, (size_t)h->nx * sizeof(double),
                           cudaMemcpyDeviceToDevice, h->st));
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        const int g = std::max(1, std::min((int)(((long long)S.rows * h->nx + kThreads - 1) / kThreads), h->sms * 4));
        k_count_row_mismatch<<<g, kThreads, 0, h->st>>>(h->nx, S.rows, h->pitch, S.v[VB], S.brow, h->dS, h->red(s));
        CKLAUNCH();
    }
    RC(finish_reduce(h, fin(FIN_R2), 2));
    RC(sync_scal(h));
    h->bb = (h->hS->r0 == 0.0);
    return GPCG_OK;
}

// 1 / diag(A) of every slab (+ ghosts): the point-Jacobi preconditioner
int setup_jacobi(gpcg_problem* h) {
    for (Slab& S : h->slabs) {
        with_gop(h, S, [&](auto& op) {
            using Op = std::decay_t<decltype(op)>;
            k_jacobi_inverse<Op><<<S.grid, kThreads, 0, h->st>>>(op, S.v[VD]);
        });
        CKLAUNCH();
    }
    return exchange(h, {VD});
}

// ---------------------------------------------------------------- stencil slabs: operator
int setup_stencil_slabs(gpcg_problem* h, const double* wx, const double* wy, const double* shift) {
    const int nx = h->nx;
    double bad = 0.0;
    std::vector<const double*> arrs(h->nslabs());
    std::vector<long long> cnts(h->nslabs());
    const long long wx_int = h->wx_ld ? nx + 1 : 0, wy_int = h->wy_ld ? nx : 0;   // internal face layout
    for (Slab& S : h->slabs) {
        // wx: (glo + rows + ghi) rows of nx+1 (or one broadcast row); wy: face rows [-glo, rows + ghi]
        const long long wxr = h->wx_ld ? (S.glo + S.rows + S.ghi) : 1;
        const long long wyr = h->wy_ld ? (S.glo + S.rows + 1 + S.ghi) : 1;
        CK(dalloc(h, &S.wxb, (size_t)(wxr * (nx + 1)) * sizeof(double)));
        CK(dalloc(h, &S.wyb, (size_t)(wyr * nx) * sizeof(double)));
        CK(cudaMemsetAsync(S.wxb, 0, (size_t)(wxr * (nx + 1)) * sizeof(double), h->st));
        CK(cudaMemsetAsync(S.wyb, 0, (size_t)(wyr * nx) * sizeof(double), h->st));
        double* wxo = S.wxb + (h->wx_ld ? (long long)S.glo * (nx + 1) : 0);
        double* wyo = S.wyb + (h->wy_ld ? (long long)S.glo * nx : 0);
        const cudaMemcpyKind kx = (cudaMemcpyKind)copy_kind(wx, true), ky = (cudaMemcpyKind)copy_kind(wy, true);
        if (h->wx_ld)
            CK(cudaMemcpy2DAsync(wxo, (size_t)(nx + 1) * sizeof(double), wx + (long long)S.uoff * h->wx_ld,
                                 (size_t)h->wx_ld * sizeof(double), (size_t)(nx + 1) * sizeof(double), S.rows, kx, h->st));
        else
            CK(cudaMemcpyAsync(wxo, wx, (size_t)(nx + 1) * sizeof(double), kx, h->st));
        if (h->wy_ld)
            CK(cudaMemcpy2DAsync(wyo, (size_t)nx * sizeof(double), wy + (long long)S.uoff * h->wy_ld,
                                 (size_t)h->wy_ld * sizeof(double), (size_t)nx * sizeof(double), S.rows + 1, ky, h->st));
        else
            CK(cudaMemcpyAsync(wyo, wy, (size_t)nx * sizeof(double), ky, h->st));
        double* sho = nullptr;
        if (shift) {
            CK(dalloc(h, &S.shb, (size_t)S.nalloc * sizeof(double)));
            CK(cudaMemsetAsync(S.shb, 0, (size_t)S.nalloc * sizeof(double), h->st));
            sho = S.shb + (long long)S.glo * h->pitch;
            CK(cudaMemcpy2DAsync(sho, (size_t)h->pitch * sizeof(double), shift + (long long)S.uoff * nx,
                                 (size_t)nx * sizeof(double), (size_t)nx * sizeof(double), S.rows,
                                 (cudaMemcpyKind)copy_kind(shift, true), h->st));
        }
        S.sop = StencilOp{nx, S.rows, h->pitch, wxo, wyo, sho, wx_int, wy_int, -S.glo, S.rows + S.ghi};
        S.grid = std::max(1, std::min(((nx + 31) / 32) * ((S.rows + 7) / 8), h->sms * 16));
    }
    // validation of the owned weights (all slabs, all ranks)
    for (int pass = 0; pass < 3; ++pass) {
        for (int s = 0; s < h->nslabs(); ++s) {
            Slab& S = h->slabs[s];
            if (pass == 0) { arrs[s] = S.sop.wx; cnts[s] = h->wx_ld ? (long long)S.rows * (nx + 1) : nx + 1; }
            if (pass == 1) { arrs[s] = S.sop.wy; cnts[s] = h->wy_ld ? (long long)(S.rows + 1) * nx : nx; }
            if (pass == 2) { arrs[s] = S.shb ? S.shb : S.v[VB]; cnts[s] = S.shb ? S.nalloc : 0; }
        }
        if (pass == 2 && !shift) break;
        double t = 0.0;
        RC(count_nonfinite(h, arrs.data(), cnts.data(), &t));
        bad += t;
    }
    if (bad != 0.0) return set_err(GPCG_EINVAL, "%.0f non-finite stencil weights", bad);
    // ghost rows of the face arrays and the shift
    if (has_ghosts(h)) {
        RowArray arr[3];
        int na = 0;
        auto wxbase = [](gpcg_problem* hh, Slab& S, int) {
            return reinterpret_cast<char*>(const_cast<double*>(S.sop.wx));
        };
        auto wybase = [](gpcg_problem* hh, Slab& S, int) {
            return reinterpret_cast<char*>(const_cast<double*>(S.sop.wy));
        };
        auto shbase = [](gpcg_problem* hh, Slab& S, int) {
            return reinterpret_cast<char*>(const_cast<double*>(S.sop.shift));
        };
        if (h->wx_ld) arr[na++] = RowArray{wxbase, 0, (size_t)(nx + 1), sizeof(double), ncclDouble, 0, 0};
        if (h->wy_ld) arr[na++] = RowArray{wybase, 0, (size_t)nx, sizeof(double), ncclDouble, 1, 1};
        if (shift) arr[na++] = RowArray{shbase, 0, (size_t)h->pitch, sizeof(double), ncclDouble, 0, 0};
        if (na) RC(exchange_arrays(h, arr, na));
    }
    return GPCG_OK;
}

int create_stencil(gpcg_problem** out, const gpcg_dist* dist, void* stream, int64_t nx, int64_t ny,
                   const double* wx, int64_t wx_ld, const double* wy, int64_t wy_ld, const double* shift,
                   const double* b, const double* l, const double* u, double c) {
    g_err.clear();
    if (!out) return set_err(GPCG_EINVAL, "out is NULL");
    *out = nullptr;
    if (nx <= 0 || ny <= 0 || nx * ny >= (1LL << 31))
        return set_err(GPCG_EINVAL, "grid %lld x %lld out of range (need 0 < n < 2^31)", (long long)nx, (long long)ny);
    if (!wx || !wy || !b || !l || !u) return set_err(GPCG_EINVAL, "NULL array argument");
    if ((wx_ld != 0 && wx_ld < nx + 1) || (wy_ld != 0 && wy_ld < nx) || wx_ld < 0 || wy_ld < 0)
        return set_err(GPCG_EINVAL, "bad leading dimension (wx_ld %lld, wy_ld %lld)", (long long)wx_ld, (long long)wy_ld);
    if (!std::isfinite(c)) return set_err(GPCG_EINVAL, "c is not finite");
    long long rb = 0, re = ny;
    int nsl = 1;
    if (dist) {
        if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks)
            return set_err(GPCG_EINVAL, "bad rank %d / nranks %d", dist->rank, dist->nranks);
        rb = dist->row_begin;
        re = dist->row_end;
        nsl = dist->local_slabs > 0 ? dist->local_slabs : 1;
        if (rb < 0 || re > ny || re <= rb) return set_err(GPCG_EINVAL, "bad row range [%lld, %lld)", rb, re);
        if ((dist->rank == 0) != (rb == 0) || (dist->rank == dist->nranks - 1) != (re == ny))
            return set_err(GPCG_EINVAL, "row range [%lld, %lld) inconsistent with rank %d of %d", rb, re, dist->rank,
                           dist->nranks);
    }
    const long long pitch = (nx + 31) / 32 * 32;
    if (pitch * (re - rb + 4 * nsl) >= (1LL << 31)) return set_err(GPCG_EINVAL, "pitched grid too large");
    gpcg_problem* h = new gpcg_problem();
    auto fail = [&](int r) { free_all(h); return r; };
    h->is_csr = false;
    h->nx = (int)nx;
    h->rowlen = (int)nx;
    h->pitch = (int)pitch;
    h->wx_ld = wx_ld;
    h->wy_ld = wy_ld;
    h->n_global = nx * ny;
    h->n_local = nx * (re - rb);
    h->rank_row0 = rb;
    h->generic = getenv("GPCG_GENERIC") != nullptr && getenv("GPCG_GENERIC")[0] == '1';
    int rc;
    if ((rc = create_streams(h, stream))) return fail(rc);
    if ((rc = setup_comm(h, dist))) return fail(rc);
    // ghost rows: 3 -- the g-free GP accept sweep (k5, march_tma.cuh) applies the operator three
    // times on top of y (g, A yn, A d), the other sweeps twice
    if ((rc = layout_slabs(h, re - rb, nsl, 3))) return fail(rc);
    if ((rc = create_vectors(h, b, l, u))) return fail(rc);
    h->c = c;
    if ((rc = setup_stencil_slabs(h, wx, wy, shift))) return fail(rc);
    h->bc = (wx_ld == 0 && wy_ld == 0 && shift == nullptr);
    if ((rc = setup_jacobi(h))) return fail(rc);
    if ((rc = detect_b_rows(h))) return fail(rc);
    {
        const char* e = getenv("GPCG_TILE");
        if (e && *e) h->tile_mask = atoi(e) & 127;
        if (h->bc && !h->generic && h->tile_mask != 0 && (rc = setup_tile(h))) return fail(rc);
    }
    if (h->nranks > 1 && getenv("GPCG_XRANK") && atoi(getenv("GPCG_XRANK")) != 0 && h->tile && h->gfree &&
        (rc = setup_xrank_real(h)))
        return fail(rc);
    h->nnz = 5 * h->n_global - 2 * nx - 2 * ny;
    if ((rc = leave(h))) return fail(rc);
    *out = h;
    return GPCG_OK;
}

// ---------------------------------------------------------------- 3-D stencil slabs (z-planes)
int create_stencil3(gpcg_problem** out, const gpcg_dist* dist, void* stream, int64_t nx, int64_t ny, int64_t nz,
                    const double* wx, const double* wy, const double* wz, const double* shift, const double* b,
                    const double* l, const double* u, double c) {
    g_err.clear();
    if (!out) return set_err(GPCG_EINVAL, "out is NULL");
    *out = nullptr;
    if (nx <= 0 || ny <= 0 || nz <= 0 || nx * ny * nz >= (1LL << 31))
        return set_err(GPCG_EINVAL, "grid %lld x %lld x %lld out of range (need 0 < n < 2^31)", (long long)nx,
                       (long long)ny, (long long)nz);
    if (!wx || !wy || !wz || !b || !l || !u) return set_err(GPCG_EINVAL, "NULL array argument");
    if (!std::isfinite(c)) return set_err(GPCG_EINVAL, "c is not finite");
    long long rb = 0, re = nz;
    int nsl = 1;
    if (dist) {
        if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks)
            return set_err(GPCG_EINVAL, "bad rank %d / nranks %d", dist->rank, dist->nranks);
        rb = dist->row_begin;
        re = dist->row_end;
        nsl = dist->local_slabs > 0 ? dist->local_slabs : 1;
        if (rb < 0 || re > nz || re <= rb) return set_err(GPCG_EINVAL, "bad plane range [%lld, %lld)", rb, re);
        if ((dist->rank == 0) != (rb == 0) || (dist->rank == dist->nranks - 1) != (re == nz))
            return set_err(GPCG_EINVAL, "plane range [%lld, %lld) inconsistent with rank %d of %d", rb, re,
                           dist->rank, dist->nranks);
    }
    const long long plane = nx * ny;
    if (plane * (re - rb + 2 * nsl + 1) >= (1LL << 31)) return set_err(GPCG_EINVAL, "slab too large");
    gpcg_problem* h = new gpcg_problem();
    auto fail = [&](int r) { free_all(h); return r; };
    h->is3d = true;
    h->nx = (int)nx;
    h->rowlen = (int)plane;
    h->pitch = (int)plane;
    h->n_global = plane * nz;
    h->n_local = plane * (re - rb);
    h->rank_row0 = rb;
    int rc;
    if ((rc = create_streams(h, stream))) return fail(rc);
    if ((rc = setup_comm(h, dist))) return fail(rc);
    if ((rc = layout_slabs(h, re - rb, nsl, 1))) return fail(rc);
    if ((rc = create_vectors(h, b, l, u))) return fail(rc);
    h->c = c;
    const long long lx = (nx + 1) * ny, ly = nx * (ny + 1), lz = plane;   // elements per (face) plane
    std::vector<const double*> arrs(h->nslabs());
    std::vector<long long> cnts(h->nslabs());
    double bad = 0.0;
    for (Slab& S : h->slabs) {
        const long long planes = S.glo + S.rows + S.ghi;
        double *wxo, *wyo, *wzo, *sho = nullptr;
        // reuse the 2-D face slots: wxb <- wx, wyb <- wy, brow <- wz
        if (dalloc(h, &S.wxb, (size_t)(planes * lx) * sizeof(double)) != cudaSuccess ||
            dalloc(h, &S.wyb, (size_t)(planes * ly) * sizeof(double)) != cudaSuccess ||
            dalloc(h, &S.brow, (size_t)((planes + 1) * lz) * sizeof(double)) != cudaSuccess)
            return fail(set_err(GPCG_ENOMEM, "3-D face arrays"));
        cudaMemsetAsync(S.wxb, 0, (size_t)(planes * lx) * sizeof(double), h->st);
        cudaMemsetAsync(S.wyb, 0, (size_t)(planes * ly) * sizeof(double), h->st);
        cudaMemsetAsync(S.brow, 0, (size_t)((planes + 1) * lz) * sizeof(double), h->st);
        wxo = S.wxb + S.glo * lx;
        wyo = S.wyb + S.glo * ly;
        wzo = S.brow + S.glo * lz;
        if (cudaMemcpyAsync(wxo, wx + (long long)S.uoff * lx, (size_t)(S.rows * lx) * sizeof(double),
                            (cudaMemcpyKind)copy_kind(wx, true), h->st) != cudaSuccess ||
            cudaMemcpyAsync(wyo, wy + (long long)S.uoff * ly, (size_t)(S.rows * ly) * sizeof(double),
                            (cudaMemcpyKind)copy_kind(wy, true), h->st) != cudaSuccess ||
            cudaMemcpyAsync(wzo, wz + (long long)S.uoff * lz, (size_t)((S.rows + 1) * lz) * sizeof(double),
                            (cudaMemcpyKind)copy_kind(wz, true), h->st) != cudaSuccess)
            return fail(set_err(GPCG_ECUDA, "3-D face upload"));
        if (shift) {
            if (dalloc(h, &S.shb, (size_t)S.nalloc * sizeof(double)) != cudaSuccess)
                return fail(set_err(GPCG_ENOMEM, "shift"));
            cudaMemsetAsync(S.shb, 0, (size_t)S.nalloc * sizeof(double), h->st);
            sho = S.shb + S.glo * plane;
            if (cudaMemcpyAsync(sho, shift + (long long)S.uoff * plane, (size_t)(S.rows * plane) * sizeof(double),
                                (cudaMemcpyKind)copy_kind(shift, true), h->st) != cudaSuccess)
                return fail(set_err(GPCG_ECUDA, "shift upload"));
        }
        S.s3op = Stencil3Op{(int)nx, (int)ny, S.rows, plane, wxo, wyo, wzo, sho, -S.glo, S.rows + S.ghi};
        S.grid = std::max(1, (int)std::min<long long>((plane * S.rows + kThreads - 1) / kThreads, (long long)h->sms * 16));
        const long long items7 = ((nx + m3::OX - 1) / m3::OX) * ((ny + m3::OY - 1) / m3::OY) *
                                 (((long long)S.rows + m3::KZ - 1) / m3::KZ);
        S.grid7 = (int)std::max<long long>(1, std::min<long long>(items7, (long long)h->sms * 8));
    }
    for (int pass = 0; pass < 4; ++pass) {
        if (pass == 3 && !shift) break;
        for (int s = 0; s < h->nslabs(); ++s) {
            Slab& S = h->slabs[s];
            const double* a[4] = {S.s3op.wx, S.s3op.wy, S.s3op.wz, S.s3op.shift};
            const long long n[4] = {S.rows * lx, S.rows * ly, (S.rows + 1) * lz, S.rows * plane};
            arrs[s] = a[pass];
            cnts[s] = n[pass];
        }
        double t = 0.0;
        if ((rc = count_nonfinite(h, arrs.data(), cnts.data(), &t))) return fail(rc);
        bad += t;
    }
    if (bad != 0.0) return fail(set_err(GPCG_EINVAL, "%.0f non-finite stencil weights", bad));
    if (has_ghosts(h)) {
        auto bx = [](gpcg_problem*, Slab& S, int) { return reinterpret_cast<char*>(const_cast<double*>(S.s3op.wx)); };
        auto by = [](gpcg_problem*, Slab& S, int) { return reinterpret_cast<char*>(const_cast<double*>(S.s3op.wy)); };
        auto bz = [](gpcg_problem*, Slab& S, int) { return reinterpret_cast<char*>(const_cast<double*>(S.s3op.wz)); };
        auto bs = [](gpcg_problem*, Slab& S, int) { return reinterpret_cast<char*>(const_cast<double*>(S.s3op.shift)); };
        RowArray arr[4] = {RowArray{bx, 0, (size_t)lx, sizeof(double), ncclDouble, 0, 0},
                           RowArray{by, 0, (size_t)ly, sizeof(double), ncclDouble, 0, 0},
                           RowArray{bz, 0, (size_t)lz, sizeof(double), ncclDouble, 1, 1},
                           RowArray{bs, 0, (size_t)plane, sizeof(double), ncclDouble, 0, 0}};
        if ((rc = exchange_arrays(h, arr, shift ? 4 : 3))) return fail(rc);
    }
    if ((rc = setup_jacobi(h))) return fail(rc);
    h->nnz = 7 * h->n_global - 2 * (ny * nz + nx * nz + nx * ny);
    if ((rc = leave(h))) return fail(rc);
    *out = h;
    return GPCG_OK;
}

// ---------------------------------------------------------------- CSR slabs
// one slab, one rank: row_ptr / col / val uploaded unchanged (from the caller's pinned or device
// memory), checked by k_check_csr and k_count_nonfinite
int create_csr_one(gpcg_problem** out, void* stream, int64_t n, const int64_t* row_ptr, const int32_t* col,
                   const double* val, const double* b, const double* l, const double* u, double c) {
    long long ends[2] = {0, 0};
    if (is_device_ptr(row_ptr)) {
        if (cudaMemcpy(&ends[0], row_ptr, sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(&ends[1], row_ptr + n, sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            return set_err(GPCG_ECUDA, "reading row_ptr");
        }
    } else {
        ends[0] = row_ptr[0];
        ends[1] = row_ptr[n];
    }
    if (ends[0] != 0 || ends[1] < n || ends[1] >= (1LL << 40))
        return set_err(GPCG_EINVAL, "row_ptr[0] = %lld, row_ptr[n] = %lld invalid", ends[0], ends[1]);
    const long long nnz = ends[1];
    gpcg_problem* h = new gpcg_problem();
    auto fail = [&](int r) { free_all(h); return r; };
    h->is_csr = true;
    h->pitch = 1;
    h->rowlen = 1;
    h->n_global = n;
    h->n_local = n;
    h->rank_row0 = 0;
    h->nnz = nnz;
    int rc;
    if ((rc = create_streams(h, stream))) return fail(rc);
    if ((rc = setup_comm(h, nullptr))) return fail(rc);
    if ((rc = layout_slabs(h, n, 1, 0))) return fail(rc);
    if ((rc = create_vectors(h, b, l, u))) return fail(rc);
    h->c = c;
    Slab& S = h->slabs[0];
    if (dalloc(h, &S.rp, (n + 1) * sizeof(long long)) != cudaSuccess ||
        dalloc(h, &S.ci, std::max<long long>(1, nnz) * sizeof(int)) != cudaSuccess ||
        dalloc(h, &S.val, std::max<long long>(1, nnz) * sizeof(double)) != cudaSuccess)
        return fail(set_err(GPCG_ENOMEM, "CSR arrays (nnz = %lld)", nnz));
    if (cudaMemcpyAsync(S.rp, row_ptr, (n + 1) * sizeof(long long), (cudaMemcpyKind)copy_kind(row_ptr, true), h->st) != cudaSuccess ||
        cudaMemcpyAsync(S.ci, col, nnz * sizeof(int), (cudaMemcpyKind)copy_kind(col, true), h->st) != cudaSuccess ||
        cudaMemcpyAsync(S.val, val, nnz * sizeof(double), (cudaMemcpyKind)copy_kind(val, true), h->st) != cudaSuccess)
        return fail(set_err(GPCG_ECUDA, "CSR upload"));
    {
        const int g = (int)std::max<long long>(1, std::min<long long>((nnz + kThreads - 1) / kThreads, (long long)h->sms * 8));
        k_check_csr<<<g, kThreads, 0, h->st>>>(n, S.rp, S.ci, nnz, h->dS, h->red(0));
        if (cudaGetLastError() != cudaSuccess) return fail(set_err(GPCG_ECUDA, "k_check_csr launch"));
        if ((rc = finish_reduce(h, fin(FIN_R2), 2)) || (rc = sync_scal(h))) return fail(rc);
        if (h->hS->r0 != 0.0) return fail(set_err(GPCG_EINVAL, "row_ptr not monotone at %.0f rows", h->hS->r0));
        if (h->hS->r1 != 0.0) return fail(set_err(GPCG_EINVAL, "%.0f column indices out of range [0, %lld)", h->hS->r1, (long long)n));
    }
    S.cop = CsrOp{S.rows, S.rp, S.ci, S.val};
    S.grid = std::max(1, std::min((S.rows + kThreads - 1) / kThreads, h->sms * 16));
    if ((rc = setup_jacobi(h))) return fail(rc);
    {
        const double* arrs[1] = {S.val};
        long long cnts[1] = {nnz};
        double t = 0.0;
        if ((rc = count_nonfinite(h, arrs, cnts, &t))) return fail(rc);
        if (t != 0.0) return fail(set_err(GPCG_EINVAL, "%.0f non-finite CSR values", t));
    }
    if ((rc = leave(h))) return fail(rc);
    *out = h;
    return GPCG_OK;
}

int create_csr(gpcg_problem** out, const gpcg_dist* dist, void* stream, int64_t n_global, const int64_t* row_ptr,
               const int32_t* col, const double* val, const double* b, const double* l, const double* u, double c) {
    g_err.clear();
    if (!out) return set_err(GPCG_EINVAL, "out is NULL");
    *out = nullptr;
    if (n_global <= 0 || n_global >= (1LL << 31)) return set_err(GPCG_EINVAL, "n = %lld out of range", (long long)n_global);
    if (!row_ptr || !col || !val || !b || !l || !u) return set_err(GPCG_EINVAL, "NULL array argument");
    if (!std::isfinite(c)) return set_err(GPCG_EINVAL, "c is not finite");
    long long rb = 0, re = n_global;
    int nsl = 1;
    if (dist) {
        if (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks)
            return set_err(GPCG_EINVAL, "bad rank %d / nranks %d", dist->rank, dist->nranks);
        rb = dist->row_begin;
        re = dist->row_end;
        nsl = dist->local_slabs > 0 ? dist->local_slabs : 1;
        if (rb < 0 || re > n_global || re <= rb) return set_err(GPCG_EINVAL, "bad row range [%lld, %lld)", rb, re);
        if ((dist->rank == 0) != (rb == 0) || (dist->rank == dist->nranks - 1) != (re == n_global))
            return set_err(GPCG_EINVAL, "row range [%lld, %lld) inconsistent with rank %d of %d", rb, re, dist->rank,
                           dist->nranks);
    }
    const long long nloc = re - rb;
    // one slab of one rank: the arrays are uploaded as given and validated on the device (no ghost
    // bands; the host would otherwise walk all nnz entries twice -- 0.7 s at C4's 117M)
    if (nsl == 1 && (!dist || dist->nranks == 1)) return create_csr_one(out, stream, n_global, row_ptr, col, val, b, l, u, c);
    // the row structure on the host (create time only): ghost bands of every slab
    std::vector<long long> rp(nloc + 1);
    const bool rp_dev = is_device_ptr(row_ptr);
    if (rp_dev) {
        if (cudaMemcpy(rp.data(), row_ptr, (nloc + 1) * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            return set_err(GPCG_ECUDA, "reading row_ptr");
        }
    } else {
        memcpy(rp.data(), row_ptr, (nloc + 1) * sizeof(long long));
    }
    if (rp[0] != 0 || rp[nloc] < nloc || rp[nloc] >= (1LL << 40))
        return set_err(GPCG_EINVAL, "row_ptr[0] = %lld, row_ptr[n] = %lld invalid", rp[0], rp[nloc]);
    for (long long i = 0; i < nloc; ++i)
        if (rp[i + 1] < rp[i]) return set_err(GPCG_EINVAL, "row_ptr not monotone at row %lld", i);
    const long long nnz = rp[nloc];
    std::vector<int32_t> colh;
    const int32_t* cols = col;
    if (is_device_ptr(col)) {
        colh.resize(nnz);
        if (cudaMemcpy(colh.data(), col, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess) {
            cudaGetLastError();
            return set_err(GPCG_ECUDA, "reading col");
        }
        cols = colh.data();
    }
    gpcg_problem* h = new gpcg_problem();
    auto fail = [&](int r) { free_all(h); return r; };
    h->is_csr = true;
    h->pitch = 1;
    h->rowlen = 1;
    h->n_global = n_global;
    h->n_local = nloc;
    h->rank_row0 = rb;
    h->nnz = nnz;
    int rc;
    if ((rc = create_streams(h, stream))) return fail(rc);
    if ((rc = setup_comm(h, dist))) return fail(rc);
    if ((rc = layout_slabs(h, nloc, nsl, 0))) return fail(rc);
    // ghost bands: columns below / above the slab's rows (global ids)
    for (Slab& S : h->slabs) {
        const long long g0 = rb + S.row0, g1 = g0 + S.rows;
        long long cmin = g0, cmax = g1 - 1;
        for (long long k = rp[S.row0]; k < rp[S.row0 + S.rows]; ++k) {
            if (cols[k] < 0 || cols[k] >= n_global) return fail(set_err(GPCG_EINVAL, "col[%lld] = %d out of range", k, cols[k]));
            cmin = std::min<long long>(cmin, cols[k]);
            cmax = std::max<long long>(cmax, cols[k]);
        }
        S.glo = (int)(g0 - cmin);
        S.ghi = (int)(cmax - (g1 - 1));
        if ((S.glo > 0 && S.nb_lo == NB_NONE) || (S.ghi > 0 && S.nb_hi == NB_NONE))
            return fail(set_err(GPCG_EINVAL, "internal: ghost band without a neighbour"));
    }
    // what each neighbour reads from a slab (local neighbours directly; remote via NCCL)
    for (int s = 0; s < h->nslabs(); ++s) {
        Slab& S = h->slabs[s];
        S.send_lo = S.nb_lo >= 0 ? h->slabs[S.nb_lo].ghi : 0;
        S.send_hi = S.nb_hi >= 0 ? h->slabs[S.nb_hi].glo : 0;
        if (S.nb_lo >= 0 && S.glo > h->slabs[S.nb_lo].rows)
            return fail(set_err(GPCG_EINVAL, "slab %d: lower band (%d rows) exceeds the neighbour slab", s, S.glo));
        if (S.nb_hi >= 0 && S.ghi > h->slabs[S.nb_hi].rows)
            return fail(set_err(GPCG_EINVAL, "slab %d: upper band (%d rows) exceeds the neighbour slab", s, S.ghi));
    }
    if (h->nranks > 1) {
        // exchange band widths with the neighbouring ranks: my glo is what rank-1 sends me
        long long* dbuf = nullptr;
        if (dalloc(h, &dbuf, 4 * sizeof(long long)) != cudaSuccess) return fail(set_err(GPCG_ENOMEM, "band buffer"));
        long long hb[4] = {h->slabs.front().glo, h->slabs.back().ghi, 0, 0};
        cudaMemcpy(dbuf, hb, 4 * sizeof(long long), cudaMemcpyHostToDevice);
        const NcclApi* N = nccl_api();
        auto nk = [&](ncclResult_t r) { return r == ncclSuccess; };
        bool ok = nk(N->GroupStart());
        if (h->rank > 0) ok = ok && nk(N->Send(dbuf, 1, ncclInt64, h->rank - 1, h->comm, h->st)) &&
                          nk(N->Recv(dbuf + 2, 1, ncclInt64, h->rank - 1, h->comm, h->st));
        if (h->rank < h->nranks - 1) ok = ok && nk(N->Send(dbuf + 1, 1, ncclInt64, h->rank + 1, h->comm, h->st)) &&
                                       nk(N->Recv(dbuf + 3, 1, ncclInt64, h->rank + 1, h->comm, h->st));
        ok = nk(N->GroupEnd()) && ok;
        cudaStreamSynchronize(h->st);
        cudaMemcpy(hb, dbuf, 4 * sizeof(long long), cudaMemcpyDeviceToHost);
        dfree(h, dbuf);
        if (!ok) return fail(set_err(GPCG_ENCCL, "band-width exchange failed"));
        h->slabs.front().send_lo = h->rank > 0 ? (int)hb[2] : 0;            // rank-1's ghi
        h->slabs.back().send_hi = h->rank < h->nranks - 1 ? (int)hb[3] : 0; // rank+1's glo
        if (h->slabs.front().send_lo > h->slabs.front().rows || h->slabs.back().send_hi > h->slabs.back().rows)
            return fail(set_err(GPCG_EINVAL, "a neighbouring rank's band exceeds this rank's rows"));
    }
    if ((rc = create_vectors(h, b, l, u))) return fail(rc);
    h->c = c;
    // per-slab CSR: rows rebased, columns as local offsets from the slab's first row
    std::vector<long long> rps;
    std::vector<int32_t> cis;
    const cudaMemcpyKind kv = (cudaMemcpyKind)copy_kind(val, true);
    for (Slab& S : h->slabs) {
        const long long k0 = rp[S.row0], k1 = rp[S.row0 + S.rows], g0 = rb + S.row0;
        rps.resize(S.rows + 1);
        for (int i = 0; i <= S.rows; ++i) rps[i] = rp[S.row0 + i] - k0;
        cis.resize(k1 - k0);
        for (long long k = k0; k < k1; ++k) cis[k - k0] = (int32_t)(cols[k] - g0);
        if (dalloc(h, &S.rp, (S.rows + 1) * sizeof(long long)) != cudaSuccess ||
            dalloc(h, &S.ci, std::max<long long>(1, k1 - k0) * sizeof(int)) != cudaSuccess ||
            dalloc(h, &S.val, std::max<long long>(1, k1 - k0) * sizeof(double)) != cudaSuccess)
            return fail(set_err(GPCG_ENOMEM, "CSR arrays (nnz = %lld)", k1 - k0));
        if (cudaMemcpy(S.rp, rps.data(), (S.rows + 1) * sizeof(long long), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(S.ci, cis.data(), (k1 - k0) * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpyAsync(S.val, val + k0, (k1 - k0) * sizeof(double), kv, h->st) != cudaSuccess)
            return fail(set_err(GPCG_ECUDA, "CSR upload"));
        S.cop = CsrOp{S.rows, S.rp, S.ci, S.val};
        S.grid = std::max(1, std::min((S.rows + kThreads - 1) / kThreads, h->sms * 16));
    }
    if ((rc = setup_jacobi(h))) return fail(rc);
    {
        std::vector<const double*> arrs;
        std::vector<long long> cnts;
        for (Slab& S : h->slabs) {
            arrs.push_back(S.val);
            cnts.push_back(rp[S.row0 + S.rows] - rp[S.row0]);
        }
        double t = 0.0;
        if ((rc = count_nonfinite(h, arrs.data(), cnts.data(), &t))) return fail(rc);
        if (t != 0.0) return fail(set_err(GPCG_EINVAL, "%.0f non-finite CSR values", t));
    }
    if ((rc = leave(h))) return fail(rc);
    *out = h;
    return GPCG_OK;
}

}  // namespace

// ============================================================================
// ABI
// ============================================================================
// A_F v over the compacted free-row list of the recorded free set (compact_ok handles, S.fmask ==
// h->free_mask): y_free[k] (|F| entries) and / or y_full at the free rows
int launch_hessvec_free(gpcg_problem* h, Slab& S, const double* v, double* y_free, double* y_full) {
    if (S.fcount <= 0) return GPCG_OK;
    if (h->is_csr) {
        // 4 rows per warp and kRowUnroll per group: one warp per 16 rows, up to 8 CTAs per SM resident
        const long long rows_per_cta = (long long)(kThreads / 32) * (32 / kRowLanes) * kRowUnroll;
        const int g = (int)std::max<long long>(
            1, std::min<long long>((S.fcount + rows_per_cta - 1) / rows_per_cta, (long long)h->sms * 8));
        k_hessvec_free_csr<<<g, kThreads, 0, h->st>>>(S.cop, S.fcount, S.flist, S.fbits, v, y_free, y_full);
    } else {
        const int g = (int)((S.fcount + kThreads - 1) / kThreads);
        with_gop(h, S, [&](auto& op) {
            using Op = std::decay_t<decltype(op)>;
            k_hessvec_free<Op><<<g, kThreads, 0, h->st>>>(op, S.fcount, S.flist, S.fbits, v, y_free, y_full);
        });
    }
    h->launches++;
    CKLAUNCH();
    return GPCG_OK;
}

extern "C" {

gpcg_params gpcg_params_default(void) {
    gpcg_params p;
    p.mu = 0.1;
    p.eta1 = 0.1;
    p.eta2 = 0.05;
    p.eta2_shrink = 0.1;
    p.eta2_floor = 1e-12;
    p.gp_cap = 100000;  // safety net only: the paper's GP phase has no cap (R13)
    p.refine_cap = 30;
    p.max_halvings = 50;
    p.cg_cap = 0;
    p.search_k = 2;
    p.cg_chunk = 32;
    p.gp_chunk = 8;
    p.precond = 0;
    p.cg_mode = 2;      // in place; CSR / 3-D with |F| < 0.3 n over the compacted free-row list
    return p;
}

const char* gpcg_last_error(void) { return g_err.c_str(); }

int64_t gpcg_size(const gpcg_problem* h) { return h ? h->n_local : -1; }

void gpcg_partition_rows(int64_t total, int32_t parts, int32_t part, int64_t* begin, int64_t* end) {
    long long b = 0, e = 0;
    if (total >= 0 && parts > 0 && part >= 0 && part < parts) partition(total, parts, part, &b, &e);
    if (begin) *begin = b;
    if (end) *end = e;
}

int gpcg_nccl_unique_id(void* out128) {
    g_err.clear();
    if (!out128) return set_err(GPCG_EINVAL, "NULL argument");
    const NcclApi* N = nccl_api();
    if (!N) return set_err(GPCG_ENCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    NK(N->GetUniqueId(&id));
    memcpy(out128, &id, sizeof id);
    return GPCG_OK;
}

int gpcg_create_stencil2d(gpcg_problem** out, void* cuda_stream, int64_t nx, int64_t ny, const double* wx,
                          int64_t wx_ld, const double* wy, int64_t wy_ld, const double* shift, const double* b,
                          const double* l, const double* u, double c) {
    return create_stencil(out, nullptr, cuda_stream, nx, ny, wx, wx_ld, wy, wy_ld, shift, b, l, u, c);
}

int gpcg_create_stencil2d_dist(gpcg_problem** out, const gpcg_dist* dist, void* cuda_stream, int64_t nx, int64_t ny,
                               const double* wx, int64_t wx_ld, const double* wy, int64_t wy_ld, const double* shift,
                               const double* b, const double* l, const double* u, double c) {
    return create_stencil(out, dist, cuda_stream, nx, ny, wx, wx_ld, wy, wy_ld, shift, b, l, u, c);
}

int gpcg_create_stencil3d(gpcg_problem** out, void* cuda_stream, int64_t nx, int64_t ny, int64_t nz, const double* wx,
                          const double* wy, const double* wz, const double* shift, const double* b, const double* l,
                          const double* u, double c) {
    return create_stencil3(out, nullptr, cuda_stream, nx, ny, nz, wx, wy, wz, shift, b, l, u, c);
}

int gpcg_create_stencil3d_dist(gpcg_problem** out, const gpcg_dist* dist, void* cuda_stream, int64_t nx, int64_t ny,
                               int64_t nz, const double* wx, const double* wy, const double* wz, const double* shift,
                               const double* b, const double* l, const double* u, double c) {
    return create_stencil3(out, dist, cuda_stream, nx, ny, nz, wx, wy, wz, shift, b, l, u, c);
}

int gpcg_create_csr(gpcg_problem** out, void* cuda_stream, int64_t n, const int64_t* row_ptr, const int32_t* col,
                    const double* val, const double* b, const double* l, const double* u, double c) {
    return create_csr(out, nullptr, cuda_stream, n, row_ptr, col, val, b, l, u, c);
}

int gpcg_create_csr_dist(gpcg_problem** out, const gpcg_dist* dist, void* cuda_stream, int64_t n,
                         const int64_t* row_ptr, const int32_t* col, const double* val, const double* b,
                         const double* l, const double* u, double c) {
    return create_csr(out, dist, cuda_stream, n, row_ptr, col, val, b, l, u, c);
}

int gpcg_set_params(gpcg_problem* h, const gpcg_params* p) {
    g_err.clear();
    if (!h || !p) return set_err(GPCG_EINVAL, "NULL argument");
    if (!(p->mu > 0.0 && p->mu < 0.5)) return set_err(GPCG_EINVAL, "mu must lie in (0, 1/2)");
    if (!(p->eta1 > 0.0 && p->eta1 < 1.0) || !(p->eta2 > 0.0 && p->eta2 < 1.0))
        return set_err(GPCG_EINVAL, "eta1, eta2 must lie in (0, 1)");
    if (!(p->eta2_shrink > 0.0 && p->eta2_shrink < 1.0) || !(p->eta2_floor > 0.0))
        return set_err(GPCG_EINVAL, "eta2_shrink in (0,1), eta2_floor > 0 required");
    if (p->gp_cap < 1 || p->refine_cap < 1 || p->max_halvings < 1 || p->max_halvings > 1000 || p->cg_cap < 0 ||
        p->search_k < 1 || p->search_k > kMaxK || p->cg_chunk < 1 || p->cg_chunk > 4096 || p->gp_chunk < 1 ||
        p->gp_chunk > 256 || p->precond < 0 || p->precond > 3 || (p->cg_mode < 0 || p->cg_mode > 3))
        return set_err(GPCG_EINVAL, "integer parameter out of range");
    const int old_chunk = h->prm.cg_chunk, old_pc = h->prm.precond;
    h->prm = *p;
    if ((old_chunk != p->cg_chunk || old_pc != p->precond) && h->cg_exec) {
        cudaGraphExecDestroy(h->cg_exec);
        h->cg_exec = nullptr;
    }
    // the GP graphs bake in search_k / mu (and the chunk): rebuilt at the next solve
    for (cudaGraphExec_t& g : h->gp_exec)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    for (cudaGraphExec_t& g : h->gp_exec_s)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    return GPCG_OK;
}

void gpcg_destroy(gpcg_problem* h) { free_all(h); }

int gpcg_project(gpcg_problem* h, const double* x, double* px, double* pg_norm2, int64_t* n_active,
                 int64_t* n_active_nonbinding) {
    g_err.clear();
    if (!h || !x || !px) return set_err(GPCG_EINVAL, "NULL argument");
    RC(enter(h));
    RC(upload_vec(h, VIN, x));
    RC(exchange(h, {VIN}));
    RC(launch_accept(h, VIN, NO_VEC, 0.0, NO_VEC, VY0, VG0, MK0));
    RC(download_vec(h, px, VY0));
    RC(sync_scal(h));
    h->free_mask = 0;
    if (compact_ok(h)) RC(build_free_list(h, h->slabs[0], 0));
    if (pg_norm2) *pg_norm2 = h->hS->pg2;
    if (n_active) *n_active = (int64_t)h->hS->n_active;
    if (n_active_nonbinding) *n_active_nonbinding = (int64_t)h->hS->n_nonbinding;
    return leave(h);
}

int64_t gpcg_free_count(gpcg_problem* h) {
    if (!h || h->free_mask < 0 || !compact_ok(h)) return -1;
    const Slab& S = h->slabs[0];
    return S.fmask == h->free_mask ? (int64_t)S.fcount : -1;
}

int gpcg_hessvec_free(gpcg_problem* h, const double* v, double* y_free) {
    g_err.clear();
    if (!h || !v || !y_free) return set_err(GPCG_EINVAL, "NULL argument");
    if (h->free_mask < 0)
        return set_err(GPCG_ESTATE, "reduced hessvec needs a free set: call gpcg_project or gpcg_solve first");
    if (!compact_ok(h))
        return set_err(GPCG_EINVAL, "gpcg_hessvec_free supports CSR / 3-D operators on one slab and rank");
    RC(enter(h));
    Slab& S = h->slabs[0];
    if (S.fmask != h->free_mask || S.fcount < 0) RC(build_free_list(h, S, h->free_mask));
    const long long m = S.fcount;
    const bool vdev = is_device_ptr(v), ydev = is_device_ptr(y_free);
    const double* vin = v;
    if (!vdev) {
        RC(upload_vec(h, VIN, v));
        vin = S.v[VIN];
    }
    double* yout = ydev ? y_free : S.v[VOUT];
    RC(launch_hessvec_free(h, S, vin, yout, nullptr));
    if (!ydev && m > 0) {
        CK(cudaMemcpyAsync(y_free, yout, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
    }
    return leave(h);
}

int gpcg_hessvec(gpcg_problem* h, const double* v, double* y, int reduced) {
    g_err.clear();
    if (!h || !v || !y) return set_err(GPCG_EINVAL, "NULL argument");
    if (v == y) return set_err(GPCG_EINVAL, "v and y must not alias");
    if (reduced && h->free_mask < 0)
        return set_err(GPCG_ESTATE, "reduced hessvec needs a free set: call gpcg_project or gpcg_solve first");
    RC(enter(h));
    // direct device access only for one slab with a contiguous layout (CSR, or nx a multiple of 32)
    const bool direct = h->nslabs() == 1 && !has_ghosts(h) && (h->is_csr || h->pitch == h->rowlen);
    const bool vdev = direct && is_device_ptr(v), ydev = direct && is_device_ptr(y);
    if (!vdev) {
        RC(upload_vec(h, VIN, v));
        RC(exchange(h, {VIN}));
    }
    for (Slab& S : h->slabs) {
        const double* vin = vdev ? v : S.v[VIN];
        double* yout = ydev ? y : S.v[VOUT];
        const unsigned char* mask = reduced ? S.m[h->free_mask] : nullptr;
        auto go = [&](auto& op) {
            using Op = std::decay_t<decltype(op)>;
            if (reduced) k_hessvec<Op, true><<<S.grid, kThreads, 0, h->st>>>(op, vin, yout, mask);
            else k_hessvec<Op, false><<<S.grid, kThreads, 0, h->st>>>(op, vin, yout, mask);
        };
        // broadcast-face 2-D stencils: the TMA-fed march (needs a 16-byte aligned input for its map)
        const bool k4 = h->tile && !h->generic && (reinterpret_cast<uintptr_t>(vin) & 15) == 0;
        // CSR / 3-D with a small free set: only the free rows (compacted list of the recorded set)
        const long long nown = S.rows * (long long)h->rowlen;
        const bool rows = reduced && compact_ok(h) && S.fmask == h->free_mask && S.fcount >= 0 &&
                          10 * S.fcount < 3 * nown && h->prm.cg_mode != 0;
        if (rows) {
            CK(cudaMemsetAsync(yout, 0, (size_t)nown * sizeof(double), h->st));
            RC(launch_hessvec_free(h, S, vin, nullptr, yout));
        } else if (k4) {
            CUtensorMap mv;
            if (vin == S.v[VIN]) mv = S.t4[VIN];
            else RC(make_map(h, S, &mv, vin, false, m4::kBW, m4::kBR));
            if (reduced)
                k4_hessvec<true><<<S.grid4_cg, m4::kThreadsWS, m4hv::kSmem, h->st>>>(S.sop, S.bg_cg, mv,
                                                                                     S.t4m[h->free_mask], yout);
            else
                k4_hessvec<false><<<S.grid4_cg, m4::kThreadsWS, m4hv::kSmem, h->st>>>(S.sop, S.bg_cg, mv, S.t4m[0],
                                                                                      yout);
        } else if (use_m3(h)) {
            if (reduced) k7_hessvec<true><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, vin, yout, mask);
            else k7_hessvec<false><<<S.grid7, m3::kThreads, 0, h->st>>>(S.s3op, vin, yout, mask);
        } else {
            with_gop(h, S, go);
        }
        h->launches++;
        CKLAUNCH();
    }
    if (!ydev) {
        RC(download_vec(h, y, VOUT));
        if (!is_device_ptr(y)) CK(cudaStreamSynchronize(h->st));
    }
    return leave(h);
}

int gpcg_objective(gpcg_problem* h, const double* x, double* q) {
    g_err.clear();
    if (!h || !x || !q) return set_err(GPCG_EINVAL, "NULL argument");
    RC(enter(h));
    RC(upload_vec(h, VIN, x));
    RC(exchange(h, {VIN}));
    RC(launch_objective(h, VIN));
    RC(sync_scal(h));
    *q = 0.5 * h->hS->r0 - h->hS->r1 + h->c;
    return leave(h);
}

// Algorithm GPCG, same steps as the oracle.
int gpcg_solve(gpcg_problem* h, const double* x0, double tol, int64_t max_it, double* x_out, gpcg_stats* stats) {
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
    h->t_extract_ms = 0.0;
    int rc;
    RC(enter(h));
    const gpcg_params& prm = h->prm;
    float t_cg = 0.f, t_gp = 0.f, ms = 0.f;
    int status = GPCG_NOT_CONVERGED;
    int cur = 0;
    double tau = 0.0;
    const Scal& S = *h->hS;

    // Setup: x <- P[x0], g <- A x - b
    RC(upload_vec(h, VIN, x0));
    RC(exchange(h, {VIN}));
    RC(launch_accept(h, VIN, NO_VEC, 0.0, NO_VEC, VY0, VG0, MK0));
    RC(sync_scal(h));
    st.full_spmvs++;
    if (h->gp_graph && !gp_persist(h))
        RC(build_gp_graph(h, std::max(1, h->prm.gp_chunk)));
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
            bool conv = false;
            if (h->gp_graph) {
                // device-driven: graph chunks of GP steps, one poll per chunk (k_gp_step decides)
                k_gp_begin<<<1, 32, 0, h->st>>>(h->dS, tau, prm.eta1, prm.gp_cap);
                h->launches++;
                CKLAUNCH();
                long long jdone = 0;
                const bool persist = gp_persist(h);
                bool first = true;
                for (;;) {
                    if (persist) {
                        if ((rc = launch_gp_loop(h, cur))) goto fail;
                    } else {
                        const bool small = first && h->gp_exec_s[0];
                        CK(cudaGraphLaunch(small ? h->gp_exec_s[cur] : h->gp_exec[cur], h->st));
                        h->launches += (long long)(small ? h->gp_exec_s_chunk : h->gp_exec_chunk) *
                                       launches_per_gp_step(h);
                    }
                    first = false;
                    if ((rc = sync_scal(h))) goto fail;
                    if (persist && (rc = check_xrank(h))) goto fail;
                    const long long jn = S.gp_j;
                    if (persist) st.gp_spec_rejected += S.gp_fb;
                    cur = (int)((cur + (jn - jdone)) & 1);
                    st.gp_iters += jn - jdone;
                    st.full_spmvs += 3 * (jn - jdone);
                    jdone = jn;
                    if (!S.gp_done) continue;
                    if (S.gp_reason != GP_HOST) break;
                    // the first search batch found no step: the host finishes this step (the persistent
                    // kernel reports the first step size index it has not tried in s_pad)
                    int hacc = -1;
                    const int hstart = persist ? std::max(S.s_pad, 0)
                                               : first_k(h) + ((graph_spec(h) || graph_spec5(h)) ? 1 : 0);
                    if ((rc = search_and_accept(h, cur, vg(cur), -1.0, 1, &hacc, hstart))) goto fail;
                    cur ^= 1;
                    const long long j = jdone + 1;
                    jdone = j;
                    st.gp_iters++;
                    st.full_spmvs += 3;
                    const double dec = -S.s_delta;
                    const bool stop = (S.n_changed == 0.0) || (j >= 2 && dec <= prm.eta1 * S.gp_maxdec) ||
                                      (j >= prm.gp_cap);
                    const double maxdec = std::max(S.gp_maxdec, dec);
                    const bool cv = !stop && std::sqrt(S.pg2) <= tau;
                    k_gp_set<<<1, 32, 0, h->st>>>(h->dS, j, maxdec, (stop || cv) ? 1 : 0,
                                                  stop ? GP_STOP : (cv ? GP_CONV : GP_RUNNING));
                    h->launches++;
                    CKLAUNCH();
                    if (stop || cv) { if ((rc = sync_scal(h))) goto fail; break; }
                }
                if (trace_on())
                    fprintf(stderr, "[gpcg] k=%lld GP phase: %lld steps (%d speculative sweeps rejected) reason=%d |A|=%.0f pg=%.3e t=%.2fms\n",
                            (long long)k, jdone, S.gp_fb, S.gp_reason, S.n_active, std::sqrt(S.pg2),
                            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
            } else {
                long long j = 0;
                double maxdec = 0.0;
                for (;;) {
                    if (std::sqrt(S.pg2) <= tau) { conv = true; break; }
                    if ((rc = launch_cauchy(h, vy(cur), vg(cur)))) goto fail;
                    st.full_spmvs++;
                    int hacc = -1;
                    // direction -grad q (Eq. next-y); trial points equal those of the
                    // -grad_Omega q reading for feasible y (reading R8)
                    if ((rc = search_and_accept(h, cur, vg(cur), -1.0, 1, &hacc))) goto fail;
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
            }
            CK(cudaEventRecord(h->ev_b, h->st));
            CK(cudaEventSynchronize(h->ev_b));
            CK(cudaEventElapsedTime(&ms, h->ev_a, h->ev_b));
            t_gp += ms;
            if (conv || std::sqrt(S.pg2) <= tau) { status = GPCG_OK; break; }

            // ---- CG phase with eta2 refinement -------------------
            double eta2 = prm.eta2;
            for (int64_t rep = 0; rep < prm.refine_cap; ++rep) {
                const long long m = h->n_global - (long long)S.n_active;
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
                if (graph_spec(h)) {            // the CG phase's step at alpha = 1 first (k_spec)
                    if ((rc = launch_spec(h, cur, VW, 1.0, 0, 0)) || (rc = sync_scal(h))) goto fail;
                    if (S.spec_ok) hacc = 0;
                    else if ((rc = search_and_accept(h, cur, VW, 1.0, 0, &hacc, 1))) goto fail;
                } else if ((rc = search_and_accept(h, cur, VW, 1.0, 0, &hacc))) {
                    goto fail;
                }
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
    RC(download_vec(h, x_out, vy(cur)));
    {
        // the sets and ||grad_Omega q|| of x_out are those of the last accept sweep (already in S)
        const double pg2 = S.pg2, na = S.n_active, nnb = S.n_nonbinding;
        RC(launch_objective(h, vy(cur)));
        RC(sync_scal(h));
        h->free_mask = cur;
        if (compact_ok(h)) RC(build_free_list(h, h->slabs[0], cur));
        st.q = 0.5 * S.r0 - S.r1 + h->c;
        st.pg_norm = std::sqrt(pg2);
        st.n_active = (int64_t)na;
        st.n_free = h->n_global - st.n_active;
        st.n_active_nonbinding = (int64_t)nnb;
    }
    st.t_cg_ms = t_cg;
    st.t_gp_ms = t_gp;
    st.status = status;
    st.kernel_launches = (int32_t)(h->launches & 0x7fffffff);
    st.cg_iters_timed = h->cg_iters_timed;
    st.cg_free_iters_timed = h->cg_free_iters_timed;
    st.t_cg_timed_ms = h->t_cg_timed_ms;
    st.t_extract_ms = h->t_extract_ms;
    st.t_total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    if (stats) *stats = st;
    RC(leave(h));
    return status;

fail:
    // on ESEARCH / ENOTSPD return the last feasible iterate
    {
        const std::string msg = g_err;
        cudaGetLastError();
        download_vec(h, x_out, vy(cur));
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

#ifdef GPCG_DIAG_TIMES
// diagnostic builds only: the k6_gp_loop stamps of the last launch (ns, [step][cta][5])
GPCG_API int gpcg_diag_gp_times(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, g_diag_t, sizeof(g_diag_t)) == cudaSuccess ? 0 : -1;
}
#endif
}  // extern "C"
