// march_tma.cuh -- TMA-fed column march (sm_100a) for the broadcast-face
// 5-point operator (journal-bearing family C0 / C2 / C3): the CG iteration (a5),
// the fused accept / regrad / Cauchy sweep (a1 + a2) and the projected search
// (a3) of SURVEY.md 8(a).
//
// Work item = a BAND of 4 x 28 = 112 output columns (one warp per 28-column
// strip, 2 halo lanes per side, as in march.cuh) times a SEGMENT of grid rows.
// The raw rows of the segment plus 2 rows of warm-up on each side stream
// through shared memory in blocks of kBR rows: one thread issues
// cp.async.bulk.tensor.2d loads (f64 boxes 116 columns wide, u8 mask boxes) up
// to NST blocks ahead, completion counted on one mbarrier per stage.  The
// warps march down the block rows with the column-march recurrences of
// march.cuh (values at west / east neighbours by warp shuffle, north / south
// from a register window), so each raw value is read from shared memory once
// and no register ring is needed to hide HBM latency.  Out-of-grid rows and
// columns are zero-filled by the TMA unit (the Dirichlet boundary; ghost rows
// of a slab are inside the tensor).  Each CTA takes one (band, segment) item
// (grid = bands x segments sized to the resident CTAs); the loop is persistent
// for grids wider than that, with the load pipeline running across items.
//
// Same arithmetic and reduction structure as the k2_* kernels; checked against
// the CPU oracle by the same tests.
#pragma once

#include "common.cuh"
#include "fin.cuh"
#include "march.cuh"
#include "tma.cuh"

namespace gpcg {

#ifndef GPCG_CG_NST
#define GPCG_CG_NST 4       // CG sweep pipeline stages (tuning)
#endif
#ifndef GPCG_M4_WARPS
#define GPCG_M4_WARPS 8     // consumer warps per CTA of the band engines: 8 halves the CTAs of the
                            // persistent loops (grid barrier and partial sums) against 4 (-5 % per step)
#endif
#ifndef GPCG_CG_MINB
#define GPCG_CG_MINB (16 / GPCG_M4_WARPS)   // CG sweep CTAs per SM the register budget is sized for
#endif
#ifndef GPCG_GP_BR
#define GPCG_GP_BR 6        // rows per pipeline block of the GP-family (k5 / k6_gp_loop) sweeps (tuning: 6 rows x
                            // 2 stages 3 % faster than 4 x 3 and 8 x 2 on C3)
#endif
#ifndef GPCG_GP_NST
#define GPCG_GP_NST 2       // pipeline stages of the g-free GP sweeps (k5 / k6_gp_loop; tuning: 3 stages
                            // and 3 CTAs per SM measured 3 % faster than 4 and 2 on C3)
#endif
#ifndef GPCG_GP_MINB
#define GPCG_GP_MINB 3      // CTAs per SM the GP sweeps' register budget is sized for
#endif
namespace m4 {
constexpr int kWarps = GPCG_M4_WARPS;     // consumer warps (one per 28 / 26-column strip)
constexpr int kMinB = 16 / kWarps;        // CTAs per SM the register budgets are sized for (64 warps)
constexpr int kThreads = 32 * kWarps;     // lock-step engine: thread 0 also issues the TMA loads
constexpr int kThreadsWS = 32 * (kWarps + 1);  // warp-specialised engine: + one TMA producer warp
constexpr int kOut = 28 * kWarps;         // output columns per band (224 at 8 warps)
constexpr int kBW = kOut + 4;             // box columns (2 halo each side)
constexpr int kMW = (kBW + 15 + 15) / 16 * 16;   // u8 mask box width (start floored to 16 B): 144 at 4 warps
constexpr int kBR = 4;                    // rows per pipeline block (small stages: 3-4 CTAs per SM)
constexpr int r128(int b) { return (b + 127) / 128 * 128; }
constexpr int kF = kBR * kBW * 8;         // one f64 band box
constexpr int kFo = kBR * kOut * 8;       // one f64 box of the output columns only
constexpr int kUt = kBR * kMW;            // bytes delivered for one u8 mask box
constexpr int kU = r128(kUt);             // reserved (stage arrays stay 128-byte aligned)
static_assert(kF % 128 == 0 && kFo % 128 == 0, "TMA destinations stay 128-byte aligned");
}  // namespace m4

struct BandGeom {
    int nbands, nsegs, seg;     // items = nbands * nsegs; item rows [s*seg, min((s+1)*seg, ny))
    int rlo;                    // first tensor row (StencilOp::rlo)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// The pipeline engine (warp-specialised).  Warp kWarps is the producer: its lane 0 walks
// the CTA's block sequence and, once the consumers have released a stage (empty
// mbarrier, one arrival per consumer warp), issues the TMA loads of the next block into
// it (full mbarrier, transaction bytes).  The consumer warps wait on the full barrier,
// march their rows and release the stage -- no CTA-wide barrier per block, so warps
// drift up to NST blocks apart.  issue(stage_ptr, x0, yr, bar): the loads of the block
// whose first raw row is yr (band output columns start at x0); begin(x0, y0, y1): a new
// item (consumers); row(stage_ptr, kk, r): one raw row.  OUT = output columns per band;
// the raw rows of an item run from y0 - PRE to y1 - 1 + POST.  The producer warp leaves
// with nothing accumulated and joins the block reduction afterwards.
// k0: blocks this CTA already streamed through the same barriers (a persistent kernel
// calls the engine once per sweep; the mbarriers are initialised at k0 = 0 only and
// their phases continue).  Returns the CTA's block count after the sweep.
// flags (nullable): 16 bits per (item, block) -- bit w: the block's raw rows hold a free point
// in consumer warp w's input columns, bit 8 + w: its emitted rows do in warp w's output columns
// -- passed to issue_loads so that warps whose rows are all active skip the loads they never
// read (0xffff = load everything).  Every lane of the producer warp calls issue_loads.
template <int NST, int STAGE, int OUT = m4::kOut, int PRE = 2, int POST = 2, class Issue, class Begin, class Row>
__device__ __forceinline__ int band_pipeline_ws(const BandGeom& G, int ny, unsigned char* smem, Issue&& issue_loads,
                                                Begin&& begin, Row&& row, int k0 = 0,
                                                const unsigned short* __restrict__ flags = nullptr, int bid = -1,
                                                int nb = -1) {
    using namespace m4;
    if (bid < 0) { bid = blockIdx.x; nb = gridDim.x; }
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STAGE);
    uint64_t* empty = full + NST;
    const int nitems = G.nbands * G.nsegs;
    const int nblk = (G.seg + PRE + POST + kBR - 1) / kBR;
    int nmine = 0;
    for (int t = bid; t < nitems; t += nb) nmine += nblk;
    if (k0 == 0) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < NST; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], kWarps);
            }
            fence_mbar_init();
        }
        __syncthreads();
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == kWarps) {                                 // producer (the warp fetches flags, issues loads)
        int k = k0;
        for (int t = bid; t < nitems; t += nb) {
            const int x0 = (t % G.nbands) * OUT;
            const int yb = (t / G.nbands) * G.seg - PRE;
            int f = 0xffff;
            for (int b = 0; b < nblk; ++b, ++k) {
                if (flags && (b & 31) == 0)
                    f = (b + lane < nblk) ? __ldg(flags + (long long)t * nblk + b + lane) : 0xffff;
                const int fb = flags ? __shfl_sync(0xffffffffu, f, b & 31) : 0xffff;
                const int stage = k % NST;
                if (k >= NST) mbar_wait(&empty[stage], ((k / NST) - 1) & 1);
                issue_loads(smem + stage * STAGE, x0, yb + b * kBR, &full[stage], fb);
                __syncwarp();
            }
        }
        return k0 + nmine;
    }
    int k = k0;
    for (int t = bid; t < nitems; t += nb) {
        const int x0 = (t % G.nbands) * OUT;
        const int y0 = (t / G.nbands) * G.seg, y1 = min(y0 + G.seg, ny);
        begin(x0, y0, y1);
        for (int b = 0; b < nblk; ++b, ++k) {
            const int stage = k % NST;
            unsigned char* st = smem + stage * STAGE;
            mbar_wait(&full[stage], (k / NST) & 1);
            const int yr = y0 - PRE + b * kBR;
#pragma unroll
            for (int kk = 0; kk < kBR; ++kk) row(st, kk, yr + kk);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);    // this warp is done with the stage
        }
    }
    return k0 + nmine;
}

// Lock-step variant: after the CTA barrier that retires block k, ONE lane issues the loads of
// block k + NST into the freed stage.  The issuing warp rotates with k (warp k mod W), so the
// refill work -- a few dozen instructions a block -- is spread over the warps instead of
// putting warp 0 behind the others at every barrier, and the block to issue next is kept as a
// cursor in shared memory (item, block, its x0 and first row), advanced without divisions.
// bars: NST mbarriers (null: after the stages); k0 as in band_pipeline_ws (init at 0 only).
template <int NST, int STAGE, int OUT = m4::kOut, int PRE = 2, int POST = 2, int BR = m4::kBR, class Issue,
          class Begin, class Row>
__device__ __forceinline__ int band_pipeline(const BandGeom& G, int ny, unsigned char* smem, Issue&& issue_loads,
                                             Begin&& begin, Row&& row, uint64_t* bars = nullptr, int k0 = 0,
                                             int bid = -1, int nb = -1) {
    using namespace m4;
    constexpr int NW = m4::kThreads / 32;
    if (bid < 0) { bid = blockIdx.x; nb = gridDim.x; }
    uint64_t* bar = bars ? bars : reinterpret_cast<uint64_t*>(smem + NST * STAGE);
    const int nitems = G.nbands * G.nsegs;
    const int nblk = (G.seg + PRE + POST + BR - 1) / BR;
    int nmine = 0;
    for (int t = bid; t < nitems; t += nb) nmine += nblk;
    __shared__ int cur[4];                               // next block to issue: item t, block b, x0, row
    // issue the block at the cursor into the stage of local block index k; advance the cursor
    auto issue_next = [&](int k, int& t, int& b, int& x0, int& yr) {
        if (t >= nitems) return;
        const int stage = (k0 + k) % NST;
        issue_loads(smem + stage * STAGE, x0, yr, &bar[stage]);
        yr += BR;
        if (++b == nblk) {
            b = 0;
            t += nb;
            x0 = (t % G.nbands) * OUT;
            yr = (t / G.nbands) * G.seg - PRE;
        }
    };
    if (threadIdx.x == 0) {
        if (k0 == 0) {
            for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
            fence_mbar_init();
        }
        int t = bid, b = 0, x0 = (t % G.nbands) * OUT, yr = (t / G.nbands) * G.seg - PRE;
        for (int k = 0; k < NST; ++k) issue_next(k, t, b, x0, yr);
        cur[0] = t; cur[1] = b; cur[2] = x0; cur[3] = yr;
    }
    __syncthreads();
    int k = 0;
    for (int t = bid; t < nitems; t += nb) {
        const int x0 = (t % G.nbands) * OUT;
        const int y0 = (t / G.nbands) * G.seg, y1 = min(y0 + G.seg, ny);
        begin(x0, y0, y1);
        for (int b = 0; b < nblk; ++b, ++k) {
            const int stage = (k0 + k) % NST;
            unsigned char* st = smem + stage * STAGE;
            mbar_wait(&bar[stage], ((k0 + k) / NST) & 1);
            const int yr = y0 - PRE + b * BR;
#pragma unroll
            for (int kk = 0; kk < BR; ++kk) row(st, kk, yr + kk);
            __syncthreads();                              // every warp is done with this stage
            if (threadIdx.x == (k % NW) * 32) {
                fence_proxy_async();
                int ct = cur[0], cb = cur[1], cx = cur[2], cy = cur[3];
                issue_next(k + NST, ct, cb, cx, cy);
                cur[0] = ct; cur[1] = cb; cur[2] = cx; cur[3] = cy;
            }
        }
    }
    return k0 + nmine;
}

// Several slabs of one device in ONE persistent kernel (SURVEY.md 8(e) row slabs; the
// multi-slab counterpart of k6_cg_loop / k6_gp_loop): the CTAs of slab s are the grid range
// [cta0, cta0 + nb), bid = blockIdx.x - cta0 their index within the slab.  Fused halo
// exchange: every output row a neighbour slab keeps as a ghost row is also stored straight
// into that neighbour's ghost rows by the CTA that produces it, so the ghost rows are current
// after the grid barrier that ends the sweep -- no exchange step, no extra barrier, the
// transfer overlaps the sweep.  lo_rows: owned rows of the lower neighbour (slab s - 1);
// lo_ghost / hi_ghost: ghost rows the lower / upper neighbour keeps of this slab (0: none).
struct SlabLink {
    int bid, nb;
    int lo_rows;
    int lo_ghost, hi_ghost;
};

// ============================================================================
// a5: CG iteration, same recurrences as k2_cg_iter:
//   level 1  pn(r)   = [r in F] (rho(r) + beta p(r))
//   level 2  rn(r-1) = [r-1 in F] (rho(r-1) - alpha (A pn)(r-1))
//   level 3  q(r-2)  = (A rn)(r-2);  emit r-2 (free points): w += alpha pn, rho' = rn, p' = pn,
//            gamma += rn^2, delta += rn q
// Stage: rho | p (band boxes, rows yr..) | w (output columns, rows yr-2..) | mask (rows yr..)
// ============================================================================
// Two stage layouts (a run-time choice, `pw`): band boxes (one 228-column box per array and
// block: 3 TMA operations a block, best when the vectors stay in L2, C2) or per-warp boxes
// (warp w's rho / p box holds its 32 input columns, 28 outputs + 2 halo each side, its w box
// its 28 output columns), so that a warp whose rows hold no free point skips its loads (the
// band's other warps still load theirs): fewer DRAM bytes on large grids with large active
// regions (C3), 8x the TMA operations.
namespace m4cg {
using namespace m4;
// band layout
constexpr int kRhoB = 0, kPB = kF, kWBd = 2 * kF, kMB = 2 * kF + kFo;
// per-warp layout
constexpr int kPW = 32, kWW = 28;                     // per-warp rho / p and w box columns
constexpr int kFW = kBR * kPW * 8;                    // one per-warp rho / p box (1 KB)
constexpr int kWB = kBR * kWW * 8;                    // one per-warp w box (896 B)
constexpr int kRho = 0, kP = kWarps * kFW, kW = 2 * kWarps * kFW;
constexpr int kM = r128(kW + kWarps * kWB);
constexpr int kStage = (kM > kMB ? kM : kMB) + kU;
constexpr int kNST = GPCG_CG_NST;
constexpr int kSmem = kNST * kStage + 64;
static_assert(kFW % 128 == 0 && kWB % 128 == 0 && kW % 128 == 0 && kMB % 128 == 0,
              "TMA destinations stay 128-byte aligned");
}  // namespace m4cg

// One CG sweep on this CTA's items: rho_n, p_n, w written for the free points; acc = this
// thread's (gamma, delta) contributions.  Returns the CTA's running TMA block count.
template <bool PC>
__device__ __forceinline__ int cg_sweep4(const StencilOp& A, const BandGeom& G, const CUtensorMap* m_rho,
                                         const CUtensorMap* m_p, const CUtensorMap* m_w, const CUtensorMap* m_mask,
                                         double* __restrict__ rho_n, double* __restrict__ p_n, double* __restrict__ w_out,
                                         double alpha, double beta, unsigned char* smem, double (&acc)[2], int k0,
                                         const unsigned short* __restrict__ flags = nullptr, bool pw = false,
                                         const SlabLink* L = nullptr, double* lo_rho = nullptr, double* lo_p = nullptr,
                                         double* hi_rho = nullptr, double* hi_p = nullptr) {
    using namespace m4cg;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 28 * wid + lane;                        // box column of this lane
    const bool out_lane = lane >= 2 && lane < 30;
    int gx = 0, moff = 0, y0 = 0, y1 = 0;
    bool col_ok = false;
    Op5<true> op;
    double pn_m2 = 0.0, pn_m1 = 0.0, rho_m1 = 0.0, rn_m3 = 0.0, rn_m2 = 0.0, rr_m2 = 0.0, dinv = 0.0;
    unsigned char m_m1 = 0, m_m2 = 0;
    return band_pipeline_ws<kNST, kStage>(
        G, A.ny, smem,
        [&](unsigned char* st, int x0, int yr, uint64_t* bar, int fb) {
            // (every producer lane) rho / p are read only at free points of the raw rows, w only
            // at free emitted rows: per warp strip, boxes without any (flags bits w / 8 + w)
            // are skipped (stale smem is never read: every use is masked)
            const int plane = threadIdx.x & 31;
            const unsigned fd = fb & 0xff, fw = (fb >> 8) & 0xff;
            if (!pw) {                                        // band boxes, one lane
                if (plane == 0) {
                    mbar_expect_tx(bar, kUt + (fd ? 2 * kF : 0) + (fw ? kFo : 0));
                    if (fd) {
                        tma_load_2d(st + kRhoB, m_rho, x0 - 2, yr - G.rlo, bar);
                        tma_load_2d(st + kPB, m_p, x0 - 2, yr - G.rlo, bar);
                    }
                    if (fw) tma_load_2d(st + kWBd, m_w, x0, yr - 2 - G.rlo, bar);
                    tma_load_2d(st + kMB, m_mask, floor16(x0 - 2), yr - G.rlo, bar);
                }
                return;
            }
            if (plane == 0) mbar_expect_tx(bar, kUt + __popc(fd) * 2 * kFW + __popc(fw) * kWB);
            __syncwarp();
            if (plane < kWarps) {
                if ((fd >> plane) & 1) {
                    tma_load_2d(st + kRho + plane * kFW, m_rho, x0 - 2 + 28 * plane, yr - G.rlo, bar);
                    tma_load_2d(st + kP + plane * kFW, m_p, x0 - 2 + 28 * plane, yr - G.rlo, bar);
                }
            } else if (plane < 2 * kWarps) {
                const int w = plane - kWarps;                 // w of the emitted rows (r - 2)
                if ((fw >> w) & 1) tma_load_2d(st + kW + w * kWB, m_w, x0 + 28 * w, yr - 2 - G.rlo, bar);
            } else if (plane == 2 * kWarps) {
                tma_load_2d(st + kM, m_mask, floor16(x0 - 2), yr - G.rlo, bar);
            }
        },
        [&](int x0, int yb, int ye) {
            gx = x0 - 2 + c;
            moff = (x0 - 2) - floor16(x0 - 2);
            y0 = yb;
            y1 = ye;
            col_ok = gx >= 0 && gx < A.nx;
            op.init(A, gx);
            dinv = op.dinv(A, 0);
            pn_m2 = pn_m1 = rho_m1 = rn_m3 = rn_m2 = rr_m2 = 0.0;
            m_m1 = m_m2 = 0;
        },
        [&](const unsigned char* st, int kk, int r) {
            const double* rhoS = reinterpret_cast<const double*>(st + (pw ? kRho + wid * kFW : kRhoB));
            const double* pS = reinterpret_cast<const double*>(st + (pw ? kP + wid * kFW : kPB));
            const int qi = pw ? kk * kPW + lane : kk * kBW + c;
            const unsigned char m = st[(pw ? kM : kMB) + kk * kMW + c + moff];
            const double rho = m ? rhoS[qi] : 0.0;
            const double pn0 = m ? fma(beta, pS[qi], PC ? rho * dinv : rho) : 0.0;
            const double ap = op.apply(A, r - 1, pn_m1, pn_m2, pn0);
            const double rr1 = m_m1 ? fma(-alpha, ap, rho_m1) : 0.0;
            const double rn1 = PC ? rr1 * dinv : rr1;
            const double q = op.apply(A, r - 2, rn_m2, rn_m3, rn1);
            const int r2 = r - 2;
            const double rres = PC ? rr_m2 : rn_m2;
            if (out_lane && m_m2 && col_ok && r2 >= y0 && r2 < y1) {
                const long long v = (long long)gx + (long long)A.pitch * r2;
                const double* wS = reinterpret_cast<const double*>(st + (pw ? kW + wid * kWB : kWBd));
                w_out[v] = fma(alpha, pn_m2, wS[pw ? kk * kWW + lane - 2 : kk * kOut + c - 2]);
                rho_n[v] = rres;
                p_n[v] = pn_m2;
                acc[0] = fma(rres, rn_m2, acc[0]);
                acc[1] = fma(rn_m2, q, acc[1]);
                if (L) {                                      // fused halo write (SlabLink)
                    if (r2 < L->lo_ghost) {
                        const long long vl = (long long)gx + (long long)A.pitch * (L->lo_rows + r2);
                        lo_rho[vl] = rres;
                        lo_p[vl] = pn_m2;
                    }
                    if (r2 >= A.ny - L->hi_ghost) {
                        const long long vh = (long long)gx + (long long)A.pitch * (r2 - A.ny);
                        hi_rho[vh] = rres;
                        hi_p[vh] = pn_m2;
                    }
                }
            }
            pn_m2 = pn_m1; pn_m1 = pn0;
            rho_m1 = rho;
            m_m2 = m_m1; m_m1 = m;
            rn_m3 = rn_m2; rn_m2 = rn1;
            rr_m2 = rr1;
        },
        k0, flags, L ? L->bid : -1, L ? L->nb : -1);
}

// ============================================================================
// a4: y = A v (full) or y = Z Z' A Z Z' v on the free mask (reduced), as k_hessvec, on the
// TMA-fed march (broadcast faces): level 1 u(r) = [r in F] v(r) (reduced) or v(r); level 2
// y(r-1) = (A u)(r-1), 0 off F (reduced).  Stage: v band box | mask box.
// ============================================================================
namespace m4hv {
using namespace m4;
constexpr int kV = 0, kM = kF;
constexpr int kStage = kF + kU;
constexpr int kNST = 8;
constexpr int kSmem = kNST * kStage + 64;
}  // namespace m4hv

template <bool RED>
__global__ void __launch_bounds__(m4::kThreadsWS, m4::kMinB)
k4_hessvec(StencilOp A, BandGeom G, const __grid_constant__ CUtensorMap m_v, const __grid_constant__ CUtensorMap m_mask,
           double* __restrict__ y) {
    using namespace m4hv;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 28 * wid + lane;
    const bool out_lane = lane >= 2 && lane < 30;
    int gx = 0, moff = 0, y0 = 0, y1 = 0;
    bool col_ok = false;
    Op5<true> op;
    double u_m1 = 0.0, u_m2 = 0.0;
    unsigned char m_m1 = 0;
    band_pipeline_ws<kNST, kStage, kOut, 1, 1>(
        G, A.ny, smem,
        [&](unsigned char* st, int x0, int yr, uint64_t* bar, int) {
            if ((threadIdx.x & 31) != 0) return;          // one producer lane issues
            mbar_expect_tx(bar, kF + (RED ? kUt : 0));
            tma_load_2d(st + kV, &m_v, x0 - 2, yr - G.rlo, bar);
            if (RED) tma_load_2d(st + kM, &m_mask, floor16(x0 - 2), yr - G.rlo, bar);
        },
        [&](int x0, int yb, int ye) {
            gx = x0 - 2 + c;
            moff = (x0 - 2) - floor16(x0 - 2);
            y0 = yb;
            y1 = ye;
            col_ok = gx >= 0 && gx < A.nx;
            op.init(A, gx);
            u_m1 = u_m2 = 0.0;
            m_m1 = 0;
        },
        [&](const unsigned char* st, int kk, int r) {
            const unsigned char m = RED ? st[kM + kk * kMW + c + moff] : 1;
            const double vv = reinterpret_cast<const double*>(st + kV)[kk * kBW + c];
            const double u0 = m ? vv : 0.0;
            const double q = op.apply(A, r - 1, u_m1, u_m2, u0);
            const int r1 = r - 1;
            if (out_lane && col_ok && r1 >= y0 && r1 < y1)
                y[(long long)gx + (long long)A.pitch * r1] = m_m1 ? q : 0.0;
            u_m2 = u_m1; u_m1 = u0;
            m_m1 = m;
        });
}

// Block flags of the CG sweep geometry G for the fixed CG mask, 16 bits per (item, block):
// bit w if rows [yr, yr+4) of consumer warp w's input columns [x0 + 28 w - 2, x0 + 28 w + 30)
// hold a free point, bit 8 + w if rows [yr-2, yr+2) of its output columns [x0 + 28 w,
// x0 + 28 w + 28) do.  One warp per (item, block); lanes stride the columns.
__global__ void k_cg_block_flags(int nx, int pitch, BandGeom G, const unsigned char* __restrict__ mask, int rhi,
                                 unsigned short* __restrict__ flags) {
    using namespace m4;
    const int nblk = (G.seg + 4 + kBR - 1) / kBR;
    const long long total = (long long)G.nbands * G.nsegs * nblk;
    const int lane = threadIdx.x & 31;
    const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long q = w0; q < total; q += nw) {
        const int t = (int)(q / nblk), b = (int)(q - (long long)t * nblk);
        const int x0 = (t % G.nbands) * kOut;
        const int yr = (t / G.nbands) * G.seg - 2 + b * kBR;
        unsigned int bits = 0;
        // all the block's mask bytes are independent loads: unrolled so they are in flight together
#pragma unroll
        for (int rr = 0; rr < kBR + 2; ++rr) {
            const int r = yr - 2 + rr;
            if (r < G.rlo || r >= rhi) continue;
            const unsigned char* row = mask + (long long)r * pitch;
#pragma unroll
            for (int cc = 0; cc < (kOut + 4 + 31) / 32; ++cc) {
                const int o = lane + 32 * cc - 2;             // column offset from x0: -2 .. kOut + 1
                const int c = x0 + o;
                if (o >= kOut + 2 || c < 0 || c >= nx || !row[c]) continue;
                if (r >= yr) {                                // raw rows: input strips holding o
                    const int ws = (o + 2) / 28;
                    if (ws < kWarps) bits |= 1u << ws;
                    if (ws >= 1 && o < 28 * ws + 2) bits |= 1u << (ws - 1);
                }
                if (r < yr + kBR - 2 && o >= 0 && o < kOut) bits |= 1u << (8 + o / 28);   // emitted rows
            }
        }
        bits = __reduce_or_sync(0xffffffffu, bits);
        if (lane == 0) flags[q] = (unsigned short)bits;
    }
}

template <bool PC>     // point-Jacobi PCG as in k2_cg_iter<BC, true>
__global__ void __launch_bounds__(m4::kThreadsWS, GPCG_CG_MINB)
k4_cg_iter(StencilOp A, BandGeom G, const __grid_constant__ CUtensorMap m_rho, const __grid_constant__ CUtensorMap m_p,
           const __grid_constant__ CUtensorMap m_w, const __grid_constant__ CUtensorMap m_mask,
           double* __restrict__ rho_n, double* __restrict__ p_n, double* __restrict__ w_out, Scal* S, RedScratch R,
           const unsigned short* __restrict__ flags, int pw) {
    if (*(volatile int*)&S->cg_done) return;
    const double alpha = S->cg_alpha, beta = S->cg_beta;
    extern __shared__ __align__(128) unsigned char smem[];
    double acc[2] = {0.0, 0.0};
    cg_sweep4<PC>(A, G, &m_rho, &m_p, &m_w, &m_mask, rho_n, p_n, w_out, alpha, beta, smem, acc, 0, flags, pw != 0);
    reduce_and_finish<2>(acc, R, [&](double* tt) { cg_finalize(tt[0], tt[1], S); });
}

// ============================================================================
// a5 as ONE persistent cooperative launch per CG call (single slab, single rank): every
// iteration is a sweep, a block reduction, a grid barrier, and the finaliser evaluated
// redundantly by every CTA on the same fixed-order sum of the block partials (so every
// CTA takes the same decision without a second barrier).  No launch per iteration, no
// host poll; the loop stops at cgstop1 / the exact-solve guard / the cap / breakdown.
// rho and p ping-pong between buffers 0 / 1 by iteration parity (same as the graph path).
// ============================================================================
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks, unsigned int& gen) {
    // this thread's global writes become visible to the async proxy (the next sweep's TMA loads)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();                                  // release the CTA's writes at gpu scope
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

// ---------------------------------------------------------------- cross-rank groups
// The persistent loops spanning several ranks (one device each, or -- the one-launch emulation
// GPCG_XRANK_EMU -- several CTA groups of one launch).  Every rank owns, in its own memory, a
// local counter (its CTAs' arrivals), a go flag, a cross counter (one arrival per rank and
// barrier) and a partial-sum mailbox with a row per global CTA id; the other ranks reach the
// cross counter and the mailbox through peer mappings.  One reduction:
//   1. every CTA stores its block partials into EVERY rank's mailbox at its global id and
//      arrives on its rank's local counter (release, gpu scope);
//   2. the rank's leader (its first CTA) waits for the rank's CTAs (acquire, gpu), fences at
//      system scope and arrives on EVERY rank's cross counter; it waits for its own cross
//      counter to count every rank (relaxed polls, then an acquire fence at system scope) and
//      releases its rank through the go flag (gpu scope);
//   3. every CTA sums its own rank's mailbox over all global ids in order -- so every rank
//      forms the same bits and takes the same decision with no second round trip.
// The PTX memory model's causality order is transitive: a CTA's stores to a peer (ghost rows,
// partials) precede its local release, which the leader acquires before its system-scope
// release -- so only the leaders' two operations per reduction need system scope (gpu scope in
// the one-device emulation, whose ranks share the device).  One NVLink
// round trip per reduction and nr cross arrivals per rank, whatever the CTA count.
// Counters are never reset: a rank's base (its counters and barrier count before the running
// launch) is advanced by the rank's leader at the end of each launch; every rank runs the same
// barriers (identical decisions), so all bases agree.  The mailbox slot is the parity of the
// GLOBAL barrier count and the slots' layout does not depend on the launch's CTA count, so a
// fast rank's first partials of the next launch never land in the slot a slow rank is still
// summing.  A spin that outlasts kXrSpinNs sets *err and lets the CTA go on (the host turns it
// into an error instead of a hang).
constexpr int kMaxRanks = 8;
constexpr int kXrSums = 8;                    // sums per reduction (GP accept: 8, CG: 2)
constexpr int kXrLine = 16;                   // u64 per counter: one 128-byte line each
constexpr unsigned long long kXrSpinNs = 20ull * 1000 * 1000 * 1000;
struct XRank {
    int nr;                                   // ranks
    int cta_base;                             // global id of this launch's CTA 0
    int cta_total;                            // CTAs over all ranks in this launch
    int cta_stride;                           // mailbox row length (>= cta_total of every launch)
    int cta0[kMaxRanks + 1];                  // global CTA range of rank r: [cta0[r], cta0[r + 1])
    unsigned long long* lbar[kMaxRanks];      // rank r's local counter (own rank only); lbar + kXrLine: its go flag
    unsigned long long* bar[kMaxRanks];       // rank r's cross counter
    unsigned long long* base[kMaxRanks];      // rank r's {local, cross, barriers} before the launch (own rank only)
    double* part[kMaxRanks];                  // rank r's mailbox: [2 slots][kXrSums][cta_stride]
    int* err;                                 // this rank's spin-timeout flag
    int sys;                                  // ranks on several devices: the leaders' operations at system
                                              // scope (the one-device emulation: gpu scope suffices)
};
struct XCtx {
    int me;                                   // this CTA's rank
    int gid;                                  // global CTA id
    int tr;                                   // CTAs of this rank
    bool leader;                              // the rank's first CTA
    unsigned long long lb0, xb0, n0;          // the rank's base (local, cross arrivals; barriers)
};

__device__ __forceinline__ XCtx xr_ctx(const XRank& X) {
    XCtx c;
    c.gid = X.cta_base + (int)blockIdx.x;
    c.me = 0;
    while (c.me + 1 < X.nr && c.gid >= X.cta0[c.me + 1]) ++c.me;
    c.tr = X.cta0[c.me + 1] - X.cta0[c.me];
    c.leader = c.gid == X.cta0[c.me];
    const volatile unsigned long long* b = X.base[c.me];
    c.lb0 = b[0];
    c.xb0 = b[1];
    c.n0 = b[2];
    return c;
}

__device__ __forceinline__ unsigned long long xr_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// spin until *ctr >= target: acquire loads at gpu scope, or (cross) relaxed loads and one acquire
// fence at system scope (gpu scope when sys == 0)
template <bool CROSS>
__device__ __forceinline__ void xr_wait(const unsigned long long* ctr, unsigned long long target, int* err,
                                        int sys = 0) {
    unsigned long long v;
    const unsigned long long t0 = xr_now();
    for (;;) {
        if (CROSS && sys) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        else if (CROSS) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        if (v >= target) break;
        if (xr_now() - t0 > kXrSpinNs) { atomicExch(err, 1); break; }
    }
    if (CROSS && sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else if (CROSS) asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// reduction number gen of this launch (every thread counts)
__device__ __forceinline__ void xr_barrier(const XRank& X, const XCtx& c, unsigned int& gen) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long xtarget = c.xb0 + (unsigned long long)(gen + 1) * (unsigned long long)X.nr;
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(X.lbar[c.me]) : "memory");
        if (c.leader) {
            xr_wait<false>(X.lbar[c.me], c.lb0 + (unsigned long long)(gen + 1) * (unsigned long long)c.tr, X.err);
            if (X.sys) {
                asm volatile("fence.acq_rel.sys;" ::: "memory");
                for (int r = 0; r < X.nr; ++r)
                    asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(X.bar[r]) : "memory");
            } else {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                for (int r = 0; r < X.nr; ++r)
                    asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(X.bar[r]) : "memory");
            }
            xr_wait<true>(X.bar[c.me], xtarget, X.err, X.sys);
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(X.lbar[c.me] + kXrLine), "l"(xtarget)
                         : "memory");
        } else {
            xr_wait<false>(X.lbar[c.me] + kXrLine, xtarget, X.err);
        }
    }
    ++gen;
    __syncthreads();
    asm volatile("fence.proxy.async.global;" ::: "memory");  // peers' ghost-row stores before this CTA's TMA loads
}

// fixed-order sum of NS block partials over every rank's CTAs (the same bits on every rank)
template <int NS>
__device__ __forceinline__ void xr_grid_sum(double (&acc)[NS], const XRank& X, const XCtx& c, unsigned int& gen,
                                            double* red, double* tot) {
    block_reduce<NS>(acc, red);
    const size_t T = (size_t)X.cta_stride;
    const size_t off = (size_t)((c.n0 + gen) & 1ull) * kXrSums * T;
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < NS; ++q) tot[q] = acc[q];
    __syncthreads();
    for (int i = threadIdx.x; i < X.nr * NS; i += blockDim.x) {      // this CTA's row, into every mailbox
        const int r = i / NS, q = i - r * NS;
        X.part[r][off + q * T + c.gid] = tot[q];
    }
    xr_barrier(X, c, gen);
    const double* pp = X.part[c.me] + off;
    double t[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) t[q] = 0.0;
    for (unsigned int b = threadIdx.x; b < (unsigned int)X.cta_total; b += blockDim.x)
#pragma unroll
        for (int q = 0; q < NS; ++q) t[q] += __ldcg(pp + q * T + b);
    block_reduce<NS>(t, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < NS; ++q) tot[q] = t[q];
    __syncthreads();
}

// end of a launch: the rank's leader advances the rank's base by the launch's barriers
__device__ __forceinline__ void xr_close(const XRank& X, const XCtx& c, unsigned int gen) {
    if (threadIdx.x == 0 && c.leader) {
        unsigned long long* b = X.base[c.me];
        b[0] = c.lb0 + (unsigned long long)gen * (unsigned long long)c.tr;
        b[1] = c.xb0 + (unsigned long long)gen * (unsigned long long)X.nr;
        b[2] = c.n0 + gen;
    }
}

// The CG call loop shared by the single- and multi-slab persistent kernels: per iteration
// sweep(a, alpha, beta, acc, k) -> block partials -> grid barrier -> fixed-order sum of all
// CTAs' partials (the same in every CTA) -> cg_finalize evaluated in every CTA.
template <bool XR = false, class Sweep>
__device__ __forceinline__ void cg_loop(Scal* S, double* __restrict__ part, unsigned int* gbar, Sweep&& sweep,
                                        const XRank* X = nullptr) {
    __shared__ double red[2 * 32];
    __shared__ double tot[2];
    // CG state (identical in every CTA)
    double alpha = S->cg_alpha, beta = S->cg_beta, gamma_old = S->cg_gamma, maxdec = S->cg_maxdec;
    const double eta2 = S->cg_eta2, rnorm0 = S->cg_rnorm0;
    long long it = S->cg_it;
    const long long cap = S->cg_cap;
    int done = S->cg_done, reason = S->cg_reason;
    unsigned int gen = 0;
    int k = 0;
    const unsigned int G_ = gridDim.x;
    __shared__ XCtx xc;                           // in shared memory: no registers held across the sweeps
    if constexpr (XR) {
        if (threadIdx.x == 0) xc = xr_ctx(*X);
        __syncthreads();
        if (X->sys) xr_barrier(*X, xc, gen);      // ranks: no fused store before every peer left its last kernel
    }
    while (!done) {
        const int a = (int)(it & 1);
        double acc[2] = {0.0, 0.0};
        k = sweep(a, alpha, beta, acc, k);
        if constexpr (XR) {
            xr_grid_sum<2>(acc, *X, xc, gen, red, tot);
        } else {
            // block partials -> part[parity][s][block]
            block_reduce<2>(acc, red);
            double* pp = part + (it & 1) * 2 * G_;
            if (threadIdx.x == 0) {
                pp[blockIdx.x] = acc[0];
                pp[G_ + blockIdx.x] = acc[1];
            }
            grid_barrier(gbar, G_, gen);
            // fixed-order sum of the partials, same in every CTA
            double t[2] = {0.0, 0.0};
            for (unsigned int b = threadIdx.x; b < G_; b += blockDim.x) {
                t[0] += __ldcg(pp + b);
                t[1] += __ldcg(pp + G_ + b);
            }
            block_reduce<2>(t, red);
            if (threadIdx.x == 0) { tot[0] = t[0]; tot[1] = t[1]; }
            __syncthreads();
        }
        const double gamma = tot[0], delta = tot[1];
        // cg_finalize (fin.cuh), evaluated in every CTA
        const double dec = 0.5 * alpha * gamma_old;
        ++it;
        reason = CG_RUNNING;
        if (it >= 2 && dec <= eta2 * maxdec) reason = CG_PROGRESS;
        else if (sqrt(gamma) <= 1e-14 * (1.0 + rnorm0)) reason = CG_EXACT;
        else if (it >= cap) reason = CG_CAP;
        if (dec > maxdec) maxdec = dec;
        if (reason == CG_RUNNING) {
            const double beta_n = gamma / gamma_old;
            const double pap = delta - beta_n * gamma / alpha;
            beta = beta_n;
            if (!(pap > 0.0)) reason = CG_NOTSPD;
            else alpha = gamma / pap;
        }
        gamma_old = gamma;
        if (reason != CG_RUNNING) done = 1;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            S->cg_it = it;
            S->cg_dec = dec;
            S->cg_maxdec = maxdec;
            S->cg_gamma = gamma;
            S->cg_beta = beta;
            S->cg_alpha = alpha;
            S->cg_reason = reason;
            S->cg_done = done;
        }
    }
    if constexpr (XR) xr_close(*X, xc, gen);
    // (one device: the host zeroes the barrier counter before each launch)
}

template <bool PC>
__global__ void __launch_bounds__(m4::kThreadsWS, GPCG_CG_MINB)
k6_cg_loop(StencilOp A, BandGeom G, const __grid_constant__ CUtensorMap m_rho0, const __grid_constant__ CUtensorMap m_rho1,
           const __grid_constant__ CUtensorMap m_p0, const __grid_constant__ CUtensorMap m_p1,
           const __grid_constant__ CUtensorMap m_w, const __grid_constant__ CUtensorMap m_mask,
           double* __restrict__ rho0, double* __restrict__ rho1, double* __restrict__ p0, double* __restrict__ p1,
           double* __restrict__ w_out, Scal* S, double* __restrict__ part, unsigned int* gbar,
           const unsigned short* __restrict__ flags, int pw) {
    extern __shared__ __align__(128) unsigned char smem[];
    cg_loop(S, part, gbar, [&](int a, double alpha, double beta, double (&acc)[2], int k) {
        return cg_sweep4<PC>(A, G, a ? &m_rho1 : &m_rho0, a ? &m_p1 : &m_p0, &m_w, &m_mask, a ? rho0 : rho1,
                             a ? p0 : p1, w_out, alpha, beta, smem, acc, k, flags, pw != 0);
    });
}

// k6_cg_loop over several slabs of one device (SlabLink): each slab's CTAs sweep its rows and
// write the rows its neighbours keep as ghosts into their ghost rows as well; one grid
// barrier and one fixed-order sum over all CTAs per iteration, as with one slab.  XR: the
// reductions through the cross-rank protocol (XRank) instead of the one-device grid barrier.
constexpr int kMaxMs = 8;
struct CgMsSlab {
    CUtensorMap m_rho0, m_rho1, m_p0, m_p1, m_w, m_mask;
    StencilOp A;
    BandGeom G;
    double *rho0, *rho1, *p0, *p1, *w;
    const unsigned short* flags;
    double *lo_rho0, *lo_rho1, *lo_p0, *lo_p1;    // lower neighbour's origins (slab s - 1)
    double *hi_rho0, *hi_rho1, *hi_p0, *hi_p1;    // upper neighbour's origins (slab s + 1)
    SlabLink L;                                   // bid is set in the kernel
    int cta0;
};
struct CgMsArgs {
    CgMsSlab s[kMaxMs];
    int nslabs;
    int pw;                                       // per-warp boxes (cg_sweep4)
};

template <bool PC, bool XR>
__global__ void __launch_bounds__(m4::kThreadsWS, GPCG_CG_MINB)
k6_cg_loop_ms(const __grid_constant__ CgMsArgs P, Scal* S, double* __restrict__ part, unsigned int* gbar,
              const __grid_constant__ XRank XRk) {
    extern __shared__ __align__(128) unsigned char smem[];
    int si = 0;
    while (si + 1 < P.nslabs && (int)blockIdx.x >= P.s[si + 1].cta0) ++si;
    const CgMsSlab& X = P.s[si];
    SlabLink L = X.L;
    L.bid = (int)blockIdx.x - X.cta0;
    auto body = [&](int a, double alpha, double beta, double (&acc)[2], int k) {
        return cg_sweep4<PC>(X.A, X.G, a ? &X.m_rho1 : &X.m_rho0, a ? &X.m_p1 : &X.m_p0, &X.m_w, &X.m_mask,
                             a ? X.rho0 : X.rho1, a ? X.p0 : X.p1, X.w, alpha, beta, smem, acc, k, X.flags,
                             P.pw != 0, &L,
                             a ? X.lo_rho0 : X.lo_rho1, a ? X.lo_p0 : X.lo_p1, a ? X.hi_rho0 : X.hi_rho1,
                             a ? X.hi_p0 : X.hi_p1);
    };
    cg_loop<XR>(S, part, gbar, body, &XRk);
}

// ============================================================================
// a1 + a2 fused (as k2_accept): accept / project, regrad, free mask, set counts
// and the Cauchy form of the new point.
//   level 1  yn(r)   = mid(l, u, y(r) + alpha sgn dir(r))   (or mid(l, u, y) without dir)
//   level 2  gn(r-1) = (A yn)(r-1) - b,  d(r-1) = grad_Omega q(yn)(r-1)
//   level 3  Ad(r-2) = (A d)(r-2);  emit row r-2
// Stage: y | dir | b | l | u (band boxes, rows yr..; dir, l/u optional) | mask_prev (rows yr-2..)
// ============================================================================
// BB: b is the same in every grid row (detected at create; the journal-bearing b depends on xi_1
// only) -> read once per column from brow, not streamed.
template <bool SB, bool HasDir, bool BB>
struct AccLayout4 {
    static constexpr int kY = 0;
    static constexpr int kD = m4::kF;
    static constexpr int kB = kD + (HasDir ? m4::kF : 0);
    static constexpr int kL = kB + (BB ? 0 : m4::kF);
    static constexpr int kU = kL + (SB ? 0 : m4::kF);
    static constexpr int kMP = kU + (SB ? 0 : m4::kF);
    static constexpr int kStage = kMP + m4::kU;
    static constexpr int kNST = 4;
    static constexpr int kSmem = kNST * kStage + 64;
};

template <bool SB, bool HasDir, bool BB>
__global__ void __launch_bounds__(m4::kThreads, m4::kMinB)
k4_accept(StencilOp A, BandGeom G, Bounds Bd, const double* __restrict__ brow, const __grid_constant__ CUtensorMap m_y,
          const __grid_constant__ CUtensorMap m_dir, const __grid_constant__ CUtensorMap m_b,
          const __grid_constant__ CUtensorMap m_l, const __grid_constant__ CUtensorMap m_u,
          const __grid_constant__ CUtensorMap m_mp, int has_mp, double sgn, double* __restrict__ y_out,
          double* __restrict__ g_out, unsigned char* __restrict__ mask_out, Scal* S, RedScratch R, int gp) {
    using namespace m4;
    using L = AccLayout4<SB, HasDir, BB>;
    if (gp && *(volatile int*)&S->gp_done) return;   // device-driven GP phase already over
    double alpha = 0.0;
    if (HasDir) {
        if (S->s_h < 0) return;                   // uniform: no accepted step in this batch
        alpha = S->s_alpha;
    }
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 28 * wid + lane;
    const bool out_lane = lane >= 2 && lane < 30;
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int gx = 0, moff = 0, y0 = 0, y1 = 0;
    bool col_ok = false;
    Op5<true> op;
    double yn_m2 = 0.0, yn_m1 = 0.0, b_m1 = 0.0, l_m1 = 0.0, u_m1 = 0.0, l_m2 = 0.0, u_m2 = 0.0;
    double gn_m2 = 0.0, d_m3 = 0.0, d_m2 = 0.0, bcol = 0.0;
    const uint32_t tx = L::kMP + (has_mp ? kUt : 0);
    band_pipeline<L::kNST, L::kStage>(
        G, A.ny, smem,
        [&](unsigned char* st, int x0, int yr, uint64_t* bar) {
            mbar_expect_tx(bar, tx);
            const int yt = yr - G.rlo;
            tma_load_2d(st + L::kY, &m_y, x0 - 2, yt, bar);
            if (HasDir) tma_load_2d(st + L::kD, &m_dir, x0 - 2, yt, bar);
            if (!BB) tma_load_2d(st + L::kB, &m_b, x0 - 2, yt, bar);
            if (!SB) {
                tma_load_2d(st + L::kL, &m_l, x0 - 2, yt, bar);
                tma_load_2d(st + L::kU, &m_u, x0 - 2, yt, bar);
            }
            if (has_mp) tma_load_2d(st + L::kMP, &m_mp, floor16(x0 - 2), yt - 2, bar);
        },
        [&](int x0, int yb, int ye) {
            gx = x0 - 2 + c;
            moff = (x0 - 2) - floor16(x0 - 2);
            y0 = yb;
            y1 = ye;
            col_ok = gx >= 0 && gx < A.nx;
            op.init(A, gx);
            if (BB) bcol = col_ok ? __ldg(brow + gx) : 0.0;
            yn_m2 = yn_m1 = b_m1 = l_m1 = u_m1 = l_m2 = u_m2 = gn_m2 = d_m3 = d_m2 = 0.0;
        },
        [&](const unsigned char* st, int kk, int r) {
            const int q = kk * kBW + c;
            // raw values; outside the readable rows / columns the bounds are 0 so yn = 0 (Dirichlet)
            const bool in = col_ok && r >= A.rlo && r < A.rhi;
            const double yv = reinterpret_cast<const double*>(st + L::kY)[q];
            const double bv = BB ? ((r >= A.rlo && r < A.rhi) ? bcol : 0.0)
                                 : reinterpret_cast<const double*>(st + L::kB)[q];
            const double lv = in ? (SB ? Bd.lc : reinterpret_cast<const double*>(st + L::kL)[q]) : 0.0;
            const double uv = in ? (SB ? Bd.uc : reinterpret_cast<const double*>(st + L::kU)[q]) : 0.0;
            double yn0;
            if constexpr (HasDir) yn0 = trial(yv, reinterpret_cast<const double*>(st + L::kD)[q], sgn, alpha, lv, uv);
            else yn0 = mid(lv, uv, yv);
            const double ay = op.apply(A, r - 1, yn_m1, yn_m2, yn0);
            const double gn1 = ay - b_m1;
            const double d1 = pgrad(yn_m1, gn1, l_m1, u_m1);      // 0 outside the grid
            const double ad = op.apply(A, r - 2, d_m2, d_m3, d1);
            const int r2 = r - 2;
            if (out_lane && col_ok && r2 >= y0 && r2 < y1) {
                const long long v = (long long)gx + (long long)A.pitch * r2;
                y_out[v] = yn_m2;
                g_out[v] = gn_m2;
                const bool act = (yn_m2 == l_m2) || (yn_m2 == u_m2);
                const unsigned char m = act ? 0 : 1;
                mask_out[v] = m;
                acc[0] = fma(d_m2, d_m2, acc[0]);
                acc[1] = fma(gn_m2, gn_m2, acc[1]);
                acc[2] += act ? 1.0 : 0.0;
                if (has_mp) acc[3] += (st[L::kMP + kk * kMW + c + moff] != m) ? 1.0 : 0.0;
                const bool binding = (yn_m2 == l_m2 && gn_m2 >= 0.0) || (yn_m2 == u_m2 && gn_m2 <= 0.0);
                acc[4] += (act && !binding) ? 1.0 : 0.0;
                acc[5] = fma(d_m2, ad, acc[5]);
            }
            yn_m2 = yn_m1; yn_m1 = yn0;
            l_m2 = l_m1; u_m2 = u_m1;
            l_m1 = lv; u_m1 = uv; b_m1 = bv;
            gn_m2 = gn1;
            d_m3 = d_m2; d_m2 = d1;
        });
    reduce_and_finish<6>(acc, R, [&](double* t) { fin_accept(t, true, S); });
}

// ============================================================================
// a3: projected search, K = 2 step sizes per sweep (as k2_search, H = 1; the
// band's 2-lane halo is kept, only the 28 centre lanes accumulate).
//   level 1  s_h(r) = mid(l, u, y + alpha_h sgn dir) - y
//   level 2  sums <g, s_h>(r-1), <s_h, A s_h>(r-1)
// Stage: y | dir | g (if dir != g) | l | u (if array bounds)
// ============================================================================
template <bool SB, bool DG>
struct SrchLayout4 {
    static constexpr int kY = 0;
    static constexpr int kD = m4::kF;
    static constexpr int kG = DG ? kD : kD + m4::kF;
    static constexpr int kL = kG + m4::kF;
    static constexpr int kU = kL + (SB ? 0 : m4::kF);
    static constexpr int kStage = kU + (SB ? 0 : m4::kF);
    static constexpr int kNST = 4;
    static constexpr int kSmem = kNST * kStage + 64;
};

template <bool SB, bool DG>
__global__ void __launch_bounds__(m4::kThreads, m4::kMinB)
k4_search(StencilOp A, BandGeom G, Bounds Bd, const __grid_constant__ CUtensorMap m_y,
          const __grid_constant__ CUtensorMap m_dir, const __grid_constant__ CUtensorMap m_g,
          const __grid_constant__ CUtensorMap m_l, const __grid_constant__ CUtensorMap m_u, double sgn,
          int use_alpha0, int h0, double mu, Scal* S, RedScratch R, int gp) {
    using namespace m4;
    using L = SrchLayout4<SB, DG>;
    constexpr int K = 2;
    if (gp && *(volatile int*)&S->gp_done) return;   // device-driven GP phase already over
    if (use_alpha0 && !S->cauchy_ok) {           // <d,Ad> <= 0: no step (host reports ENOTSPD)
        if (blockIdx.x == 0 && threadIdx.x == 0) S->s_h = -1;
        return;
    }
    const double base = use_alpha0 ? S->alpha0 : 1.0;
    const double al0 = scalbn(base, -h0), al1 = scalbn(base, -(h0 + 1));
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 28 * wid + lane;
    const bool out_lane = lane >= 2 && lane < 30;
    double acc[2 * K] = {0.0, 0.0, 0.0, 0.0};
    int gx = 0, y0 = 0, y1 = 0;
    bool col_ok = false;
    Op5<true> op;
    double s0_m2 = 0.0, s0_m1 = 0.0, s1_m2 = 0.0, s1_m1 = 0.0, g_m1 = 0.0;
    band_pipeline<L::kNST, L::kStage>(
        G, A.ny, smem,
        [&](unsigned char* st, int x0, int yr, uint64_t* bar) {
            mbar_expect_tx(bar, L::kStage);
            const int yt = yr - G.rlo;
            tma_load_2d(st + L::kY, &m_y, x0 - 2, yt, bar);
            tma_load_2d(st + L::kD, &m_dir, x0 - 2, yt, bar);
            if (!DG) tma_load_2d(st + L::kG, &m_g, x0 - 2, yt, bar);
            if (!SB) {
                tma_load_2d(st + L::kL, &m_l, x0 - 2, yt, bar);
                tma_load_2d(st + L::kU, &m_u, x0 - 2, yt, bar);
            }
        },
        [&](int x0, int yb, int ye) {
            gx = x0 - 2 + c;
            y0 = yb;
            y1 = ye;
            col_ok = gx >= 0 && gx < A.nx;
            op.init(A, gx);
            s0_m2 = s0_m1 = s1_m2 = s1_m1 = g_m1 = 0.0;
        },
        [&](const unsigned char* st, int kk, int r) {
            const int q = kk * kBW + c;
            const bool in = col_ok && r >= A.rlo && r < A.rhi;
            const double yv = reinterpret_cast<const double*>(st + L::kY)[q];
            const double dv = reinterpret_cast<const double*>(st + L::kD)[q];
            const double gv = reinterpret_cast<const double*>(st + L::kG)[q];
            const double lv = in ? (SB ? Bd.lc : reinterpret_cast<const double*>(st + L::kL)[q]) : 0.0;
            const double uv = in ? (SB ? Bd.uc : reinterpret_cast<const double*>(st + L::kU)[q]) : 0.0;
            const double s0 = trial(yv, dv, sgn, al0, lv, uv) - yv;      // 0 outside
            const double s1 = trial(yv, dv, sgn, al1, lv, uv) - yv;
            const double a0 = op.apply(A, r - 1, s0_m1, s0_m2, s0);
            const double a1 = op.apply(A, r - 1, s1_m1, s1_m2, s1);
            const int r1 = r - 1;
            if (out_lane && col_ok && r1 >= y0 && r1 < y1) {
                acc[0] = fma(g_m1, s0_m1, acc[0]);
                acc[1] = fma(s0_m1, a0, acc[1]);
                acc[2] = fma(g_m1, s1_m1, acc[2]);
                acc[3] = fma(s1_m1, a1, acc[3]);
            }
            s0_m2 = s0_m1; s0_m1 = s0;
            s1_m2 = s1_m1; s1_m1 = s1;
            g_m1 = gv;
        });
    reduce_and_finish<2 * K>(acc, R, [&](double* tt) { fin_search(tt, K, h0, base, mu, S); });
}




// ============================================================================
// g-free GP / search sweeps (k5_*).  The gradient g = A y - b is never stored:
// every sweep recomputes it from y at the rows and columns it needs, with the
// arithmetic of the accept sweep that used to store it (op.apply(...) - b, so
// the values are bitwise those of the stored-g kernels).  A GP step then
// streams y (search) and y + masks (accept): 26 instead of 50 B per point.
// The accept sweep of a GP step applies the operator three times (g of y, then
// A yn, then A d), so the warps keep 26 output lanes with 3 halo lanes per
// side; f64 boxes start at the even column x0 - 4 (16-byte aligned): lane L of
// warp w <-> box column 26 w + L + 1 <-> grid column x0 - 3 + 26 w + L.
// MODE: GP (direction -g, base alpha_0), CG (direction w, base 1), PROJ (no
// direction: y_out = P[y]).
// ============================================================================
namespace m5 {
constexpr int kOut = 26 * m4::kWarps;        // output columns per band (208 at 8 warps)
constexpr int kBW = kOut + 8;                // f64 box columns (x0 - 4 .. x0 + kOut + 3): 112 at 4 warps
constexpr int kMW = (kBW + 15 + 31) / 32 * 32;  // u8 mask box width (start floored to 16 B): 128 at 4 warps
constexpr int kBR5 = GPCG_GP_BR;             // rows per pipeline block of the GP-family sweeps
constexpr int kF = kBR5 * kBW * 8;
constexpr int kUt = kBR5 * kMW;
static_assert(kF % 128 == 0 && kUt % 128 == 0, "TMA destinations stay 128-byte aligned");
enum Mode : int { GP = 0, CG = 1, PROJ = 2 };
}  // namespace m5

// Stage: y | w (CG) | b (!BB) | l | u (!SB) | mask_prev
template <bool SB, bool BB, int MODE>
struct AccLayout5 {
    static constexpr int kY = 0;
    static constexpr int kD = m5::kF;
    static constexpr int kB = kD + (MODE == m5::CG ? m5::kF : 0);
    static constexpr int kL = kB + (BB ? 0 : m5::kF);
    static constexpr int kU = kL + (SB ? 0 : m5::kF);
    static constexpr int kMP = kU + (SB ? 0 : m5::kF);
    static constexpr int kStage = kMP + m5::kUt;
    static constexpr int kNST = GPCG_GP_NST;
    static constexpr int kSmem = kNST * kStage + 64;
    static constexpr int kLag = MODE == m5::GP ? 3 : 2;     // emitted row = raw row - kLag
};

// a1 + a2, g-free.  Per raw row r: (GP) g(r-1) = (A y)(r-1) - b, yn(r-1) = P[y - alpha g];
// (CG) yn(r) = P[y + alpha w]; (PROJ) yn(r) = P[y].  With ry the yn row: gn(ry-1) = A yn - b,
// d(ry-1) = grad_Omega q(yn); emit ry-2 with (A d)(ry-2).  y_out, mask_out, the six sums.
template <bool SB, bool BB, int MODE>
__device__ __forceinline__ int accept_sweep5(const StencilOp& A, const BandGeom& G, const Bounds& Bd,
                                             const double* __restrict__ brow, const CUtensorMap* m_y,
                                             const CUtensorMap* m_dir, const CUtensorMap* m_b, const CUtensorMap* m_l,
                                             const CUtensorMap* m_u, const CUtensorMap* m_mp, int has_mp, double alpha,
                                             double* __restrict__ y_out, unsigned char* __restrict__ mask_out,
                                             unsigned char* smem, double (&acc)[6], uint64_t* bars, int k0,
                                             const SlabLink* SL = nullptr, double* lo_y = nullptr,
                                             unsigned char* lo_m = nullptr, double* hi_y = nullptr,
                                             unsigned char* hi_m = nullptr) {
    using namespace m4;
    using L = AccLayout5<SB, BB, MODE>;
    constexpr int LAG = L::kLag;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 26 * wid + lane + 1;            // box column
    const bool out_lane = lane >= 3 && lane < 29;
    int gx = 0, moff = 0, y0 = 0, y1 = 0;
    bool col_ok = false;
    Op5<true> op;
    double bcol = 0.0;
    double y_m1 = 0.0, y_m2 = 0.0, l_r1 = 0.0, u_r1 = 0.0, b_r1 = 0.0;   // GP: raw rows r-1, r-2
    double yn_a = 0.0, yn_b = 0.0;                // yn(ry-1), yn(ry-2)
    double l_a = 0.0, u_a = 0.0, b_a = 0.0;       // bounds / b of row ry-1
    double d_a = 0.0, d_b = 0.0;                  // d(ry-2), d(ry-3)
    double yn_e = 0.0, gn_e = 0.0, l_e = 0.0, u_e = 0.0;   // row ry-2 (emitted)
    const uint32_t tx = L::kMP + (has_mp ? m5::kUt : 0);
    return band_pipeline<L::kNST, L::kStage, m5::kOut, LAG + 1, LAG, m5::kBR5>(
        G, A.ny, smem,
        [&](unsigned char* st, int x0, int yr, uint64_t* bar) {
            mbar_expect_tx(bar, tx);
            const int yt = yr - G.rlo;
            tma_load_2d(st + L::kY, m_y, x0 - 4, yt, bar);
            if (MODE == m5::CG) tma_load_2d(st + L::kD, m_dir, x0 - 4, yt, bar);
            if (!BB) tma_load_2d(st + L::kB, m_b, x0 - 4, yt, bar);
            if (!SB) {
                tma_load_2d(st + L::kL, m_l, x0 - 4, yt, bar);
                tma_load_2d(st + L::kU, m_u, x0 - 4, yt, bar);
            }
            if (has_mp) tma_load_2d(st + L::kMP, m_mp, floor16(x0 - 4), yt - LAG, bar);
        },
        [&](int x0, int yb, int ye) {
            gx = x0 - 3 + 26 * wid + lane;
            moff = (x0 - 4) - floor16(x0 - 4);
            y0 = yb;
            y1 = ye;
            col_ok = gx >= 0 && gx < A.nx;
            op.init(A, gx);
            if (BB) bcol = col_ok ? __ldg(brow + gx) : 0.0;
            y_m1 = y_m2 = l_r1 = u_r1 = b_r1 = yn_a = yn_b = l_a = u_a = b_a = d_a = d_b = 0.0;
            yn_e = gn_e = l_e = u_e = 0.0;
        },
        [&](const unsigned char* st, int kk, int r) {
            const int q = kk * m5::kBW + c;
            const bool rin = r >= A.rlo && r < A.rhi;
            const bool in = col_ok && rin;
            const double yv = reinterpret_cast<const double*>(st + L::kY)[q];
            const double bv = BB ? (rin ? bcol : 0.0) : reinterpret_cast<const double*>(st + L::kB)[q];
            const double lv = in ? (SB ? Bd.lc : reinterpret_cast<const double*>(st + L::kL)[q]) : 0.0;
            const double uv = in ? (SB ? Bd.uc : reinterpret_cast<const double*>(st + L::kU)[q]) : 0.0;
            double yn, ln, un, bn;                // the new iterate and its row data, row ry
            int ry;
            if constexpr (MODE == m5::GP) {
                ry = r - 1;
                const double g1 = op.apply(A, r - 1, y_m1, y_m2, yv) - b_r1;   // g(r-1)
                yn = trial(y_m1, g1, -1.0, alpha, l_r1, u_r1);
                ln = l_r1; un = u_r1; bn = b_r1;
                y_m2 = y_m1; y_m1 = yv;
                l_r1 = lv; u_r1 = uv; b_r1 = bv;
            } else {
                ry = r;
                if constexpr (MODE == m5::CG)
                    yn = trial(yv, reinterpret_cast<const double*>(st + L::kD)[q], 1.0, alpha, lv, uv);
                else
                    yn = mid(lv, uv, yv);
                ln = lv; un = uv; bn = bv;
            }
            const double gn1 = op.apply(A, ry - 1, yn_a, yn_b, yn) - b_a;        // gn(ry-1)
            const double d1 = pgrad(yn_a, gn1, l_a, u_a);                       // d(ry-1)
            const double ad = op.apply(A, ry - 2, d_a, d_b, d1);                // (A d)(ry-2)
            const int re = ry - 2;
            if (out_lane && col_ok && re >= y0 && re < y1) {
                const long long v = (long long)gx + (long long)A.pitch * re;
                y_out[v] = yn_e;
                const bool act = (yn_e == l_e) || (yn_e == u_e);
                const unsigned char m = act ? 0 : 1;
                mask_out[v] = m;
                acc[0] = fma(d_a, d_a, acc[0]);
                acc[1] = fma(gn_e, gn_e, acc[1]);
                acc[2] += act ? 1.0 : 0.0;
                if (has_mp) acc[3] += (st[L::kMP + kk * m5::kMW + c + moff] != m) ? 1.0 : 0.0;
                const bool binding = (yn_e == l_e && gn_e >= 0.0) || (yn_e == u_e && gn_e <= 0.0);
                acc[4] += (act && !binding) ? 1.0 : 0.0;
                acc[5] = fma(d_a, ad, acc[5]);
                if (SL) {                                     // fused halo write (SlabLink)
                    if (re < SL->lo_ghost) {
                        const long long vl = (long long)gx + (long long)A.pitch * (SL->lo_rows + re);
                        lo_y[vl] = yn_e;
                        lo_m[vl] = m;
                    }
                    if (re >= A.ny - SL->hi_ghost) {
                        const long long vh = (long long)gx + (long long)A.pitch * (re - A.ny);
                        hi_y[vh] = yn_e;
                        hi_m[vh] = m;
                    }
                }
            }
            yn_e = yn_a; gn_e = gn1; l_e = l_a; u_e = u_a;
            d_b = d_a; d_a = d1;
            yn_b = yn_a; yn_a = yn;
            l_a = ln; u_a = un; b_a = bn;
        },
        bars, k0, SL ? SL->bid : -1, SL ? SL->nb : -1);
}

template <bool SB, bool BB, int MODE>
__global__ void __launch_bounds__(m4::kThreads, GPCG_GP_MINB)
k5_accept(StencilOp A, BandGeom G, Bounds Bd, const double* __restrict__ brow, const __grid_constant__ CUtensorMap m_y,
          const __grid_constant__ CUtensorMap m_dir, const __grid_constant__ CUtensorMap m_b,
          const __grid_constant__ CUtensorMap m_l, const __grid_constant__ CUtensorMap m_u,
          const __grid_constant__ CUtensorMap m_mp, int has_mp, double* __restrict__ y_out,
          unsigned char* __restrict__ mask_out, Scal* S, RedScratch R, int gp) {
    if (gp && gp_skip(S)) return;      // GP phase over / k5_spec accepted
    double alpha = 0.0;
    if (MODE != m5::PROJ) {
        if (S->s_h < 0) return;                   // uniform: no accepted step in this batch
        alpha = S->s_alpha;
    }
    extern __shared__ __align__(128) unsigned char smem[];
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    accept_sweep5<SB, BB, MODE>(A, G, Bd, brow, &m_y, &m_dir, &m_b, &m_l, &m_u, &m_mp, has_mp, alpha, y_out, mask_out,
                                smem, acc, nullptr, 0);
    reduce_and_finish<6>(acc, R, [&](double* t) { fin_accept(t, true, S); });
}

// a3, g-free: K step sizes.  GP: g(r-1) from y, s_h(r-1) = P[y - alpha_h g] - y; CG: s_h(r) =
// P[y + alpha_h w] - y, g(r-1) from y.  Emit <g, s_h>, <s_h, A s_h> one row behind the s row.
template <bool SB, bool BB, int MODE, int K>
struct SrchLayout5 {
    static constexpr int kY = 0;
    static constexpr int kD = m5::kF;
    static constexpr int kB = kD + (MODE == m5::CG ? m5::kF : 0);
    static constexpr int kL = kB + (BB ? 0 : m5::kF);
    static constexpr int kU = kL + (SB ? 0 : m5::kF);
    static constexpr int kStage = kU + (SB ? 0 : m5::kF);
    static constexpr int kNST = GPCG_GP_NST;
    static constexpr int kSmem = kNST * kStage + 64;
};

template <bool SB, bool BB, int MODE, int K>
__device__ __forceinline__ int search_sweep5(const StencilOp& A, const BandGeom& G, const Bounds& Bd,
                                             const double* __restrict__ brow, const CUtensorMap* m_y,
                                             const CUtensorMap* m_dir, const CUtensorMap* m_b, const CUtensorMap* m_l,
                                             const CUtensorMap* m_u, const double (&al)[K], unsigned char* smem,
                                             double (&acc)[2 * K], uint64_t* bars, int k0,
                                             const SlabLink* SL = nullptr) {
    using namespace m4;
    using L = SrchLayout5<SB, BB, MODE, K>;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 26 * wid + lane + 1;
    const bool out_lane = lane >= 3 && lane < 29;
    int gx = 0, y0 = 0, y1 = 0;
    bool col_ok = false;
    Op5<true> op;
    double bcol = 0.0;
    double y_m1 = 0.0, y_m2 = 0.0, l_r1 = 0.0, u_r1 = 0.0, b_r1 = 0.0;
    double g_e = 0.0;                             // g of the emitted row
    double s_a[K], s_b[K];                        // s_h at the s row - 1, - 2
#pragma unroll
    for (int h = 0; h < K; ++h) { s_a[h] = 0.0; s_b[h] = 0.0; }
    return band_pipeline<L::kNST, L::kStage, m5::kOut, 2, 2, m5::kBR5>(
        G, A.ny, smem,
        [&](unsigned char* st, int x0, int yr, uint64_t* bar) {
            mbar_expect_tx(bar, L::kStage);
            const int yt = yr - G.rlo;
            tma_load_2d(st + L::kY, m_y, x0 - 4, yt, bar);
            if (MODE == m5::CG) tma_load_2d(st + L::kD, m_dir, x0 - 4, yt, bar);
            if (!BB) tma_load_2d(st + L::kB, m_b, x0 - 4, yt, bar);
            if (!SB) {
                tma_load_2d(st + L::kL, m_l, x0 - 4, yt, bar);
                tma_load_2d(st + L::kU, m_u, x0 - 4, yt, bar);
            }
        },
        [&](int x0, int yb, int ye) {
            gx = x0 - 3 + 26 * wid + lane;
            y0 = yb;
            y1 = ye;
            col_ok = gx >= 0 && gx < A.nx;
            op.init(A, gx);
            if (BB) bcol = col_ok ? __ldg(brow + gx) : 0.0;
            y_m1 = y_m2 = l_r1 = u_r1 = b_r1 = g_e = 0.0;
#pragma unroll
            for (int h = 0; h < K; ++h) { s_a[h] = 0.0; s_b[h] = 0.0; }
        },
        [&](const unsigned char* st, int kk, int r) {
            const int q = kk * m5::kBW + c;
            const bool rin = r >= A.rlo && r < A.rhi;
            const bool in = col_ok && rin;
            const double yv = reinterpret_cast<const double*>(st + L::kY)[q];
            const double bv = BB ? (rin ? bcol : 0.0) : reinterpret_cast<const double*>(st + L::kB)[q];
            const double lv = in ? (SB ? Bd.lc : reinterpret_cast<const double*>(st + L::kL)[q]) : 0.0;
            const double uv = in ? (SB ? Bd.uc : reinterpret_cast<const double*>(st + L::kU)[q]) : 0.0;
            const double g1 = op.apply(A, r - 1, y_m1, y_m2, yv) - b_r1;     // g(r-1)
            double sn[K];                         // s_h at the s row rs
            int rs;
            if constexpr (MODE == m5::GP) {
                rs = r - 1;
#pragma unroll
                for (int h = 0; h < K; ++h) sn[h] = trial(y_m1, g1, -1.0, al[h], l_r1, u_r1) - y_m1;
            } else {
                rs = r;
                const double dv = reinterpret_cast<const double*>(st + L::kD)[q];
#pragma unroll
                for (int h = 0; h < K; ++h) sn[h] = trial(yv, dv, 1.0, al[h], lv, uv) - yv;
            }
            // emit row rs-1: <g, s_h>, <s_h, A s_h>;  g(rs-1) is g1 (CG) or the previous g1 (GP)
            const int re = rs - 1;
            const double ge = (MODE == m5::GP) ? g_e : g1;
            const bool emit = out_lane && col_ok && re >= y0 && re < y1;
#pragma unroll
            for (int h = 0; h < K; ++h) {
                const double as = op.apply(A, re, s_a[h], s_b[h], sn[h]);
                if (emit) {
                    acc[2 * h] = fma(ge, s_a[h], acc[2 * h]);
                    acc[2 * h + 1] = fma(s_a[h], as, acc[2 * h + 1]);
                }
            }
#pragma unroll
            for (int h = 0; h < K; ++h) { s_b[h] = s_a[h]; s_a[h] = sn[h]; }
            g_e = g1;
            y_m2 = y_m1; y_m1 = yv;
            l_r1 = lv; u_r1 = uv; b_r1 = bv;
        },
        bars, k0, SL ? SL->bid : -1, SL ? SL->nb : -1);
}

template <bool SB, bool BB, int MODE, int K>
__global__ void __launch_bounds__(m4::kThreads, (K <= 2 ? GPCG_GP_MINB : (m4::kMinB > 1 ? m4::kMinB / 2 : 1)))
k5_search(StencilOp A, BandGeom G, Bounds Bd, const double* __restrict__ brow, const __grid_constant__ CUtensorMap m_y,
          const __grid_constant__ CUtensorMap m_dir, const __grid_constant__ CUtensorMap m_b,
          const __grid_constant__ CUtensorMap m_l, const __grid_constant__ CUtensorMap m_u, int h0, double mu,
          Scal* S, RedScratch R, int gp) {
    constexpr bool use_alpha0 = MODE == m5::GP;
    if (gp && gp_skip(S)) return;      // GP phase over / k5_spec accepted
    if (use_alpha0 && !S->cauchy_ok) {           // <d,Ad> <= 0: no step (host reports ENOTSPD)
        if (blockIdx.x == 0 && threadIdx.x == 0) S->s_h = -1;
        return;
    }
    const double base = use_alpha0 ? S->alpha0 : 1.0;
    double al[K];
#pragma unroll
    for (int h = 0; h < K; ++h) al[h] = scalbn(base, -(h0 + h));
    extern __shared__ __align__(128) unsigned char smem[];
    double acc[2 * K];
#pragma unroll
    for (int s = 0; s < 2 * K; ++s) acc[s] = 0.0;
    search_sweep5<SB, BB, MODE, K>(A, G, Bd, brow, &m_y, &m_dir, &m_b, &m_l, &m_u, al, smem, acc, nullptr, 0);
    reduce_and_finish<2 * K>(acc, R, [&](double* tt) { fin_search(tt, K, h0, base, mu, S); });
}

// a5 init, g-free: rho_0 = -[v in F] (A y - b)_v, u_0 = rho_0 (/ A_vv with PC); q_0 = A_F u_0;
// gamma_0 = rho_0'u_0, delta_0 = u_0'q_0.  Writes rho, p = 0, w = 0 and the CG mask copy.
// Stage: y | b (!BB) | mask
template <bool BB>
struct CgInitLayout5 {
    static constexpr int kY = 0;
    static constexpr int kB = m5::kF;
    static constexpr int kM = kB + (BB ? 0 : m5::kF);
    static constexpr int kStage = kM + m5::kUt;
    static constexpr int kNST = 4;
    static constexpr int kSmem = kNST * kStage + 64;
};

template <bool BB, bool PC>
__global__ void __launch_bounds__(m4::kThreads, m4::kMinB)
k5_cg_init(StencilOp A, BandGeom G, const double* __restrict__ brow, const __grid_constant__ CUtensorMap m_y,
           const __grid_constant__ CUtensorMap m_b, const __grid_constant__ CUtensorMap m_mask,
           unsigned char* __restrict__ mask_cg, double* __restrict__ rho, double* __restrict__ p,
           double* __restrict__ w, double eta2, long long cap, Scal* S, RedScratch R) {
    using namespace m4;
    using L = CgInitLayout5<BB>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 26 * wid + lane + 1;
    const bool out_lane = lane >= 3 && lane < 29;
    double acc[2] = {0.0, 0.0};
    int gx = 0, moff = 0, y0 = 0, y1 = 0;
    bool col_ok = false;
    Op5<true> op;
    double bcol = 0.0, dinv = 0.0;
    double y_m1 = 0.0, y_m2 = 0.0, b_r1 = 0.0;
    unsigned char m_r1 = 0, m_a = 0;
    double u_a = 0.0, u_b = 0.0, rho_a = 0.0;     // u at rows r-2, r-3; rho at r-2
    const uint32_t tx = L::kM + m5::kUt;
    band_pipeline<L::kNST, L::kStage, m5::kOut, 2, 2, m5::kBR5>(
        G, A.ny, smem,
        [&](unsigned char* st, int x0, int yr, uint64_t* bar) {
            mbar_expect_tx(bar, tx);
            const int yt = yr - G.rlo;
            tma_load_2d(st + L::kY, &m_y, x0 - 4, yt, bar);
            if (!BB) tma_load_2d(st + L::kB, &m_b, x0 - 4, yt, bar);
            tma_load_2d(st + L::kM, &m_mask, floor16(x0 - 4), yt, bar);
        },
        [&](int x0, int yb, int ye) {
            gx = x0 - 3 + 26 * wid + lane;
            moff = (x0 - 4) - floor16(x0 - 4);
            y0 = yb;
            y1 = ye;
            col_ok = gx >= 0 && gx < A.nx;
            op.init(A, gx);
            dinv = op.dinv(A, 0);
            if (BB) bcol = col_ok ? __ldg(brow + gx) : 0.0;
            y_m1 = y_m2 = b_r1 = u_a = u_b = rho_a = 0.0;
            m_r1 = m_a = 0;
        },
        [&](const unsigned char* st, int kk, int r) {
            const int q = kk * m5::kBW + c;
            const bool rin = r >= A.rlo && r < A.rhi;
            const double yv = reinterpret_cast<const double*>(st + L::kY)[q];
            const double bv = BB ? (rin ? bcol : 0.0) : reinterpret_cast<const double*>(st + L::kB)[q];
            const unsigned char mv = st[L::kM + kk * m5::kMW + c + moff];
            const double g1 = op.apply(A, r - 1, y_m1, y_m2, yv) - b_r1;     // g(r-1)
            const double rho1 = m_r1 ? -g1 : 0.0;                            // rho_0(r-1)
            const double u1 = PC ? rho1 * dinv : rho1;
            const double qv = op.apply(A, r - 2, u_a, u_b, u1);              // (A_F u_0)(r-2) on F
            const int re = r - 2;
            if (out_lane && col_ok && re >= y0 && re < y1) {
                const long long v = (long long)gx + (long long)A.pitch * re;
                mask_cg[v] = m_a;
                rho[v] = rho_a;
                p[v] = 0.0;
                w[v] = 0.0;
                acc[0] = fma(rho_a, u_a, acc[0]);
                acc[1] = m_a ? fma(u_a, qv, acc[1]) : acc[1];
            }
            u_b = u_a; u_a = u1; rho_a = rho1; m_a = m_r1;
            y_m2 = y_m1; y_m1 = yv; b_r1 = bv; m_r1 = mv;
        });
    reduce_and_finish<2>(acc, R, [&](double* t) { cg_init_finalize(t[0], t[1], eta2, cap, S); });
}


// Speculative GP step (used by k6_gp_loop): the accept sweep of the GP mode at the first
// step size alpha_0, which also accumulates the h = 0 search sums <g, s> and <s, A s>
// (s = yn - y, A s applied to s exactly as search_sweep5 does).  If Eq. gplsstop accepts
// h = 0 -- the common case -- the step costs one sweep instead of two; otherwise the caller
// discards y_out / mask_out and runs search (h >= 1) + accept.  acc: the six accept sums,
// then <g, s>, <s, A s>.
template <bool SB, bool BB>
__device__ __forceinline__ int spec_sweep5(const StencilOp& A, const BandGeom& G, const Bounds& Bd,
                                           const double* __restrict__ brow, const CUtensorMap* m_y,
                                           const CUtensorMap* m_b, const CUtensorMap* m_l, const CUtensorMap* m_u,
                                           const CUtensorMap* m_mp, double alpha, double* __restrict__ y_out,
                                           unsigned char* __restrict__ mask_out, unsigned char* smem,
                                           double (&acc)[8], uint64_t* bars, int k0) {
    using namespace m4;
    using L = AccLayout5<SB, BB, m5::GP>;
    constexpr int LAG = L::kLag;                  // 3: emitted row = raw row - 3
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 26 * wid + lane + 1;
    const bool out_lane = lane >= 3 && lane < 29;
    int gx = 0, moff = 0, y0 = 0, y1 = 0;
    bool col_ok = false;
    Op5<true> op;
    double bcol = 0.0;
    double y_m1 = 0.0, y_m2 = 0.0, l_r1 = 0.0, u_r1 = 0.0, b_r1 = 0.0;
    double yn_a = 0.0, yn_b = 0.0, l_a = 0.0, u_a = 0.0, b_a = 0.0, d_a = 0.0, d_b = 0.0;
    double yn_e = 0.0, gn_e = 0.0, l_e = 0.0, u_e = 0.0;
    double s_a = 0.0, s_b = 0.0;                  // s(r-2), s(r-3)
    double g_a = 0.0, g_b = 0.0;                  // g(r-2), g(r-3)
    double as_p = 0.0;                            // (A s)(r-3), from the previous row step
    const uint32_t tx = L::kMP + m5::kUt;
    return band_pipeline<L::kNST, L::kStage, m5::kOut, LAG + 1, LAG, m5::kBR5>(
        G, A.ny, smem,
        [&](unsigned char* st, int x0, int yr, uint64_t* bar) {
            mbar_expect_tx(bar, tx);
            const int yt = yr - G.rlo;
            tma_load_2d(st + L::kY, m_y, x0 - 4, yt, bar);
            if (!BB) tma_load_2d(st + L::kB, m_b, x0 - 4, yt, bar);
            if (!SB) {
                tma_load_2d(st + L::kL, m_l, x0 - 4, yt, bar);
                tma_load_2d(st + L::kU, m_u, x0 - 4, yt, bar);
            }
            tma_load_2d(st + L::kMP, m_mp, floor16(x0 - 4), yt - LAG, bar);
        },
        [&](int x0, int yb, int ye) {
            gx = x0 - 3 + 26 * wid + lane;
            moff = (x0 - 4) - floor16(x0 - 4);
            y0 = yb;
            y1 = ye;
            col_ok = gx >= 0 && gx < A.nx;
            op.init(A, gx);
            if (BB) bcol = col_ok ? __ldg(brow + gx) : 0.0;
            y_m1 = y_m2 = l_r1 = u_r1 = b_r1 = yn_a = yn_b = l_a = u_a = b_a = d_a = d_b = 0.0;
            yn_e = gn_e = l_e = u_e = s_a = s_b = g_a = g_b = as_p = 0.0;
        },
        [&](const unsigned char* st, int kk, int r) {
            const int q = kk * m5::kBW + c;
            const bool rin = r >= A.rlo && r < A.rhi;
            const bool in = col_ok && rin;
            const double yv = reinterpret_cast<const double*>(st + L::kY)[q];
            const double bv = BB ? (rin ? bcol : 0.0) : reinterpret_cast<const double*>(st + L::kB)[q];
            const double lv = in ? (SB ? Bd.lc : reinterpret_cast<const double*>(st + L::kL)[q]) : 0.0;
            const double uv = in ? (SB ? Bd.uc : reinterpret_cast<const double*>(st + L::kU)[q]) : 0.0;
            const double g1 = op.apply(A, r - 1, y_m1, y_m2, yv) - b_r1;     // g(r-1)
            const double yn = trial(y_m1, g1, -1.0, alpha, l_r1, u_r1);      // yn(r-1)
            const double s1 = yn - y_m1;                                      // s(r-1)
            const double as2 = op.apply(A, r - 2, s_a, s_b, s1);              // (A s)(r-2)
            const double gn1 = op.apply(A, r - 2, yn_a, yn_b, yn) - b_a;      // gn(r-2)
            const double d1 = pgrad(yn_a, gn1, l_a, u_a);                     // d(r-2)
            const double ad = op.apply(A, r - 3, d_a, d_b, d1);               // (A d)(r-3)
            const int re = r - 3;
            if (out_lane && col_ok && re >= y0 && re < y1) {
                const long long v = (long long)gx + (long long)A.pitch * re;
                y_out[v] = yn_e;
                const bool act = (yn_e == l_e) || (yn_e == u_e);
                const unsigned char m = act ? 0 : 1;
                mask_out[v] = m;
                acc[0] = fma(d_a, d_a, acc[0]);
                acc[1] = fma(gn_e, gn_e, acc[1]);
                acc[2] += act ? 1.0 : 0.0;
                acc[3] += (st[L::kMP + kk * m5::kMW + c + moff] != m) ? 1.0 : 0.0;
                const bool binding = (yn_e == l_e && gn_e >= 0.0) || (yn_e == u_e && gn_e <= 0.0);
                acc[4] += (act && !binding) ? 1.0 : 0.0;
                acc[5] = fma(d_a, ad, acc[5]);
                acc[6] = fma(g_b, s_b, acc[6]);                               // <g, s>(r-3)
                acc[7] = fma(s_b, as_p, acc[7]);                              // <s, A s>(r-3)
            }
            yn_e = yn_a; gn_e = gn1; l_e = l_a; u_e = u_a;
            d_b = d_a; d_a = d1;
            yn_b = yn_a; yn_a = yn;
            l_a = l_r1; u_a = u_r1; b_a = b_r1;
            s_b = s_a; s_a = s1;
            g_b = g_a; g_a = g1;
            as_p = as2;
            y_m2 = y_m1; y_m1 = yv;
            l_r1 = lv; u_r1 = uv; b_r1 = bv;
        },
        bars, k0);
}

// The speculative GP step with one operator application less and a 2-row lag (default;
// GPCG_GP_SPEC6=0 selects spec_sweep5 above).  Same sums, evaluated as
//   g(r-1)  = (A y)(r-1) - b,   yn(r-1) = P[y - alpha_0 g],   s(r-1) = yn - y
//   As(r-2) = (A s)(r-2),       gn(r-2) = g(r-2) + As(r-2)       (A yn - b = A y - b + A s)
//   d(r-2)  = grad_Omega q(yn)(r-2)
//   <d, A d> as its face form  sum_faces w_f (d_a - d_b)^2  (+ w_f d^2 on boundary faces;
//            A = sum_f w_f (e_a - e_b)(e_a - e_b)' + boundary terms, BASELINE configs[0]):
//            each point adds its west and south faces, the last column / row its east /
//            north boundary face, so only the west neighbour (shuffle) and the row below
//            (register) are needed -- no A d, no third row of lag.
// gn and <d, A d> differ from spec_sweep5's only in rounding (one add instead of a fresh
// stencil application; a sum of squares instead of d'(A d)); the iterate yn is the same.
template <bool SB, bool BB>
__device__ __forceinline__ int spec_sweep6(const StencilOp& A, const BandGeom& G, const Bounds& Bd,
                                           const double* __restrict__ brow, const CUtensorMap* m_y,
                                           const CUtensorMap* m_b, const CUtensorMap* m_l, const CUtensorMap* m_u,
                                           const CUtensorMap* m_mp, double alpha, double* __restrict__ y_out,
                                           unsigned char* __restrict__ mask_out, unsigned char* smem,
                                           double (&acc)[8], uint64_t* bars, int k0, const SlabLink* SL = nullptr,
                                           double* lo_y = nullptr, unsigned char* lo_m = nullptr,
                                           double* hi_y = nullptr, unsigned char* hi_m = nullptr) {
    using namespace m4;
    using L = AccLayout5<SB, BB, m5::GP>;
    constexpr int LAG = 2;                        // emitted row = raw row - 2
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 26 * wid + lane + 1;
    const bool out_lane = lane >= 3 && lane < 29;
    int gx = 0, moff = 0, y0 = 0, y1 = 0;
    bool col_ok = false;
    Op5<true> op;
    double bcol = 0.0, fe_bd = 0.0, fen_bd = 0.0; // b of the column; east boundary face weight (last
                                                  // column), + the north one (last grid row)
    int r_last = 0;                               // raw row whose emitted row is the last grid row
    bool bnd_warp = false;                        // this warp holds the last grid column
    double* yrow = nullptr;                       // y_out / mask_out at (gx, emitted row), advanced per row
    unsigned char* mrow = nullptr;
    int n_act = 0, n_chg = 0, n_nb = 0;           // the three set counts, as integers (exact)
    double y_m1 = 0.0, y_m2 = 0.0, l_r1 = 0.0, u_r1 = 0.0, b_r1 = 0.0;   // raw rows r-1, r-2
    double g_a = 0.0, yn_a = 0.0, l_a = 0.0, u_a = 0.0;                 // row r-2
    double s_a = 0.0, s_b = 0.0;                                        // s(r-2), s(r-3)
    double d_b = 0.0;                                                   // d(r-3)
    // mask_prev is not loaded: the previous free mask is !(y == l || y == u) of the row's y itself
    // (every mask is written from the same comparison of the iterate it belongs to)
    const uint32_t tx = L::kMP;
    const int k = band_pipeline<L::kNST, L::kStage, m5::kOut, LAG + 1, LAG, m5::kBR5>(
        G, A.ny, smem,
        [&](unsigned char* st, int x0, int yr, uint64_t* bar) {
            mbar_expect_tx(bar, tx);
            const int yt = yr - G.rlo;
            tma_load_2d(st + L::kY, m_y, x0 - 4, yt, bar);
            if (!BB) tma_load_2d(st + L::kB, m_b, x0 - 4, yt, bar);
            if (!SB) {
                tma_load_2d(st + L::kL, m_l, x0 - 4, yt, bar);
                tma_load_2d(st + L::kU, m_u, x0 - 4, yt, bar);
            }
        },
        [&](int x0, int yb, int ye) {
            gx = x0 - 3 + 26 * wid + lane;
            moff = (x0 - 4) - floor16(x0 - 4);
            y0 = yb;
            y1 = ye;
            col_ok = gx >= 0 && gx < A.nx;
            op.init(A, gx);
            fe_bd = gx == A.nx - 1 ? op.fe : 0.0;
            fen_bd = fe_bd + op.fn;
            bnd_warp = __any_sync(0xffffffffu, gx == A.nx - 1);
            r_last = A.rhi + 1;
            if (BB) bcol = col_ok ? __ldg(brow + gx) : 0.0;
            {
                const long long v = (long long)gx + (long long)A.pitch * (yb - (LAG + 1) - LAG);
                yrow = y_out + v;                 // (rows before the item: never dereferenced)
                mrow = mask_out + v;
            }
            y_m1 = y_m2 = l_r1 = u_r1 = b_r1 = g_a = yn_a = l_a = u_a = s_a = s_b = d_b = 0.0;
        },
        [&](const unsigned char* st, int kk, int r) {
            const int q = kk * m5::kBW + c;
            const bool in = col_ok && r >= A.rlo && r < A.rhi;
            const double yv = reinterpret_cast<const double*>(st + L::kY)[q];
            // b is not masked outside the grid rows: there y = l = u = 0, so yn = s = d = 0 whatever g is;
            // array bounds need no mask either: the TMA unit zero-fills everything outside the tensor
            const double bv = BB ? bcol : reinterpret_cast<const double*>(st + L::kB)[q];
            const double lv = SB ? (in ? Bd.lc : 0.0) : reinterpret_cast<const double*>(st + L::kL)[q];
            const double uv = SB ? (in ? Bd.uc : 0.0) : reinterpret_cast<const double*>(st + L::kU)[q];
            const double g1 = op.apply(A, r - 1, y_m1, y_m2, yv) - b_r1;     // g(r-1)
            const double yn1 = trial(y_m1, g1, -1.0, alpha, l_r1, u_r1);     // yn(r-1)
            const double s1 = yn1 - y_m1;                                     // s(r-1)
            const double as2 = op.apply(A, r - 2, s_a, s_b, s1);              // (A s)(r-2)
            const double gn2 = g_a + as2;                                     // gn(r-2)
            // d(r-2) = pgrad(yn, gn, l, u) (common.cuh) written out, so that its bound tests and
            // its zero flag serve the mask, the active count and the binding test below as well
            const bool al = yn_a == l_a, au = yn_a == u_a;
            const bool zero = (al && !(gn2 < 0.0)) || (au && !(gn2 > 0.0));   // pgrad's zero case
            const double d2 = zero ? 0.0 : gn2;                               // d(r-2)
            const double dw = __shfl_up_sync(0xffffffffu, d2, 1);             // d(r-2) one column west
            const int re = r - 2;
            double* const yp = yrow;
            unsigned char* const mp = mrow;
            yrow += A.pitch;
            mrow += A.pitch;
            if (out_lane && col_ok && re >= y0 && re < y1) {
                *yp = yn_a;
                const bool act = al || au;
                const unsigned char m = act ? 0 : 1;
                *mp = m;
                // face form of <d, A d>: west and south faces, + the boundary faces of the last
                // column / row (coefficient fe_bd, and fn on the last grid row)
                const double ew = d2 - dw, es = d2 - d_b;
                acc[5] = fma(op.fw * ew, ew, acc[5]);                        // <d, A d>, west face
                acc[5] = fma(op.fs * es, es, acc[5]);                        // ... south face
                if (bnd_warp || r == r_last) {                // (warp-uniform) boundary faces
                    const double kb = r == r_last ? fen_bd : fe_bd;
                    acc[5] = fma(kb * d2, d2, acc[5]);
                }
                acc[0] = fma(d2, d2, acc[0]);
                // acc[1] (||g||^2 of the new point) is not formed: no GP-phase decision reads it
                // (the solve's ||g(x0)|| comes from the initial projection)
                n_act += act ? 1 : 0;
                const bool act_prev = (y_m2 == l_a) || (y_m2 == u_a);     // y(r-2) before the step
                n_chg += (act_prev != act) ? 1 : 0;
                // binding: (al && gn >= 0) || (au && gn <= 0) -- pgrad's zero case (finite gn)
                n_nb += (act && !zero) ? 1 : 0;
                acc[6] = fma(g_a, s_a, acc[6]);                               // <g, s>(r-2)
                acc[7] = fma(s_a, as2, acc[7]);                               // <s, A s>(r-2)
                if (SL) {                                     // fused halo write (SlabLink)
                    if (re < SL->lo_ghost) {
                        const long long vl = (long long)gx + (long long)A.pitch * (SL->lo_rows + re);
                        lo_y[vl] = yn_a;
                        lo_m[vl] = m;
                    }
                    if (re >= A.ny - SL->hi_ghost) {
                        const long long vh = (long long)gx + (long long)A.pitch * (re - A.ny);
                        hi_y[vh] = yn_a;
                        hi_m[vh] = m;
                    }
                }
            }
            d_b = d2;
            s_b = s_a; s_a = s1;
            g_a = g1; yn_a = yn1; l_a = l_r1; u_a = u_r1;
            y_m2 = y_m1; y_m1 = yv;
            l_r1 = lv; u_r1 = uv; b_r1 = bv;
        },
        bars, k0, SL ? SL->bid : -1, SL ? SL->nb : -1);
    acc[2] += (double)n_act;
    acc[3] += (double)n_chg;
    acc[4] += (double)n_nb;
    return k;
}

#ifndef GPCG_GP_SPEC6
#define GPCG_GP_SPEC6 1
#endif

// ============================================================================
// a1-a3 + a7: the whole GP phase as ONE persistent cooperative launch
// (single slab, single rank, g-free sweeps).  Per GP step: search sweep (K = 2) ->
// grid barrier -> every CTA sums the block partials in the same fixed order and takes
// the Eq. gplsstop decision -> accept sweep -> grid barrier -> fin_accept sums ->
// k_gp_step's stop rules (pgstop1, pgstop2, cap, convergence).  A first batch without
// an acceptable step (or <d,Ad> <= 0) hands the step back to the host (GP_HOST), as the
// graph path does.  y, mask ping-pong between buffers 0 / 1 starting from cur0.
// ============================================================================
#ifdef GPCG_DIAG_TIMES
// diagnostic builds only (scripts/gp_step_times.py): per (GP step of the last launch, CTA)
// globaltimer stamps -- step start, sweep done (after the block reduction), grid barrier
// passed, sums formed -- and the CTA's SM
constexpr int kDiagSteps = 64, kDiagCtas = 512;
__device__ unsigned long long g_diag_t[kDiagSteps][kDiagCtas][5];
__device__ int g_diag_step[kDiagCtas];            // each CTA's step of the running launch
__device__ __forceinline__ void diag_stamp(int slot) {
    if (threadIdx.x != 0 || blockIdx.x >= kDiagCtas) return;
    const int st = g_diag_step[blockIdx.x];
    if (st >= kDiagSteps) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_diag_t[st][blockIdx.x][slot] = t;
    if (slot == 0) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_diag_t[st][blockIdx.x][4] = smid;
    }
}
#else
__device__ __forceinline__ void diag_stamp(int) {}
#endif

template <int NS>
__device__ __forceinline__ void grid_sum(double (&acc)[NS], double* part, unsigned int G_, unsigned int* gbar,
                                         unsigned int& gen, double* red, double* tot) {
    block_reduce<NS>(acc, red);
    diag_stamp(1);
    if (threadIdx.x == 0)
        for (int q = 0; q < NS; ++q) part[q * G_ + blockIdx.x] = acc[q];
    grid_barrier(gbar, G_, gen);
    diag_stamp(2);
    double t[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) t[q] = 0.0;
    for (unsigned int b = threadIdx.x; b < G_; b += blockDim.x)
#pragma unroll
        for (int q = 0; q < NS; ++q) t[q] += __ldcg(part + q * G_ + b);
    block_reduce<NS>(t, red);
    if (threadIdx.x == 0)
        for (int q = 0; q < NS; ++q) tot[q] = t[q];
    __syncthreads();
    diag_stamp(3);
}

// The GP phase loop shared by the single- and multi-slab persistent kernels.  spec(cur, alpha_0,
// acc8, k), search(cur, al, acc4, k), accept(cur, alpha, acc6, k) run one sweep of this CTA's
// items from the y / mask buffers `cur` and return the CTA's running TMA block count.
template <bool XR = false, class Spec, class Search, class Accept>
__device__ __forceinline__ void gp_loop(int cur0, double mu, Scal* S, double* __restrict__ part, unsigned int* gbar,
                                        int spec, Spec&& spec_fn, Search&& search_fn, Accept&& accept_fn,
                                        const XRank* X = nullptr) {
    __shared__ double red[8 * 32];
    __shared__ double tot[8];
    if (S->gp_done) return;
    const double tau = S->gp_tau, eta1 = S->gp_eta1;
    const long long gp_cap = S->gp_cap;
    long long j = S->gp_j;
    double maxdec = S->gp_maxdec, last_dec = S->gp_last_dec;
    double alpha0 = S->alpha0;
    int cauchy_ok = S->cauchy_ok;
    double pg2 = S->pg2, g2 = S->g2, n_active = S->n_active, n_changed = S->n_changed, n_nb = S->n_nonbinding;
    double dd = S->dd, dAd = S->dAd;
    int s_h = S->s_h;
    double s_alpha = S->s_alpha, s_delta = S->s_delta, s_gs = S->s_gs;
    int done = 0, reason = GP_RUNNING;
    int s_spec = 0;                               // GP_HOST: the first step size index still to try
    int nfb = 0;                                  // rejected speculative sweeps (diagnostic)
    const unsigned int G_ = gridDim.x;
    unsigned int gen = 0;
    int k = 0, red_i = 0;
    int cur = cur0;
    __shared__ XCtx xc;                           // in shared memory: no registers held across the sweeps
    if constexpr (XR) {
        if (threadIdx.x == 0) xc = xr_ctx(*X);
        __syncthreads();
        if (X->sys) xr_barrier(*X, xc, gen);      // ranks: no fused store before every peer left its last kernel
    }
    // one reduction: the one-device grid sum, or the cross-rank one
    auto gsum = [&](auto& acc) {
        constexpr int NS = (int)(sizeof(acc) / sizeof(double));
        if constexpr (XR) xr_grid_sum<NS>(acc, *X, xc, gen, red, tot);
        else grid_sum<NS>(acc, part + (red_i & 1) * 8 * G_, G_, gbar, gen, red, tot);
        ++red_i;
    };
    while (!done) {
        if (!cauchy_ok) { s_h = -1; done = 1; reason = GP_HOST; break; }
        bool have_accept = false;
#ifdef GPCG_DIAG_TIMES
        if (threadIdx.x == 0 && blockIdx.x < kDiagCtas) g_diag_step[blockIdx.x] = (int)(j - S->gp_j);
        diag_stamp(0);
#endif
        if (spec) {
            // speculative accept at alpha_0 with the h = 0 search sums (one sweep when accepted)
            double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            k = spec_fn(cur, alpha0, acc, k);
            gsum(acc);
            const double gs = tot[6], sAs = tot[7];
            const double dq = gs + 0.5 * sAs;
            if (dq <= mu * gs) {                         // Eq. gplsstop at h = 0
                s_h = 0; s_alpha = alpha0; s_delta = dq; s_gs = gs;
                have_accept = true;
            }
        }
        if (!have_accept) {
            nfb += spec ? 1 : 0;
            // ---- search, alpha_h = alpha_0 2^-h for the next two h
            const int h0 = spec ? 1 : 0;
            const double al[2] = {scalbn(alpha0, -h0), scalbn(alpha0, -(h0 + 1))};
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            k = search_fn(cur, al, acc, k);
            gsum(acc);
            s_h = -1;
            for (int h = 0; h < 2; ++h) {
                const double gs = tot[2 * h], sAs = tot[2 * h + 1];
                const double dq = gs + 0.5 * sAs;
                if (dq <= mu * gs) {
                    s_h = h0 + h;
                    s_alpha = al[h];
                    s_delta = dq;
                    s_gs = gs;
                    break;
                }
            }
            if (s_h < 0) { s_h = -1; s_spec = h0 + 2; done = 1; reason = GP_HOST; break; }
            // ---- accept y' = P[y - s_alpha g], regrad sums, free mask, next Cauchy form
            double acc6[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            k = accept_fn(cur, s_alpha, acc6, k);
            gsum(acc6);
        }
        pg2 = tot[0]; g2 = tot[1]; n_active = tot[2]; n_changed = tot[3]; n_nb = tot[4];
        dd = tot[0]; dAd = tot[5];
        cauchy_ok = (tot[5] > 0.0) ? 1 : 0;
        alpha0 = (tot[5] > 0.0) ? tot[0] / tot[5] : 0.0;
        cur ^= 1;
        // ---- k_gp_step
        ++j;
        const double dec = -s_delta;
        last_dec = dec;
        const bool stop = (n_changed == 0.0) || (j >= 2 && dec <= eta1 * maxdec) || (j >= gp_cap);
        if (dec > maxdec) maxdec = dec;
        if (stop) { done = 1; reason = GP_STOP; }
        else if (sqrt(pg2) <= tau) { done = 1; reason = GP_CONV; }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        S->pg2 = pg2; S->g2 = g2; S->n_active = n_active; S->n_changed = n_changed; S->n_nonbinding = n_nb;
        S->dd = dd; S->dAd = dAd; S->cauchy_ok = cauchy_ok; S->alpha0 = alpha0;
        S->s_h = s_h; S->s_alpha = s_alpha; S->s_delta = s_delta; S->s_gs = s_gs;
        S->gp_j = j; S->gp_maxdec = maxdec; S->gp_last_dec = last_dec;
        S->gp_done = done; S->gp_reason = reason;
        S->s_pad = s_spec;                         // GP_HOST after a search: resume the search at h = s_spec
        S->gp_fb = nfb;
    }
    if constexpr (XR) xr_close(*X, xc, gen);
}

template <bool SB, bool BB>
__global__ void __launch_bounds__(m4::kThreads, GPCG_GP_MINB)
k6_gp_loop(StencilOp A, BandGeom Gs, BandGeom Ga, Bounds Bd, const double* __restrict__ brow,
           const __grid_constant__ CUtensorMap m_y0, const __grid_constant__ CUtensorMap m_y1,
           const __grid_constant__ CUtensorMap m_b, const __grid_constant__ CUtensorMap m_l,
           const __grid_constant__ CUtensorMap m_u, const __grid_constant__ CUtensorMap m_m0,
           const __grid_constant__ CUtensorMap m_m1, double* __restrict__ y0p, double* __restrict__ y1p,
           unsigned char* __restrict__ mk0, unsigned char* __restrict__ mk1, int cur0, double mu, Scal* S,
           double* __restrict__ part, unsigned int* gbar, int spec) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[4];
    gp_loop(
        cur0, mu, S, part, gbar, spec,
        [&](int cur, double alpha0, double (&acc)[8], int k) {
            if (GPCG_GP_SPEC6)
                return spec_sweep6<SB, BB>(A, Ga, Bd, brow, cur ? &m_y1 : &m_y0, &m_b, &m_l, &m_u,
                                           cur ? &m_m1 : &m_m0, alpha0, cur ? y0p : y1p, cur ? mk0 : mk1, smem, acc,
                                           bars, k);
            return spec_sweep5<SB, BB>(A, Ga, Bd, brow, cur ? &m_y1 : &m_y0, &m_b, &m_l, &m_u, cur ? &m_m1 : &m_m0,
                                       alpha0, cur ? y0p : y1p, cur ? mk0 : mk1, smem, acc, bars, k);
        },
        [&](int cur, const double (&al)[2], double (&acc)[4], int k) {
            return search_sweep5<SB, BB, m5::GP, 2>(A, Gs, Bd, brow, cur ? &m_y1 : &m_y0, cur ? &m_y1 : &m_y0, &m_b,
                                                    &m_l, &m_u, al, smem, acc, bars, k);
        },
        [&](int cur, double alpha, double (&acc)[6], int k) {
            return accept_sweep5<SB, BB, m5::GP>(A, Ga, Bd, brow, cur ? &m_y1 : &m_y0, cur ? &m_y1 : &m_y0, &m_b,
                                                 &m_l, &m_u, cur ? &m_m1 : &m_m0, 1, alpha, cur ? y0p : y1p,
                                                 cur ? mk0 : mk1, smem, acc, bars, k);
        });
}

// The speculative GP step as ONE graph node (the GP graph chunks of slabs / ranks, which cannot
// run the persistent loop): spec_sweep6 at alpha_0 from y(cur) into y(nxt), mask(nxt) -- the
// accepted point, its set counts and next Cauchy form, and the h = 0 search sums, the same sweep
// and sums as k6_gp_loop's -- then fin_spec6: Eq. gplsstop at h = 0 keeps the step (the step's
// search / accept nodes return at once) or lets them run from h = 1.
template <bool SB, bool BB>
__global__ void __launch_bounds__(m4::kThreads, GPCG_GP_MINB)
k5_spec(StencilOp A, BandGeom G, Bounds Bd, const double* __restrict__ brow, const __grid_constant__ CUtensorMap m_y,
        const __grid_constant__ CUtensorMap m_b, const __grid_constant__ CUtensorMap m_l,
        const __grid_constant__ CUtensorMap m_u, const __grid_constant__ CUtensorMap m_m,
        double* __restrict__ y_out, unsigned char* __restrict__ mask_out, double mu, Scal* S, RedScratch R) {
    if (*(volatile int*)&S->gp_done) return;
    if (!S->cauchy_ok) {                          // <d,Ad> <= 0: no step (uniform; k_finalize mirrors it)
        if (blockIdx.x == 0 && threadIdx.x == 0) { S->spec_ok = 0; S->s_h = -1; }
        return;
    }
    const double alpha0 = S->alpha0;
    extern __shared__ __align__(128) unsigned char smem[];
    double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    spec_sweep6<SB, BB>(A, G, Bd, brow, &m_y, &m_b, &m_l, &m_u, &m_m, alpha0, y_out, mask_out, smem, acc, nullptr, 0);
    reduce_and_finish<8>(acc, R, [&](double* t) { fin_spec6(t, mu, S); });
}

// k6_gp_loop over several slabs of one device (SlabLink): the accepted y and the new mask of
// every row a neighbour keeps as a ghost row also go straight into its ghost rows.
struct GpMsSlab {
    CUtensorMap m_y0, m_y1, m_b, m_l, m_u, m_m0, m_m1;
    StencilOp A;
    BandGeom Gs, Ga;
    Bounds Bd;
    const double* brow;
    double *y0p, *y1p;
    unsigned char *mk0, *mk1;
    double *lo_y0, *lo_y1, *hi_y0, *hi_y1;            // neighbours' origins of the y buffers
    unsigned char *lo_m0, *lo_m1, *hi_m0, *hi_m1;     // ... and of the mask buffers
    SlabLink Ls, La;                                  // search / accept geometries (bid set in the kernel)
    int cta0;
};
struct GpMsArgs {
    GpMsSlab s[kMaxMs];
    int nslabs;
};

template <bool SB, bool BB, bool XR>
__global__ void __launch_bounds__(m4::kThreads, GPCG_GP_MINB)
k6_gp_loop_ms(const __grid_constant__ GpMsArgs P, int cur0, double mu, Scal* S, double* __restrict__ part,
              unsigned int* gbar, int spec, const __grid_constant__ XRank XRk) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[4];
    int si = 0;
    while (si + 1 < P.nslabs && (int)blockIdx.x >= P.s[si + 1].cta0) ++si;
    const GpMsSlab& X = P.s[si];
    SlabLink Ls = X.Ls, La = X.La;
    Ls.bid = La.bid = (int)blockIdx.x - X.cta0;
    auto sp = [&](int cur, double alpha0, double (&acc)[8], int k) {
        return spec_sweep6<SB, BB>(X.A, X.Ga, X.Bd, X.brow, cur ? &X.m_y1 : &X.m_y0, &X.m_b, &X.m_l, &X.m_u,
                                   cur ? &X.m_m1 : &X.m_m0, alpha0, cur ? X.y0p : X.y1p, cur ? X.mk0 : X.mk1,
                                   smem, acc, bars, k, &La, cur ? X.lo_y0 : X.lo_y1, cur ? X.lo_m0 : X.lo_m1,
                                   cur ? X.hi_y0 : X.hi_y1, cur ? X.hi_m0 : X.hi_m1);
    };
    auto se = [&](int cur, const double (&al)[2], double (&acc)[4], int k) {
        return search_sweep5<SB, BB, m5::GP, 2>(X.A, X.Gs, X.Bd, X.brow, cur ? &X.m_y1 : &X.m_y0,
                                                cur ? &X.m_y1 : &X.m_y0, &X.m_b, &X.m_l, &X.m_u, al, smem, acc,
                                                bars, k, &Ls);
    };
    auto ac = [&](int cur, double alpha, double (&acc)[6], int k) {
        return accept_sweep5<SB, BB, m5::GP>(X.A, X.Ga, X.Bd, X.brow, cur ? &X.m_y1 : &X.m_y0,
                                             cur ? &X.m_y1 : &X.m_y0, &X.m_b, &X.m_l, &X.m_u,
                                             cur ? &X.m_m1 : &X.m_m0, 1, alpha, cur ? X.y0p : X.y1p,
                                             cur ? X.mk0 : X.mk1, smem, acc, bars, k, &La,
                                             cur ? X.lo_y0 : X.lo_y1, cur ? X.lo_m0 : X.lo_m1,
                                             cur ? X.hi_y0 : X.hi_y1, cur ? X.hi_m0 : X.hi_m1);
    };
    gp_loop<XR>(cur0, mu, S, part, gbar, spec, sp, se, ac, &XRk);
}

}  // namespace gpcg
