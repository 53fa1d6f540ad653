// march_tma.cuh -- TMA-fed column march (sm_100a) for the broadcast-face
// 5-point operator (journal-bearing family C0 / C2 / C3): the CG iteration (a5)
// of SURVEY.md 8(a).
//
// Work item = a BAND of 4 x 28 = 112 output columns (one warp per 28-column
// strip, 2 halo lanes per side, as in march.cuh) times a SEGMENT of kSeg grid
// rows.  The raw rows of the segment plus 2 rows of warm-up on each side stream
// through shared memory in blocks of kBR rows: one thread issues
// cp.async.bulk.tensor.2d loads (rho, p, w boxes of 116 / 112 columns and a u8
// mask box) up to kNST blocks ahead, completion counted on one mbarrier per
// stage.  The warps march down the block rows with the column-march recurrences
// of k2_cg_iter (values at west / east neighbours by warp shuffle, north /
// south from a register window), so each raw value is read from shared memory
// once -- the smem traffic of the tile kernels' five-point reads is gone, and
// no register ring is needed to hide HBM latency.  CTAs are persistent over
// the items; the load pipeline runs across item boundaries.
//
// Same arithmetic and reduction structure as k2_cg_iter / k3_cg_iter; checked
// against the CPU oracle by the same tests.
#pragma once

#include "common.cuh"
#include "fin.cuh"
#include "march.cuh"
#include "tile.cuh"

namespace gpcg {

namespace m4 {
constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kOut = 28 * kWarps;         // 112 output columns per band
constexpr int kBW = kOut + 4;             // 116 box columns (2 halo each side)
constexpr int kBR = 8;                    // rows per pipeline block
constexpr int kNST = 4;                   // pipeline stages
constexpr int kMW = 144;                  // u8 mask box width (start floored to 16 B, 116 + 15 < 144)
constexpr int kRowF = kBW * 8;            // 928 B per f64 box row
constexpr int kRho = 0;
constexpr int kP = kBR * kRowF;                       // 7424
constexpr int kW = 2 * kBR * kRowF;                   // 14848
constexpr int kM = kW + kBR * kOut * 8;               // 14848 + 7168 = 22016
constexpr int kStage = kM + kBR * kMW;                // 22016 + 1152 = 23168 (multiple of 128)
constexpr int kTx = 2 * kBR * kBW * 8 + kBR * kOut * 8 + kBR * kMW;
constexpr int kSmem = kNST * kStage + 64;
static_assert(kStage % 128 == 0, "stage alignment");
}  // namespace m4

struct BandGeom {
    int nbands, nsegs, seg;     // items = nbands * nsegs; rows [s*seg, min((s+1)*seg, ny))
    int rlo;                    // first tensor row (StencilOp::rlo)
};

// CG iteration, same recurrences as k2_cg_iter:
//   level 1  pn(r)   = [r in F] (rho(r) + beta p(r))
//   level 2  rn(r-1) = [r-1 in F] (rho(r-1) - alpha (A pn)(r-1))
//   level 3  q(r-2)  = (A rn)(r-2);  emit r-2 (free points): w += alpha pn, rho' = rn, p' = pn,
//            gamma += rn^2, delta += rn q
__global__ void __launch_bounds__(m4::kThreads, 2)
k4_cg_iter(StencilOp A, BandGeom G, const __grid_constant__ CUtensorMap m_rho, const __grid_constant__ CUtensorMap m_p,
           const __grid_constant__ CUtensorMap m_w, const __grid_constant__ CUtensorMap m_mask,
           double* __restrict__ rho_n, double* __restrict__ p_n, double* __restrict__ w_out, Scal* S, RedScratch R) {
    using namespace m4;
    if (*(volatile int*)&S->cg_done) return;
    const double alpha = S->cg_alpha, beta = S->cg_beta;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kNST * kStage);
    const int nitems = G.nbands * G.nsegs;
    const int nblk_item = (G.seg + 4 + kBR - 1) / kBR;    // blocks per item (raw rows y0-2 .. y1+2)

    // flat block sequence of this CTA: (item t = blockIdx.x + i*gridDim.x, block b)
    auto block_of = [&](int k, int& t, int& b) {
        const int i = k / nblk_item;
        t = blockIdx.x + i * (int)gridDim.x;
        b = k - i * nblk_item;
        return t < nitems;
    };
    auto issue = [&](int k) {
        int t, b;
        if (!block_of(k, t, b)) return;
        const int stage = k % kNST;
        unsigned char* st = smem + stage * kStage;
        const int band = t % G.nbands, segi = t / G.nbands;
        const int x0 = band * kOut;                       // first output column
        const int yr = segi * G.seg - 2 + b * kBR;        // first raw row of the block
        mbar_expect_tx(&bar[stage], kTx);
        tma_load_2d(st + kRho, &m_rho, x0 - 2, yr - G.rlo, &bar[stage]);
        tma_load_2d(st + kP, &m_p, x0 - 2, yr - G.rlo, &bar[stage]);
        tma_load_2d(st + kW, &m_w, x0, yr - 2 - G.rlo, &bar[stage]);    // w of the emitted rows (r - 2)
        tma_load_2d(st + kM, &m_mask, floor16(x0 - 2), yr - G.rlo, &bar[stage]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNST; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (int k = 0; k < kNST; ++k) issue(k);
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = 28 * wid + lane;                        // box column of this lane
    const bool out_lane = lane >= 2 && lane < 30;
    double acc[2] = {0.0, 0.0};
    int k = 0;
    for (int t = blockIdx.x; t < nitems; t += gridDim.x) {
        const int band = t % G.nbands, segi = t / G.nbands;
        const int x0 = band * kOut;
        const int gx = x0 - 2 + c;                        // grid column of this lane
        const int moff = (x0 - 2) - floor16(x0 - 2);
        const int y0 = segi * G.seg, y1 = min(y0 + G.seg, A.ny);
        const bool col_ok = gx >= 0 && gx < A.nx;
        Op5<true> op;
        op.init(A, gx);
        double pn_m2 = 0.0, pn_m1 = 0.0, rho_m1 = 0.0, rn_m3 = 0.0, rn_m2 = 0.0;
        unsigned char m_m1 = 0, m_m2 = 0;
        for (int b = 0; b < nblk_item; ++b, ++k) {
            const int stage = k % kNST;
            const unsigned char* st = smem + stage * kStage;
            const double* rhoS = reinterpret_cast<const double*>(st + kRho);
            const double* pS = reinterpret_cast<const double*>(st + kP);
            const double* wS = reinterpret_cast<const double*>(st + kW);
            const unsigned char* mS = st + kM;
            mbar_wait(&bar[stage], (k / kNST) & 1);
            const int yr = y0 - 2 + b * kBR;
#pragma unroll
            for (int kk = 0; kk < kBR; ++kk) {
                const int r = yr + kk;
                const unsigned char m = mS[kk * kMW + c + moff];
                const double rho = rhoS[kk * kBW + c];
                const double pn0 = m ? fma(beta, pS[kk * kBW + c], rho) : 0.0;
                const double ap = op.apply(A, r - 1, pn_m1, pn_m2, pn0);
                const double rn1 = m_m1 ? fma(-alpha, ap, rho_m1) : 0.0;
                const double q = op.apply(A, r - 2, rn_m2, rn_m3, rn1);
                const int r2 = r - 2;
                if (out_lane && m_m2 && col_ok && r2 >= y0 && r2 < y1) {
                    const long long v = (long long)gx + (long long)A.pitch * r2;
                    w_out[v] = fma(alpha, pn_m2, wS[kk * kOut + c - 2]);
                    rho_n[v] = rn_m2;
                    p_n[v] = pn_m2;
                    acc[0] = fma(rn_m2, rn_m2, acc[0]);
                    acc[1] = fma(rn_m2, q, acc[1]);
                }
                pn_m2 = pn_m1; pn_m1 = pn0;
                rho_m1 = rho;
                m_m2 = m_m1; m_m1 = m;
                rn_m3 = rn_m2; rn_m2 = rn1;
            }
            __syncthreads();                              // every warp is done with this stage
            if (threadIdx.x == 0) {
                fence_proxy_async();
                issue(k + kNST);
            }
        }
    }
    reduce_and_finish<2>(acc, R, [&](double* tt) { cg_finalize(tt[0], tt[1], S); });
}

}  // namespace gpcg
