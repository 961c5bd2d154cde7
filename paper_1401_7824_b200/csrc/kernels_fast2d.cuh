// kernels_fast2d.cuh -- tuned fine-level 2D kernels (sm_100a): TMA-staged tiles, register-rolled
// vertical stencil windows, fused sweeps.  Every value is produced by the canonical expression
// trees of DESIGN.md §4 in the same order as the generic kernels, so results are bit-identical.
#pragma once
#include "common.cuh"
#include "tma.cuh"
#include <type_traits>

namespace f2d {

// ---------------------------------------------------------------------------------------------
// Fused two-sweep weighted Jacobi (one HBM pass: read u, b; write u''), DESIGN.md §6.1.
// Tile: 64 x TY outputs per CTA (TY = 16 by default; 24 / 8 on big / small levels, the TY_
// template), 256 threads (8 warps).  Smem: u box 68 x (TY+4) at (x0-2, y0-2), b box 68 x (TY+2)
// at (x0-2, y0-1) (TMA, zero fill outside the domain), t = first sweep on the 66 x (TY+2) region
// at (x0-1, y0-1) (zero outside the domain).  Warp w owns the 32-column half (w & 1) of a band of
// rows (w >> 1); each lane rolls a 3-row register window down its column.
// Optional: NORM -> ||b - S u||_inf over the tile (the SDC defect test of the incoming iterate).
// ---------------------------------------------------------------------------------------------
constexpr int TX = 64, TY = 16, NT = 256;   // 16-row tiles: ~33 KB smem -> 6 CTAs / SM to overlap TMA and compute
constexpr int SB1 = (TY + 2 + 3) / 4, SB2 = TY / 4;   // rows per warp band in sweep 1 / sweep 2
constexpr int UW = TX + 4, UH = TY + 4;
constexpr int BW = TX + 4, BH = TY + 2;
constexpr int TW = TX + 2, TH = TY + 2;

// MODE 0: u from memory.  MODE 1: u == 0 (first smoothing of a coarse correction: nothing is
// read, the same expressions run on zeros).  MODE 2: u + P e first (fused bilinear prolongation
// + correction): coarse box EW x EH at (x0/2 - 2, y0/2 - 2) by TMA (zero fill
// = the coarse zero ring), correction applied to every in-domain point of the u box.
constexpr int EW = 36, EH = TY / 2 + 3;

// tile height as a parameter: TY_ = 16 (above) or 32 on the large levels (fewer band starts)
template <int TY_>
struct __align__(128) SmemSmoothT {
    alignas(128) double u[TY_ + 4][UW];
    alignas(128) double b[TY_ + 2][BW];
    alignas(128) double t[TY_ + 2][TW];
    alignas(128) double e[TY_ / 2 + 3][EW];
    uint64_t bar;
};
using SmemSmooth = SmemSmoothT<TY>;

template <bool NORM, int MODE = 0, int TY_ = 16>
__global__ void __launch_bounds__(NT) k_smooth2(const __grid_constant__ CUtensorMap tu,
                                                const __grid_constant__ CUtensorMap tb, double *__restrict__ out,
                                                int n, int pitch, SCoef c, unsigned long long *slot,
                                                const __grid_constant__ CUtensorMap te) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // the tile-height dependent sizes (shadow the 16-row namespace constants)
    constexpr int TY = TY_, SB1 = (TY + 2 + 3) / 4, SB2 = TY / 4, UH = TY + 4, BH = TY + 2, TH = TY + 2;
    constexpr int EH = TY / 2 + 3;
    SmemSmoothT<TY_> &S = *reinterpret_cast<SmemSmoothT<TY_> *>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    if (tid == 0) {
        if (MODE != 1) tma_prefetch_desc(&tu);
        tma_prefetch_desc(&tb);
        mbar_init(&S.bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&S.bar, ((MODE == 1 ? 0 : UW * UH) + BW * BH + (MODE == 2 ? EW * EH : 0)) * 8);
        if (MODE != 1) tma_load_2d(&S.u[0][0], &tu, x0 - 2, y0 - 2, &S.bar);
        tma_load_2d(&S.b[0][0], &tb, x0 - 2, y0 - 1, &S.bar);
        if (MODE == 2) tma_load_2d(&S.e[0][0], &te, x0 / 2 - 2, y0 / 2 - 2, &S.bar);
    }
    if (MODE == 1) {
        for (int q = tid; q < UW * UH; q += NT) (&S.u[0][0])[q] = 0.0;
        __syncthreads();   // every thread reads zeros written by others
    }
    mbar_wait(&S.bar, 0);
    if (MODE == 2) {
        // u += P e on the u box (fine (x0-2+lx, y0-2+ly)); local coarse index of the pair / single
        // coarse neighbour: even lx -> (lx/2, lx/2+1), odd lx -> (lx+1)/2 (same for rows)
        // Column pairs (lx, lx+1), lx = 2k even: the even point takes the coarse pair (k, k+1),
        // the odd one coarse k+1, so one row of e serves both; 16-byte u accesses.  Same trees
        // as the per-point form: sx(r) = e[r][xa] (+ e[r][xa+1]); sz = sx(ya) (+ sx(ya+1)).
        // two fine rows per thread, (2r, 2r+1): the even row takes coarse rows (r, r+1), the odd one
        // row r+1, so three of the four coarse values per column pair serve both rows
        constexpr int PW = UW / 2;
        static_assert(UH % 2 == 0, "row pairs");
        for (int q = tid; q < PW * (UH / 2); q += NT) {
            const int lr = q / PW, k = q - lr * PW, lx = 2 * k, ly = 2 * lr;
            const int gx = x0 - 2 + lx, gy = y0 - 2 + ly;
            if (gx + 1 < 0 || gx >= n) continue;
            const int ya = ly / 2;                  // even row: coarse rows ya, ya + 1; odd row: ya + 1
            const double ea0 = S.e[ya][k], ea1 = S.e[ya][k + 1];
            const double eb0 = S.e[ya + 1][k], eb1 = S.e[ya + 1][k + 1];
            if (gy >= 0 && gy < n) {                // even row (ye): weights 0.25 / 0.5
                const double sze = (ea0 + ea1) + (eb0 + eb1), szo = ea1 + eb1;
                double2 v = *reinterpret_cast<const double2 *>(&S.u[ly][lx]);
                if (gx >= 0) v.x = v.x + sze * 0.25;
                if (gx + 1 < n) v.y = v.y + szo * 0.5;
                *reinterpret_cast<double2 *>(&S.u[ly][lx]) = v;
            }
            if (gy + 1 >= 0 && gy + 1 < n) {        // odd row: weights 0.5 / 1
                const double sze = eb0 + eb1, szo = eb1;
                double2 v = *reinterpret_cast<const double2 *>(&S.u[ly + 1][lx]);
                if (gx >= 0) v.x = v.x + sze * 0.5;
                if (gx + 1 < n) v.y = v.y + szo * 1.0;
                *reinterpret_cast<double2 *>(&S.u[ly + 1][lx]) = v;
            }
        }
        __syncthreads();
    }

    const double c0 = c.c0, c1 = c.c1, c2 = c.c2, wd = c.wd;
    double dmax = 0.0;
    // ---- sweep 1, main columns 0..63 of the t region (rows -1..TY, 4 bands of SB1 rows).  Row
    // pointers and three rotating register roles per 3-row step: no index arithmetic and no
    // register moves per row (the loop is issue-bound).
    {
        const int band = w >> 1, hh = w & 1;
        const int rs = -1 + SB1 * band, re = min(rs + SB1, TY + 1);
        const int x = lane + 32 * hh;              // tile column; u smem col x+2
        const bool xin = x0 + x < n;
        const double *sp = &S.u[rs + 1][x + 2];    // row rs-1
        double qa = sp[0], ra = sp[-1] + sp[1];
        sp += UW;
        double qb = sp[0], rb = sp[-1] + sp[1];    // row rs
        double qc, rc;
        const double *bp = &S.b[rs + 1][x + 2];
        double *tp = &S.t[rs + 1][x + 1];
        int y = rs, gy = y0 + rs;
#define ISDC_S1_ROW(QM, QC, QN, RM, RC, RN)                                                  \
        {                                                                                    \
            sp += UW;                                                                        \
            QN = sp[0]; RN = sp[-1] + sp[1];                                                 \
            const double f = RC + (QM + QN);                                                 \
            const double e = RM + RN;                                                        \
            const double su = (c0 * QC + c1 * f) + c2 * e;                                   \
            const bool in = xin && (unsigned)gy < (unsigned)n;                               \
            const double d = *bp - su;                                                       \
            if (NORM && in && y >= 0 && y < TY) dmax = amax(dmax, fabs(d));                 \
            *tp = in ? QC + wd * d : 0.0;                                                    \
            bp += BW; tp += TW; ++y; ++gy;                                                   \
        }
        while (y + 3 <= re) {
            ISDC_S1_ROW(qa, qb, qc, ra, rb, rc)
            ISDC_S1_ROW(qb, qc, qa, rb, rc, ra)
            ISDC_S1_ROW(qc, qa, qb, rc, ra, rb)
        }
        if (y < re) ISDC_S1_ROW(qa, qb, qc, ra, rb, rc)
        if (y < re) ISDC_S1_ROW(qb, qc, qa, rb, rc, ra)
#undef ISDC_S1_ROW
    }
    // ---- sweep 1, halo columns -1 and 64 (rows -1..32): 68 points, direct 9-point reads
    if (tid < 2 * TH) {
        const int x = (tid < TH) ? -1 : TX;
        const int y = (tid < TH ? tid : tid - TH) - 1;
        const int gx = x0 + x, gy = y0 + y;
        double v = 0.0;
        if (gx >= 0 && gx < n && gy >= 0 && gy < n) {
            const int cx = x + 2, cy = y + 2;
            double r_m = S.u[cy - 1][cx - 1] + S.u[cy - 1][cx + 1];
            double r_c = S.u[cy][cx - 1] + S.u[cy][cx + 1];
            double r_p = S.u[cy + 1][cx - 1] + S.u[cy + 1][cx + 1];
            double f = r_c + (S.u[cy - 1][cx] + S.u[cy + 1][cx]);
            double e = r_m + r_p;
            double uc = S.u[cy][cx];
            double su = (c0 * uc + c1 * f) + c2 * e;
            v = uc + wd * (S.b[y + 1][x + 2] - su);
        }
        S.t[y + 1][x + 1] = v;
    }
    if (NORM) block_max_to(slot, dmax);  // contains a __syncthreads
    __syncthreads();
    // ---- sweep 2 on the 64 x TY tile (4 bands of SB2 rows), same row-pointer / rotating form
    {
        const int band = w >> 1, hh = w & 1;
        const int rs = SB2 * band, re = rs + SB2;
        const int x = lane + 32 * hh;              // t smem col x+1
        const int gx = x0 + x;
        const double *sp = &S.t[rs][x + 1];        // row rs-1
        double qa = sp[0], ra = sp[-1] + sp[1];
        sp += TW;
        double qb = sp[0], rb = sp[-1] + sp[1];    // row rs
        double qc, rc;
        const double *bp = &S.b[rs + 1][x + 2];
        double *gp = out + (long long)(y0 + rs) * pitch + gx;
        int gy = y0 + rs, y = rs;
#define ISDC_S2_ROW(QM, QC, QN, RM, RC, RN)                                                  \
        {                                                                                    \
            sp += TW;                                                                        \
            QN = sp[0]; RN = sp[-1] + sp[1];                                                 \
            const double f = RC + (QM + QN);                                                 \
            const double e = RM + RN;                                                        \
            const double su = (c0 * QC + c1 * f) + c2 * e;                                   \
            const double v = QC + wd * (*bp - su);                                           \
            if (gx < n && gy < n) *gp = v;                                                   \
            bp += BW; gp += pitch; ++gy; ++y;                                                \
        }
        while (y + 3 <= re) {
            ISDC_S2_ROW(qa, qb, qc, ra, rb, rc)
            ISDC_S2_ROW(qb, qc, qa, rb, rc, ra)
            ISDC_S2_ROW(qc, qa, qb, rc, ra, rb)
        }
        if (y < re) ISDC_S2_ROW(qa, qb, qc, ra, rb, rc)
        if (y < re) ISDC_S2_ROW(qb, qc, qa, rb, rc, ra)
#undef ISDC_S2_ROW
    }
}

// ---------------------------------------------------------------------------------------------
// Defect + full-weighting restriction (one pass: read u, b; write b_c), DESIGN.md §6.2.
// Coarse tile 32 x 16 -> fine defect region x in [2I0, 2I0+64], y in [2J0, 2J0+32].
// Smem: u box 68x35 at (2I0-2, 2J0-1), b box 68x33 at (2I0-2, 2J0), d (65 x 33).
// ---------------------------------------------------------------------------------------------
constexpr int RCX = 32, RCY = 16, RNT = 256;
constexpr int RUW = 2 * RCX + 4, RUH = 2 * RCY + 3;
constexpr int RBW = 2 * RCX + 4, RBH = 2 * RCY + 1;
constexpr int RDW = 2 * RCX + 1, RDH = 2 * RCY + 1;

struct __align__(128) SmemRestrict {
    alignas(128) double u[RUH][RUW];
    alignas(128) double b[RBH][RBW];
    alignas(128) double d[RDH][RDW + 1];
    uint64_t bar;
};

__global__ void __launch_bounds__(RNT) k_restrict(const __grid_constant__ CUtensorMap tu,
                                                  const __grid_constant__ CUtensorMap tb, double *__restrict__ bc,
                                                  int nf, int nc, int pitch_c, SCoef c) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SmemRestrict &S = *reinterpret_cast<SmemRestrict *>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    const int tid = threadIdx.x;
    const int I0 = blockIdx.x * RCX, J0 = blockIdx.y * RCY;
    const int fx0 = 2 * I0, fy0 = 2 * J0;   // fine origin of the d region
    if (tid == 0) {
        tma_prefetch_desc(&tu);
        tma_prefetch_desc(&tb);
        mbar_init(&S.bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&S.bar, (RUW * RUH + RBW * RBH) * 8);
        tma_load_2d(&S.u[0][0], &tu, fx0 - 2, fy0 - 1, &S.bar);
        tma_load_2d(&S.b[0][0], &tb, fx0 - 2, fy0, &S.bar);
    }
    mbar_wait(&S.bar, 0);
    const double c0 = c.c0, c1 = c.c1, c2 = c.c2;
    // defect on the (2RCX+1) x (2RCY+1) fine region; d(x,y) with u smem (x+2, y+1).
    // Columns 0..63: warp w owns column half (w & 1) of row band (w >> 1) (4 bands of <= 9 rows)
    // with a rolling 3-row register window; column 64 by threads 0..32 directly.
    {
        const int lane = tid & 31, w = tid >> 5;
        const int band = w >> 1, hh = w & 1;
        const int rs = 9 * band, re = min(rs + 9, RDH);
        const int x = lane + 32 * hh, cx = x + 2;
        double um = S.u[rs][cx], rm = S.u[rs][cx - 1] + S.u[rs][cx + 1];           // row rs-1
        double uc = S.u[rs + 1][cx], rc = S.u[rs + 1][cx - 1] + S.u[rs + 1][cx + 1];
        for (int y = rs; y < re; ++y) {
            double up = S.u[y + 2][cx], rp = S.u[y + 2][cx - 1] + S.u[y + 2][cx + 1];
            double f = rc + (um + up);
            double e = rm + rp;
            double su = (c0 * uc + c1 * f) + c2 * e;
            S.d[y][x] = S.b[y][x + 2] - su;
            um = uc; uc = up; rm = rc; rc = rp;
        }
        if (tid < RDH) {
            const int y = tid, xx = RDW - 1, cxx = xx + 2, cy = y + 1;
            double r_m = S.u[cy - 1][cxx - 1] + S.u[cy - 1][cxx + 1];
            double r_c = S.u[cy][cxx - 1] + S.u[cy][cxx + 1];
            double r_p = S.u[cy + 1][cxx - 1] + S.u[cy + 1][cxx + 1];
            double f = r_c + (S.u[cy - 1][cxx] + S.u[cy + 1][cxx]);
            double e = r_m + r_p;
            double su = (c0 * S.u[cy][cxx] + c1 * f) + c2 * e;
            S.d[y][xx] = S.b[y][xx + 2] - su;
        }
    }
    __syncthreads();
    for (int p = tid; p < RCX * RCY; p += RNT) {
        const int I = p % RCX, J = p / RCX;
        const int gI = I0 + I, gJ = J0 + J;
        if (gI >= nc || gJ >= nc) continue;
        const int x = 2 * I + 1, y = 2 * J + 1;   // d-region coordinates of the coarse point
        double rd0 = S.d[y - 1][x - 1] + S.d[y - 1][x + 1];
        double rd1 = S.d[y][x - 1] + S.d[y][x + 1];
        double rd2 = S.d[y + 1][x - 1] + S.d[y + 1][x + 1];
        double fd = rd1 + (S.d[y - 1][x] + S.d[y + 1][x]);
        double ed = rd0 + rd2;
        bc[(long long)gJ * pitch_c + gI] = ((4.0 * S.d[y][x] + 2.0 * fd) + ed) * 0.0625;
    }
}

// ---------------------------------------------------------------------------------------------
// Bilinear prolongation + correction u += P e, two fine points (2t, 2t+1) per thread with 16-byte
// accesses on u, DESIGN.md §6.3.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_prolong(double *__restrict__ u, int nf, int pitch_f,
                                                 const double *__restrict__ e, int nc, int pitch_c) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;   // column pair
    const int y = blockIdx.y;
    const int x = 2 * t;
    if (x >= nf) return;
    auto E = [&](int X, int Y) -> double {
        return (X >= 0 && X < nc && Y >= 0 && Y < nc) ? e[(long long)Y * pitch_c + X] : 0.0;
    };
    const bool ye = !(y & 1);
    const int Ya = ye ? y / 2 - 1 : (y - 1) / 2, Yb = y / 2;
    // even column x = 2t: coarse pair (t-1, t); odd column 2t+1: coarse t
    double se, so;
    {
        double sx_a = E(t - 1, Ya) + E(t, Ya);
        double so_a = E(t, Ya);
        if (ye) {
            double sx_b = E(t - 1, Yb) + E(t, Yb);
            double so_b = E(t, Yb);
            se = (sx_a + sx_b) * 0.25;
            so = (so_a + so_b) * 0.5;
        } else {
            se = sx_a * 0.5;
            so = so_a;
        }
    }
    double *row = u + (long long)y * pitch_f;
    if (x + 1 < nf) {
        double2 v = *reinterpret_cast<double2 *>(row + x);
        v.x = v.x + se;
        v.y = v.y + so;
        *reinterpret_cast<double2 *>(row + x) = v;
    } else {
        row[x] = row[x] + se;
    }
}

}  // namespace f2d

namespace f2d {

// ---------------------------------------------------------------------------------------------
// Single-pass RHS of Eq. (5): v and w on the tile + 1 halo are formed
// from the M+1 node fields (and G) straight from global memory into shared memory, then
// b = B v + L w is applied from shared memory.  f^E kinds none / cubic / forcing (pointwise).
// ---------------------------------------------------------------------------------------------
constexpr int QX = 64, QY = 32, QNT = 256;
constexpr int QW = QX + 2, QH = QY + 2;

struct RhsArgs {
    const double *uold[ISDC_MAXM];
    const double *unew_m;
    const double *G;
    const double *ct;
    int M, m, fe, n, pitch;
    double dtm, gm;
    double a[ISDC_MAXM], beta[ISDC_MAXM];
    BLConst bl;
};

template <int FE>
__global__ void __launch_bounds__(QNT) k_rhs(RhsArgs A, double *__restrict__ bout, unsigned long long *slot) {
    __shared__ double vs[QH][QW];
    __shared__ double ws[QH][QW];
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * QX, y0 = blockIdx.y * QY;
    const int n = A.n, M = A.M, m = A.m;
    for (int p = tid; p < QW * QH; p += QNT) {
        const int lx = p % QW, ly = p / QW;
        const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
        double v = 0.0, w = 0.0;
        if (gx >= 0 && gx < n && gy >= 0 && gy < n) {
            const long long q = (long long)gy * A.pitch + gx;
            double uj[ISDC_MAXM];
#pragma unroll
            for (int j = 0; j < ISDC_MAXM; ++j)
                if (j < M) uj[j] = A.uold[j][q];
            double acc = A.beta[0] * uj[0];
#pragma unroll
            for (int j = 1; j < ISDC_MAXM; ++j)
                if (j < M) acc = acc + A.beta[j] * uj[j];
            double uo1 = 0.0;
#pragma unroll
            for (int j = 0; j < ISDC_MAXM; ++j)
                if (j == m + 1) uo1 = uj[j];
            w = acc - A.gm * uo1;
            const double un = A.unew_m[q];
            if (FE == 0) {
                v = un;
            } else {
                double uom = 0.0;
#pragma unroll
                for (int j = 0; j < ISDC_MAXM; ++j)
                    if (j == m) uom = uj[j];
                double fa, fn, fo;
                if (FE == 1) {
                    fa = A.a[0] * (uj[0] - (uj[0] * uj[0]) * uj[0]);
#pragma unroll
                    for (int j = 1; j < ISDC_MAXM; ++j)
                        if (j < M) fa = fa + A.a[j] * (uj[j] - (uj[j] * uj[j]) * uj[j]);
                    fn = un - (un * un) * un;
                    fo = uom - (uom * uom) * uom;
                } else {
                    const double g = A.G[q];
                    fa = A.a[0] * (g * A.ct[0]);
#pragma unroll
                    for (int j = 1; j < ISDC_MAXM; ++j)
                        if (j < M) fa = fa + A.a[j] * (g * A.ct[j]);
                    fn = g * A.ct[m];
                    fo = g * A.ct[m];
                }
                v = (un + A.dtm * (fn - fo)) + fa;
            }
        }
        vs[ly][lx] = v;
        ws[ly][lx] = w;
    }
    __syncthreads();
    const BLConst c = A.bl;
    double bmax = 0.0;
    for (int p = tid; p < QX * QY; p += QNT) {
        const int lx = p % QX, ly = p / QX;
        const int gx = x0 + lx, gy = y0 + ly;
        if (gx >= n || gy >= n) continue;
        const int cx = lx + 1, cy = ly + 1;
        double fv = (vs[cy][cx - 1] + vs[cy][cx + 1]) + (vs[cy - 1][cx] + vs[cy + 1][cx]);
        double rwm = ws[cy - 1][cx - 1] + ws[cy - 1][cx + 1];
        double rwc = ws[cy][cx - 1] + ws[cy][cx + 1];
        double rwp = ws[cy + 1][cx - 1] + ws[cy + 1][cx + 1];
        double fw = rwc + (ws[cy - 1][cx] + ws[cy + 1][cx]);
        double ew = rwm + rwp;
        double Bv = c.kB0 * vs[cy][cx] + c.kB1 * fv;
        double Lw = (c.kL0 * ws[cy][cx] + c.kL1 * fw) + c.kL2 * ew;
        double b = Bv + Lw;
        bout[(long long)gy * A.pitch + gx] = b;
        bmax = amax(bmax, fabs(b));
    }
    if (slot) block_max_to(slot, bmax);
}

// ---------------------------------------------------------------------------------------------
// Single-pass weighted SDC residual of nodes m = 1..M-1: p_m and z_m on
// the tile + 1 halo for every m from one read of the M node fields, then r~_m = B p_m - L z_m
// and a per-node max into slots[m-1].
// ---------------------------------------------------------------------------------------------
constexpr int ZX = 32, ZY = 32, ZNT = 256;
constexpr int ZW = ZX + 2, ZH = ZY + 2;

struct ResArgs {
    const double *u[ISDC_MAXM];
    const double *G;
    const double *ct;
    int M, fe, n, pitch;
    double qa[ISDC_MAXM][ISDC_MAXM];   // [m][j] = dt*Q_{m,j}
    double qb[ISDC_MAXM][ISDC_MAXM];   // [m][j] = (nu*dt)*Q_{m,j}
    BLConst bl;
};

template <int FE>
__global__ void __launch_bounds__(ZNT) k_resid(ResArgs A, unsigned long long *slots) {
    extern __shared__ __align__(16) double zsm[];
    const int M = A.M;
    double *ps = zsm;                                  // [M-1][ZH][ZW]
    double *zs = zsm + (size_t)(M - 1) * ZH * ZW;      // [M-1][ZH][ZW]
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * ZX, y0 = blockIdx.y * ZY, n = A.n;
    for (int p = tid; p < ZW * ZH; p += ZNT) {
        const int lx = p % ZW, ly = p / ZW;
        const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
        const bool in = gx >= 0 && gx < n && gy >= 0 && gy < n;
        double uj[ISDC_MAXM], fj[ISDC_MAXM];
        if (in) {
            const long long q = (long long)gy * A.pitch + gx;
#pragma unroll
            for (int j = 0; j < ISDC_MAXM; ++j)
                if (j < M) uj[j] = A.u[j][q];
            if (FE == 1) {
#pragma unroll
                for (int j = 0; j < ISDC_MAXM; ++j)
                    if (j < M) fj[j] = uj[j] - (uj[j] * uj[j]) * uj[j];
            } else if (FE == 2) {
                const double g = A.G[q];
#pragma unroll
                for (int j = 0; j < ISDC_MAXM; ++j)
                    if (j < M) fj[j] = g * A.ct[j];
            }
        }
#pragma unroll
        for (int m = 1; m < ISDC_MAXM; ++m) {
            if (m >= M) break;
            double pv = 0.0, zv = 0.0;
            if (in) {
                double diff = uj[m] - uj[0];
                if (FE != 0) {
                    double fa = A.qa[m][0] * fj[0];
#pragma unroll
                    for (int j = 1; j < ISDC_MAXM; ++j)
                        if (j < M) fa = fa + A.qa[m][j] * fj[j];
                    diff = diff - fa;
                }
                pv = diff;
                double acc = A.qb[m][0] * uj[0];
#pragma unroll
                for (int j = 1; j < ISDC_MAXM; ++j)
                    if (j < M) acc = acc + A.qb[m][j] * uj[j];
                zv = acc;
            }
            ps[(m - 1) * ZH * ZW + p] = pv;
            zs[(m - 1) * ZH * ZW + p] = zv;
        }
    }
    __syncthreads();
    const BLConst c = A.bl;
    for (int m = 1; m < M; ++m) {
        const double *P_ = ps + (m - 1) * ZH * ZW;
        const double *Z_ = zs + (m - 1) * ZH * ZW;
        double rmax = 0.0;
        for (int p = tid; p < ZX * ZY; p += ZNT) {
            const int lx = p % ZX, ly = p / ZX;
            if (x0 + lx >= n || y0 + ly >= n) continue;
            const int q = (ly + 1) * ZW + lx + 1;
            double fp = (P_[q - 1] + P_[q + 1]) + (P_[q - ZW] + P_[q + ZW]);
            double rzm = Z_[q - ZW - 1] + Z_[q - ZW + 1];
            double rzc = Z_[q - 1] + Z_[q + 1];
            double rzp = Z_[q + ZW - 1] + Z_[q + ZW + 1];
            double fz = rzc + (Z_[q - ZW] + Z_[q + ZW]);
            double ez = rzm + rzp;
            double Bp = c.kB0 * P_[q] + c.kB1 * fp;
            double Lz = (c.kL0 * Z_[q] + c.kL1 * fz) + c.kL2 * ez;
            rmax = amax(rmax, fabs(Bp - Lz));
        }
        block_max_to(slots + (m - 1), rmax);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// Warp-strip y-streaming RHS / residual.  Every warp owns a 32-column
// strip (lanes = columns x0-1 .. x0+30, outputs x0 .. x0+29) and walks down a chunk of rows:
// per row it loads the node fields of its column (coalesced, two rows ahead in registers), forms
// the pointwise values, takes x-neighbour sums with warp shuffles and keeps y rings in
// registers, emitting row y-1 when row y arrives.  No shared memory, no block barriers.
//   B q = kB0 q + kB1 f,   L q = (kL0 q + kL1 f) + kL2 e,
//   r = q(x-1) + q(x+1),  f = r + (q(y-1) + q(y+1)),  e = r(y-1) + r(y+1)
// ---------------------------------------------------------------------------------------------
constexpr int SW_NT = 256;          // 8 warps = 8 strips per CTA
constexpr int SW_OUT = 30;          // outputs per strip

__device__ __forceinline__ double shfl_up1(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shfl_dn1(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

struct StreamArgs {
    const double *u[ISDC_MAXM];     // RHS: old node fields; residual: current node fields
    const double *unew;             // RHS: u_m^{k+1}
    const double *G;                // forcing profile or null
    const double *ct;               // device cos(t_j)
    int M, m, n, pitch, yc;
    double dtm, gm;                 // RHS
    double a[ISDC_MAXM][ISDC_MAXM], beta[ISDC_MAXM][ISDC_MAXM];   // RHS: row 0 (dt S_mj, nu dt S_mj);
                                                                  // residual: rows m (dt Q_mj, nu dt Q_mj)
    BLConst bl;
    double *out;                    // RHS b
    unsigned long long *slot;       // RHS: ||b|| (optional); residual: per-node slots slot[m-1]
    double *rt[ISDC_MAXM];          // residual: r~_m fields at rt[m-1] (unweighted residual), or null
    // RHS folds of the next sweep: the residual pass also stores
    // w_q = sum_j (nu dt S_qj) u_j - (nu dt dtau_q) u_{q+1} for q = 0..M-2 at wf[q]; the RHS of
    // substep q then reads w_q instead of the M node fields
    double fb[ISDC_MAXM][ISDC_MAXM], fgm[ISDC_MAXM];
    double *wf[ISDC_MAXM];
    const double *wfold;            // RHS from folds: w_m
};

// fields loaded per row: u_0..u_{M-1}, [unew], [G], [u_{m+1}, u_m: L1 hits of the first M, loaded
// by pointer so that no register array is indexed at run time]
constexpr int SL_UN = 0, SL_G = 1, SL_UO1 = 2, SL_UOM = 3;
template <int MODE, int FE, int MM>
__device__ __forceinline__ void stream_load(const StreamArgs &A, long long off, bool in, double (&L)[MM + 4]) {
#pragma unroll
    for (int j = 0; j < MM; ++j) L[j] = in ? __ldcs(A.u[j] + off) : 0.0;
    if (MODE == 2) {               // RHS from folds: w_m, unew [, G]
        L[0] = in ? __ldcs(A.wfold + off) : 0.0;
        L[MM + SL_UN] = in ? __ldcs(A.unew + off) : 0.0;
        if (FE == 2) L[MM + SL_G] = in ? __ldg(A.G + off) : 0.0;
        return;
    }
    if (MODE == 0) {
        L[MM + SL_UN] = in ? __ldcs(A.unew + off) : 0.0;
        L[MM + SL_UO1] = in ? __ldg(A.u[A.m + 1] + off) : 0.0;
        if (FE == 1) L[MM + SL_UOM] = in ? __ldg(A.u[A.m] + off) : 0.0;
    }
    if (FE == 2) L[MM + SL_G] = in ? __ldg(A.G + off) : 0.0;
}

template <int FE>
__device__ __forceinline__ double fe_of(double u) { return u - (u * u) * u; }   // FE == 1

// v, w of substep m from the stored fold w_m (same trees as rhs_row, w read instead of formed)
template <int FE, int MM>
__device__ __forceinline__ void rhs_row_fold(const StreamArgs &A, const double (&L)[MM + 4], bool in, double &v,
                                             double &w) {
    static_assert(FE == 0 || FE == 2, "folds carry w only: f^E must be pointwise in x (none / forcing)");
    const int m = A.m;
    w = L[0];
    const double un = L[MM + SL_UN];
    if (FE == 0) {
        v = un;
    } else {
        const double g = L[MM + SL_G];
        double fa = A.a[0][0] * (g * A.ct[0]);
#pragma unroll
        for (int j = 1; j < MM; ++j)
            fa = fa + A.a[0][j] * (g * A.ct[j]);
        const double fn = g * A.ct[m], fo = g * A.ct[m];
        v = (un + A.dtm * (fn - fo)) + fa;
    }
    if (!in) { v = 0.0; w = 0.0; }
}

template <int FE, int MM>
__device__ __forceinline__ void rhs_row(const StreamArgs &A, const double (&L)[MM + 4], bool in, double &v, double &w) {
    const int m = A.m;
    double uj[MM];
#pragma unroll
    for (int j = 0; j < MM; ++j) uj[j] = L[j];
    double acc = A.beta[0][0] * uj[0];
#pragma unroll
    for (int j = 1; j < MM; ++j)
        acc = acc + A.beta[0][j] * uj[j];
    const double uo1 = L[MM + SL_UO1], uom = L[MM + SL_UOM];
    w = acc - A.gm * uo1;
    const double un = L[MM + SL_UN];
    if (FE == 0) {
        v = un;
    } else {
        double fa, fn, fo;
        if (FE == 1) {
            fa = A.a[0][0] * fe_of<1>(uj[0]);
#pragma unroll
            for (int j = 1; j < MM; ++j)
                fa = fa + A.a[0][j] * fe_of<1>(uj[j]);
            fn = fe_of<1>(un);
            fo = fe_of<1>(uom);
        } else {
            const double g = L[MM + SL_G];
            fa = A.a[0][0] * (g * A.ct[0]);
#pragma unroll
            for (int j = 1; j < MM; ++j)
                fa = fa + A.a[0][j] * (g * A.ct[j]);
            fn = g * A.ct[m];
            fo = g * A.ct[m];
        }
        v = (un + A.dtm * (fn - fo)) + fa;
    }
    if (!in) { v = 0.0; w = 0.0; }
}

template <int FE, int MM, bool FOLD = false>
__global__ void __launch_bounds__(SW_NT) k_rhs_s(StreamArgs A) {
    const int lane = threadIdx.x & 31, strip = blockIdx.x * (SW_NT / 32) + (threadIdx.x >> 5);
    const int n = A.n;
    const int x = strip * SW_OUT - 1 + lane;
    if (strip * SW_OUT >= n) return;                 // whole warp leaves together
    const int y0 = blockIdx.y * A.yc, y1 = min(y0 + A.yc, n);
    const bool xin = x >= 0 && x < n, xout = lane >= 1 && lane <= SW_OUT && x < n;
    const BLConst c = A.bl;
    double L[3][MM + 4];
    double vq[3], wq[3], vr[3], wr[3];
    double bmax = 0.0;
    const int nit = y1 - y0 + 2;                     // rows y0-1 .. y1
    auto rowoff = [&](int y) { return (long long)y * A.pitch + x; };
    auto load = [&](int it, double (&dst)[MM + 4]) {
        const int y = y0 - 1 + it;
        stream_load<FOLD ? 2 : 0, FE, MM>(A, rowoff(y), xin && y >= 0 && y < n && it < nit, dst);
    };
    load(0, L[0]);
    load(1, L[1]);
    auto step = [&](auto Kc, int it) {
        constexpr int k = decltype(Kc)::value;       // it % 3
        constexpr int km1 = (k + 2) % 3, km2 = (k + 1) % 3;
        load(it + 2, L[km1]);                        // slot of row it-1 is free (row it+2 = it-1 mod 3)
        const int y = y0 - 1 + it;
        const bool in = xin && y >= 0 && y < n;
        double v, w;
        if constexpr (FOLD) rhs_row_fold<FE, MM>(A, L[k], in, v, w);
        else rhs_row<FE, MM>(A, L[k], in, v, w);
        vq[k] = v; wq[k] = w;
        vr[k] = shfl_up1(v) + shfl_dn1(v);
        wr[k] = shfl_up1(w) + shfl_dn1(w);
        if (it >= 2 && xout) {                       // output row y-1
            const double fv = vr[km1] + (vq[km2] + vq[k]);
            const double fw = wr[km1] + (wq[km2] + wq[k]);
            const double ew = wr[km2] + wr[k];
            const double b = (c.kB0 * vq[km1] + c.kB1 * fv) + ((c.kL0 * wq[km1] + c.kL1 * fw) + c.kL2 * ew);
            A.out[rowoff(y - 1)] = b;
            bmax = amax(bmax, fabs(b));
        }
    };
    for (int base = 0; base < nit; base += 3) {
        step(std::integral_constant<int, 0>{}, base);
        if (base + 1 < nit) step(std::integral_constant<int, 1>{}, base + 1);
        if (base + 2 < nit) step(std::integral_constant<int, 2>{}, base + 2);
    }
    if (A.slot) {
        unsigned long long v = warp_max_u64((unsigned long long)__double_as_longlong(bmax));
        if (lane == 0 && v) atomicMax(A.slot, v);
    }
}

// RHS of substep m from the stored fold w_m with 128-bit loads (the north star's "SDC-sweep kernel
// ... with 128-bit vectorised fp64 loads"): a warp strip covers 64 columns [62 s - 2, 62 s + 62),
// lane l the column pair (62 s - 2 + 2 l, + 1) as one double2 per field and row (16-byte aligned:
// even column, pitch 2^p), and emits the 62 outputs [62 s - 1, 62 s + 61).  The x-pair sums take the
// outer neighbour from the adjacent lane: r(c0) = v(c0 - 1) + v(c0 + 1) = up(v1) + v1,
// r(c1) = v0 + down(v0) -- the trees of k_rhs_s, so the same bits.
constexpr int SP_OUT = 62;
template <int FE, int MM>
__global__ void __launch_bounds__(SW_NT) k_rhs_f2(StreamArgs A) {
    const int lane = threadIdx.x & 31, strip = blockIdx.x * (SW_NT / 32) + (threadIdx.x >> 5);
    const int n = A.n;
    const int c0 = strip * SP_OUT - 2 + 2 * lane;    // even: 16-byte aligned pair (c0, c0 + 1)
    if (strip * SP_OUT - 1 >= n) return;             // whole warp leaves together
    const int y0 = blockIdx.y * A.yc, y1 = min(y0 + A.yc, n);
    const bool in0 = c0 >= 0 && c0 < n, in1 = c0 + 1 >= 0 && c0 + 1 < n;
    const bool ld = c0 >= 0 && c0 < n;               // c0 + 1 <= n: the pad column (pitch n + 1) is readable
    const bool out0 = lane >= 1 && in0, out1 = lane <= 30 && in1;
    const BLConst c = A.bl;
    const double ctm = A.ct[A.m];
    double fa_c[MM];
#pragma unroll
    for (int j = 0; j < MM; ++j) fa_c[j] = A.ct[j];
    double2 Lw[3], Lu[3], Lg[3];
    double vq0[3], wq0[3], vr0[3], wr0[3], vq1[3], wq1[3], vr1[3], wr1[3];
    double bmax = 0.0;
    const int nit = y1 - y0 + 2;                     // rows y0-1 .. y1
    auto rowoff = [&](int y) { return (long long)y * A.pitch + c0; };
    auto load = [&](int it, int slot) {
        const int y = y0 - 1 + it;
        const bool ok = ld && y >= 0 && y < n && it < nit;
        const double2 z = make_double2(0.0, 0.0);
        Lw[slot] = ok ? __ldcs(reinterpret_cast<const double2 *>(A.wfold + rowoff(y))) : z;
        Lu[slot] = ok ? __ldcs(reinterpret_cast<const double2 *>(A.unew + rowoff(y))) : z;
        if (FE == 2) Lg[slot] = ok ? __ldg(reinterpret_cast<const double2 *>(A.G + rowoff(y))) : z;
    };
    // v of one point from (w, unew, G) -- rhs_row_fold's tree
    auto vpt = [&](double un, double g) {
        if (FE == 0) return un;
        double fa = A.a[0][0] * (g * fa_c[0]);
#pragma unroll
        for (int j = 1; j < MM; ++j) fa = fa + A.a[0][j] * (g * fa_c[j]);
        const double fn = g * ctm, fo = g * ctm;
        return (un + A.dtm * (fn - fo)) + fa;
    };
    load(0, 0);
    load(1, 1);
    auto step = [&](auto Kc, int it) {
        constexpr int k = decltype(Kc)::value;       // it % 3
        constexpr int km1 = (k + 2) % 3, km2 = (k + 1) % 3;
        load(it + 2, km1);                           // slot of row it-1 is free
        const int y = y0 - 1 + it;
        const bool yin = y >= 0 && y < n;
        double v0 = vpt(Lu[k].x, FE == 2 ? Lg[k].x : 0.0), v1 = vpt(Lu[k].y, FE == 2 ? Lg[k].y : 0.0);
        double w0 = Lw[k].x, w1 = Lw[k].y;
        if (!(yin && in0)) { v0 = 0.0; w0 = 0.0; }
        if (!(yin && in1)) { v1 = 0.0; w1 = 0.0; }
        vq0[k] = v0; wq0[k] = w0; vq1[k] = v1; wq1[k] = w1;
        vr0[k] = shfl_up1(v1) + v1;
        vr1[k] = v0 + shfl_dn1(v0);
        wr0[k] = shfl_up1(w1) + w1;
        wr1[k] = w0 + shfl_dn1(w0);
        if (it >= 2) {                               // output row y-1
            double *op = A.out + rowoff(y - 1);
            if (out0) {
                const double fv = vr0[km1] + (vq0[km2] + vq0[k]);
                const double fw = wr0[km1] + (wq0[km2] + wq0[k]);
                const double ew = wr0[km2] + wr0[k];
                const double b = (c.kB0 * vq0[km1] + c.kB1 * fv) + ((c.kL0 * wq0[km1] + c.kL1 * fw) + c.kL2 * ew);
                op[0] = b;
                bmax = amax(bmax, fabs(b));
            }
            if (out1) {
                const double fv = vr1[km1] + (vq1[km2] + vq1[k]);
                const double fw = wr1[km1] + (wq1[km2] + wq1[k]);
                const double ew = wr1[km2] + wr1[k];
                const double b = (c.kB0 * vq1[km1] + c.kB1 * fv) + ((c.kL0 * wq1[km1] + c.kL1 * fw) + c.kL2 * ew);
                op[1] = b;
                bmax = amax(bmax, fabs(b));
            }
        }
    };
    for (int base = 0; base < nit; base += 3) {
        step(std::integral_constant<int, 0>{}, base);
        if (base + 1 < nit) step(std::integral_constant<int, 1>{}, base + 1);
        if (base + 2 < nit) step(std::integral_constant<int, 2>{}, base + 2);
    }
    if (A.slot) {
        unsigned long long v = warp_max_u64((unsigned long long)__double_as_longlong(bmax));
        if (lane == 0 && v) atomicMax(A.slot, v);
    }
}

// residual of nodes m = 1..M-1 in one pass: p_m = (u_m - u_0) [- sum qa_mj fE(u_j)], z_m = sum qb_mj u_j,
// r~_m = B p_m - L z_m, per-node max into slot[m-1].  The M-1 nodes are split over G = (M-1)/NMW
// warps per strip (NMW nodes each; the extra loads of the same rows hit L1/L2), which halves the
// register rings and doubles the resident warps.
template <int FE, int MM, int NMW, bool WRT = false, bool WF = false>   // WRT: also store the r~_m fields (unweighted
__global__ void __launch_bounds__(SW_NT, 2) k_resid_s(StreamArgs A) {              // residual); WF: the next sweep's RHS folds
    constexpr int G = (MM - 1) / NMW;
    const int wid = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31, strip = blockIdx.x * (SW_NT / 32 / G) + wid / G;
    const int n = A.n;
    const int x = strip * SW_OUT - 1 + lane;
    if (strip * SW_OUT >= n) return;
    const int y0 = blockIdx.y * A.yc, y1 = min(y0 + A.yc, n);
    const bool xin = x >= 0 && x < n, xout = lane >= 1 && lane <= SW_OUT && x < n;
    const BLConst c = A.bl;
    // the warp's node group (role) is a compile-time constant inside `run`, so every node / fold
    // index below is an immediate (coefficients straight from the constant bank, no selects)
    auto run = [&](auto ROLE) {
    constexpr int m0 = 1 + NMW * decltype(ROLE)::value;
    double L[3][MM + 4];
    double pq[NMW][3], pr[NMW][3], zq[NMW][3], zr[NMW][3];
    double rmax[NMW];
#pragma unroll
    for (int m = 0; m < NMW; ++m) rmax[m] = 0.0;
    const int nit = y1 - y0 + 2;
    auto rowoff = [&](int y) { return (long long)y * A.pitch + x; };
    auto load = [&](int it, double (&dst)[MM + 4]) {
        const int y = y0 - 1 + it;
        stream_load<1, FE, MM>(A, rowoff(y), xin && y >= 0 && y < n && it < nit, dst);
    };
    load(0, L[0]);
    load(1, L[1]);
    auto step = [&](auto Kc, int it) {
        constexpr int k = decltype(Kc)::value;
        constexpr int km1 = (k + 2) % 3, km2 = (k + 1) % 3;
        load(it + 2, L[km1]);
        const int y = y0 - 1 + it;
        const bool in = xin && y >= 0 && y < n;
        double uj[MM], fj[MM];
#pragma unroll
        for (int j = 0; j < MM; ++j) uj[j] = L[k][j];
        if (FE == 1) {
#pragma unroll
            for (int j = 0; j < MM; ++j) fj[j] = fe_of<1>(uj[j]);
        } else if (FE == 2) {
            const double g = L[k][MM + SL_G];
#pragma unroll
            for (int j = 0; j < MM; ++j) fj[j] = g * A.ct[j];
        }
        if (WF && in && xout && y >= y0 && y < y1) {
            // this warp's folds q in [m0 - 1, m0 - 1 + NMW): w_q = sum_j fb_qj u_j - fgm_q u_{q+1}
            // (q unrolled over all folds and selected per warp, so every index is compile-time)
#pragma unroll
            for (int q = 0; q + 1 < MM; ++q) {
                if (q < m0 - 1 || q >= m0 - 1 + NMW) continue;   // compile-time
                double acc = A.fb[q][0] * uj[0];
#pragma unroll
                for (int j = 1; j < MM; ++j) acc = acc + A.fb[q][j] * uj[j];
                __stcs(A.wf[q] + rowoff(y), acc - A.fgm[q] * uj[q + 1]);   // read again only by the next sweep
            }
        }
#pragma unroll
        for (int mm = 0; mm < NMW; ++mm) {
            const int m = m0 + mm;
            double um = uj[0];
#pragma unroll
            for (int j = 1; j < MM; ++j)
                if (j == m) um = uj[j];
            double diff = um - uj[0];
            if (FE != 0) {
                double fa = A.a[m][0] * fj[0];
#pragma unroll
                for (int j = 1; j < MM; ++j) fa = fa + A.a[m][j] * fj[j];
                diff = diff - fa;
            }
            double acc = A.beta[m][0] * uj[0];
#pragma unroll
            for (int j = 1; j < MM; ++j)
                acc = acc + A.beta[m][j] * uj[j];
            const double pv = in ? diff : 0.0, zv = in ? acc : 0.0;
            pq[mm][k] = pv; zq[mm][k] = zv;
            pr[mm][k] = shfl_up1(pv) + shfl_dn1(pv);
            zr[mm][k] = shfl_up1(zv) + shfl_dn1(zv);
            if (it >= 2 && xout) {
                const double fp = pr[mm][km1] + (pq[mm][km2] + pq[mm][k]);
                const double fz = zr[mm][km1] + (zq[mm][km2] + zq[mm][k]);
                const double ez = zr[mm][km2] + zr[mm][k];
                const double Bp = c.kB0 * pq[mm][km1] + c.kB1 * fp;
                const double Lz = (c.kL0 * zq[mm][km1] + c.kL1 * fz) + c.kL2 * ez;
                const double rv = Bp - Lz;
                rmax[mm] = amax(rmax[mm], fabs(rv));
                if (WRT) A.rt[m - 1][rowoff(y - 1)] = rv;
            }
        }
    };
    for (int base = 0; base < nit; base += 3) {
        step(std::integral_constant<int, 0>{}, base);
        if (base + 1 < nit) step(std::integral_constant<int, 1>{}, base + 1);
        if (base + 2 < nit) step(std::integral_constant<int, 2>{}, base + 2);
    }
#pragma unroll
    for (int mm = 0; mm < NMW; ++mm) {
        unsigned long long v = warp_max_u64((unsigned long long)__double_as_longlong(rmax[mm]));
        if (lane == 0 && v) atomicMax(A.slot + m0 - 1 + mm, v);
    }
    };
    const int role = wid % G;
    if (role == 0) run(std::integral_constant<int, 0>{});
    if constexpr (G > 1) { if (role == 1) run(std::integral_constant<int, 1>{}); }
    if constexpr (G > 2) { if (role == 2) run(std::integral_constant<int, 2>{}); }
    if constexpr (G > 3) { if (role == 3) run(std::integral_constant<int, 3>{}); }
}

// ---------------------------------------------------------------------------------------------
// Residual of nodes m = 1..M-1 (and the next sweep's RHS folds, WF; the r~_m fields, WRT) with the
// node-field rows fed through a TMA / mbarrier ring: a CTA owns RS_SPC strips of
// 30 output columns and a chunk of rows; a producer warp streams boxes of RS_RB rows x (30 SPC + 4)
// columns of every input field (u_0..u_{M-1} [, G]) into RS_NS stages; one consumer warp per
// (strip, node m) -- which also forms fold q = m - 1 -- reads its column of every field from shared
// memory, so each field is read from HBM once per sweep and the loads in flight are set by the
// ring depth, not by per-warp register prefetch.  Every value is formed by the trees of k_resid_s.
// ---------------------------------------------------------------------------------------------
struct TMaps2 {
    CUtensorMap m[ISDC_MAXM + 1];
};
constexpr int RS_SPC = 2, RS_RB = 6;                // strips per CTA, rows per stage
constexpr int RS_BW = SW_OUT * RS_SPC + 4;           // box width (even start: x0 - 2)
template <int MM, int FE, int RS_NS = 3>           // RS_NS stages (55 KB: 4 CTAs per SM)
struct RST {
    static constexpr int K = MM + (FE == 2 ? 1 : 0);         // fields per stage
    static constexpr int NCW = RS_SPC * (MM - 1);            // consumer warps
    static constexpr int NT = 32 * (NCW + 1);                // + the producer warp
    static constexpr int FPL = RS_BW * RS_RB;                // doubles per field box
    static constexpr size_t SMEM = (size_t)RS_NS * K * FPL * 8 + 16 * RS_NS + 128;
};

template <int FE, int MM, bool WRT, bool WF, int RS_NS = 3>
__global__ void __launch_bounds__(RST<MM, FE, RS_NS>::NT) k_resid_t(const __grid_constant__ TMaps2 maps, StreamArgs A) {
    using Z = RST<MM, FE, RS_NS>;
    constexpr int K = Z::K, FPL = Z::FPL;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    double *Fs = reinterpret_cast<double *>(sm);
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)RS_NS * K * FPL * 8);
    uint64_t *empty = full + RS_NS;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = A.n;
    const int y0 = blockIdx.y * A.yc, y1 = min(y0 + A.yc, n);
    const int nit = y1 - y0 + 2;                              // rows y0-1 .. y1
    const int nst = (nit + RS_RB - 1) / RS_RB;
    const int X0 = blockIdx.x * (SW_OUT * RS_SPC) - 2;        // box origin (even)
    if (threadIdx.x == 0) {
        for (int s = 0; s < RS_NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], Z::NCW); }
        fence_mbar_init();
    }
    __syncthreads();
    if (wid == Z::NCW) {   // producer
        if (lane == 0) {
            for (int k = 0; k < K; ++k) tma_prefetch_desc(&maps.m[k]);
            for (int t = 0; t < nst; ++t) {
                const int s = t % RS_NS;
                if (t >= RS_NS) mbar_wait(&empty[s], ((t / RS_NS) - 1) & 1);
                mbar_expect_tx(&full[s], K * FPL * 8);
                for (int k = 0; k < K; ++k)
                    tma_load_2d(Fs + ((size_t)s * K + k) * FPL, &maps.m[k], X0, y0 - 1 + t * RS_RB, &full[s]);
            }
        }
        return;
    }
    const int strip_l = wid / (MM - 1), role = wid % (MM - 1);
    const int strip = blockIdx.x * RS_SPC + strip_l;
    const int x = strip * SW_OUT - 1 + lane;
    const int col = SW_OUT * strip_l + 1 + lane;             // box column of x
    const bool xin = x >= 0 && x < n, xout = lane >= 1 && lane <= SW_OUT && x < n;
    const BLConst c = A.bl;
    auto rowoff = [&](int y) { return (long long)y * A.pitch + x; };
    // node m = role + 1, fold q = role: run-time indices (one code path for every warp keeps the
    // kernel inside the instruction cache); the node selections are select chains, not indexing
    const int m = role + 1, q = role;
    // the warp's coefficient rows in registers (loaded once; no constant-bank or cos(t) loads per row)
    double ca[MM], cb[MM], cf[MM], ctr[MM];
#pragma unroll
    for (int j = 0; j < MM; ++j) {
        ca[j] = A.a[m][j];
        cb[j] = A.beta[m][j];
        cf[j] = WF ? A.fb[q][j] : 0.0;
        ctr[j] = FE == 2 ? A.ct[j] : 0.0;
    }
    const double cgm = WF ? A.fgm[q] : 0.0;
    double *const wfq = WF ? A.wf[q] : nullptr;
    double *const rtm = WRT ? A.rt[m - 1] : nullptr;
    double pq[3], pr[3], zq[3], zr[3];
    double rmax = 0.0;
    auto row = [&](auto Kc, const double *F, int it) {
        constexpr int k = decltype(Kc)::value;               // it % 3
        constexpr int km1 = (k + 2) % 3, km2 = (k + 1) % 3;
        const int y = y0 - 1 + it;
        const bool in = xin && y >= 0 && y < n;
        double uj[MM], fj[MM];
#pragma unroll
        for (int j = 0; j < MM; ++j) uj[j] = F[j * FPL];
        if (FE == 1) {
#pragma unroll
            for (int j = 0; j < MM; ++j) fj[j] = fe_of<1>(uj[j]);
        } else if (FE == 2) {
            const double g = F[MM * FPL];
#pragma unroll
            for (int j = 0; j < MM; ++j) fj[j] = g * ctr[j];
        }
        double um = uj[0];                                   // u_m (= u_{q+1} of the fold)
#pragma unroll
        for (int j = 1; j < MM; ++j)
            if (j == m) um = uj[j];
        if (WF && in && xout && y >= y0 && y < y1) {
            double acc = cf[0] * uj[0];
#pragma unroll
            for (int j = 1; j < MM; ++j) acc = acc + cf[j] * uj[j];
            __stcs(wfq + rowoff(y), acc - cgm * um);         // read again only by the next sweep
        }
        double diff = um - uj[0];
        if (FE != 0) {
            double fa = ca[0] * fj[0];
#pragma unroll
            for (int j = 1; j < MM; ++j) fa = fa + ca[j] * fj[j];
            diff = diff - fa;
        }
        double acc = cb[0] * uj[0];
#pragma unroll
        for (int j = 1; j < MM; ++j) acc = acc + cb[j] * uj[j];
        const double pv = in ? diff : 0.0, zv = in ? acc : 0.0;
        pq[k] = pv; zq[k] = zv;
        pr[k] = shfl_up1(pv) + shfl_dn1(pv);
        zr[k] = shfl_up1(zv) + shfl_dn1(zv);
        if (it >= 2 && xout) {
            const double fp = pr[km1] + (pq[km2] + pq[k]);
            const double fz = zr[km1] + (zq[km2] + zq[k]);
            const double ez = zr[km2] + zr[k];
            const double Bp = c.kB0 * pq[km1] + c.kB1 * fp;
            const double Lz = (c.kL0 * zq[km1] + c.kL1 * fz) + c.kL2 * ez;
            const double rv = Bp - Lz;
            rmax = amax(rmax, fabs(rv));
            if (WRT) rtm[rowoff(y - 1)] = rv;
        }
    };
    static_assert(RS_RB % 3 == 0, "ring index = row % 3");
    for (int t = 0; t < nst; ++t) {
        const int s = t % RS_NS;
        mbar_wait(&full[s], (t / RS_NS) & 1);
        const double *F = Fs + (size_t)s * K * FPL + col;
        const int it0 = t * RS_RB;
#pragma unroll 1
        for (int r = 0; r < RS_RB; r += 3) {
            if (it0 + r + 2 < nit) {   // three rows (the common case): no per-row guards
                row(std::integral_constant<int, 0>{}, F + r * RS_BW, it0 + r);
                row(std::integral_constant<int, 1>{}, F + (r + 1) * RS_BW, it0 + r + 1);
                row(std::integral_constant<int, 2>{}, F + (r + 2) * RS_BW, it0 + r + 2);
            } else {
                if (it0 + r < nit) row(std::integral_constant<int, 0>{}, F + r * RS_BW, it0 + r);
                if (it0 + r + 1 < nit) row(std::integral_constant<int, 1>{}, F + (r + 1) * RS_BW, it0 + r + 1);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    unsigned long long v = warp_max_u64((unsigned long long)__double_as_longlong(rmax));
    if (lane == 0 && v) atomicMax(A.slot + m - 1, v);
}

// ---------------------------------------------------------------------------------------------
// Fused pre-smoother + defect + full-weighting restriction: one pass reads
// u, b and writes the smoothed iterate u'' (tile) and b_c = R(b - S u'') (coarse tile), 26 B per
// fine point instead of 24 + 18.  Fine tile 58 x TY at (x0, y0), coarse tile 29 x TY/2 at
// (x0/2, y0/2).  Local regions (x, y relative to the tile origin):
//   t   (sweep 1)  [-2, 60] x [-2, TY+2]    u'' (sweep 2)  [-1, 59] x [-1, TY+1]
//   d   (defect)   [ 0, 58] x [ 0, TY]      u box [-4, 61] x [-3, TY+3],  b box [-2, 61] x [-2, TY+2]
// u'' overwrites the u buffer after sweep 1; the defect and the full weighting stay in registers
// (fr_defect_fw).  MODE 0: u from memory; MODE 1: u == 0 (nothing read).
// ---------------------------------------------------------------------------------------------
// Tile height TY (rows): 32 on the large levels (half the band-start loads per output of 16-row
// tiles; ~58 KB -> 3 CTAs/SM), 16 on the small ones (more CTAs).  FR_TY16 / FR_TY32 below.
constexpr int FR_TX = 58, FR_CX = 29;
constexpr int FR_UW = 66, FR_UOX = -4, FR_UOY = -3;
constexpr int FR_BW = 64, FR_BOX = -2, FR_BOY = -2;
constexpr int FR_TW = 64, FR_TOX = -2, FR_TOY = -2;
template <int TY> struct SRT {
    static constexpr int UH = TY + 7, BH = TY + 5, TH = TY + 5, CY = TY / 2;
};

template <int TY>
struct __align__(128) SmemSR {
    alignas(128) double u[SRT<TY>::UH][FR_UW];
    alignas(128) double b[SRT<TY>::BH][FR_BW];
    alignas(128) double t[SRT<TY>::TH][FR_TW];
    uint64_t bar;
};

// one stencil phase over the region [xs, xs+w) x [ys, ys+h): 2 column chunks of 32 lanes x 4 row
// bands, one (chunk, band) per warp, rolling a 3-row register window down each column.
// src/dst are arrays with origins (sox, soy) / (dox, doy) and row lengths sw / dw.
template <int KIND, int SW_, int DW_, int FR_TY, bool ZERO = false>
__device__ __forceinline__ void fr_phase(const double *__restrict__ src, int sox, int soy, double *__restrict__ dst,
                                         int dox, int doy, const double *__restrict__ B, int xs, int w, int ys,
                                         int h, int x0, int y0, int n, const SCoef &c, double *__restrict__ gout,
                                         int pitch) {
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int chunk = wp & 1, band = wp >> 1;
    const int bh = (h + 3) / 4;
    const int x = xs + 32 * chunk + lane;
    const int r0 = ys + band * bh, r1 = min(r0 + bh, ys + h);
    if (x >= xs + w || r0 >= r1) return;
    const double c0 = c.c0, c1 = c.c1, c2 = c.c2, wd = c.wd;
    if constexpr (ZERO) {
        // sweep 1 from the zero iterate: S 0 = (c0 0 + c1 0) + c2 0 = +0 for any signs of c1, c2, and
        // b - (+0) = b, so u' = 0 + wd (b - S 0) = 0.0 + wd b -- the same bits without reading u
        static_assert(KIND == 0, "zero-iterate shortcut: sweep 1 only");
        const double *bp = B + (r0 - FR_BOY) * FR_BW + (x - FR_BOX);
        double *dp = dst + (r0 - doy) * DW_ + (x - dox);
        const int gx = x0 + x;
        const bool xin = gx >= 0 && gx < n;
        for (int y = r0, gy = y0 + r0; y < r1; ++y, ++gy, bp += FR_BW, dp += DW_)
            *dp = (xin && (unsigned)gy < (unsigned)n) ? 0.0 + wd * *bp : 0.0;
        return;
    }
    // row pointers advanced by one row per step (no per-access index arithmetic)
    const double *sp = src + (r0 - 1 - soy) * SW_ + (x - sox);          // row y-1, column x
    const double *bp = B + (r0 - FR_BOY) * FR_BW + (x - FR_BOX);
    double *dp = dst + (r0 - doy) * DW_ + (x - dox);
    double qa = sp[0], ra = sp[-1] + sp[1];          // row y-1
    sp += SW_;
    double qb = sp[0], rb = sp[-1] + sp[1];          // row y
    double qc, rc;
    const int gx = x0 + x;
    const bool xin = gx >= 0 && gx < n;
    const bool xt = KIND == 1 && x >= 0 && x < FR_TX && xin;
    double *gp = (KIND == 1) ? gout + (long long)(y0 + r0) * pitch + gx : nullptr;
    int gy = y0 + r0, y = r0;
    // one output row: window rows (QM, QC, QN) with x-pair sums (RM, RC, RN); QN/RN are loaded.
    // The loop body runs three rows with rotating register roles, so no value is ever moved.
#define ISDC_FR_ROW(QM, QC, QN, RM, RC, RN)                                                   \
    {                                                                                         \
        sp += SW_;                                                                            \
        QN = sp[0]; RN = sp[-1] + sp[1];                                                      \
        const double f = RC + (QM + QN);                                                      \
        const double e = RM + RN;                                                             \
        const double su = (c0 * QC + c1 * f) + c2 * e;                                        \
        const double bv = *bp;                                                                \
        double v;                                                                             \
        if (KIND == 2) v = bv - su;                                  /* defect */             \
        else v = (xin && (unsigned)gy < (unsigned)n) ? QC + wd * (bv - su) : 0.0;            \
        *dp = v;                                                                              \
        if (KIND == 1 && xt && y >= 0 && y < FR_TY && gy < n) *gp = v;                        \
        bp += FR_BW; dp += DW_; ++gy; ++y;                                                    \
        if (KIND == 1) gp += pitch;                                                           \
    }
    while (y + 3 <= r1) {
        ISDC_FR_ROW(qa, qb, qc, ra, rb, rc)
        ISDC_FR_ROW(qb, qc, qa, rb, rc, ra)
        ISDC_FR_ROW(qc, qa, qb, rc, ra, rb)
    }
    if (y < r1) ISDC_FR_ROW(qa, qb, qc, ra, rb, rc)
    if (y < r1) ISDC_FR_ROW(qb, qc, qa, rb, rc, ra)
#undef ISDC_FR_ROW
}

// Same trees as the generic defect (apply_S) and fw_defect: rd = d(x-1) + d(x+1);
// fd = rd1 + (d0 + d2); ed = rd0 + rd2; b_c = ((4 d1 + 2 fd) + ed) * 0.0625.
template <int FR_TY>
__device__ __forceinline__ void fr_defect_fw(const SmemSR<FR_TY> &S, int x0, int y0, int nc, int pitch_c, const SCoef &c,
                                             double *__restrict__ bc) {
    constexpr int BR = FR_TY / 4;   // fine rows per band (even)
    static_assert(FR_TY % 8 == 0 && NT == 256 && FR_TX == 58, "4 bands x BR fine rows, 2 column chunks");
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int chunk = wp & 1, band = wp >> 1;
    const int x = 30 * chunk + lane, r0 = BR * band;
    const double c0 = c.c0, c1 = c.c1, c2 = c.c2;
    const double *sp = &S.u[r0 - 1 - FR_UOY][x - FR_UOX];
    const double *bp = &S.b[r0 - FR_BOY][x - FR_BOX];
    double qm = sp[0], rm = sp[-1] + sp[1];
    sp += FR_UW;
    double qc = sp[0], rc = sp[-1] + sp[1];
    const bool xo = (x & 1) && (chunk ? x >= 31 : x <= 29) && x <= 57;
    const int gI = x0 / 2 + (x - 1) / 2;
    double D0 = 0.0, R0 = 0.0, D1 = 0.0, R1 = 0.0;
#pragma unroll
    for (int yy = 0; yy <= BR; ++yy) {
        sp += FR_UW;
        const double qn = sp[0], rn = sp[-1] + sp[1];
        const double f = rc + (qm + qn);
        const double e = rm + rn;
        const double su = (c0 * qc + c1 * f) + c2 * e;
        const double d = bp[yy * FR_BW] - su;
        const double rd = __shfl_up_sync(0xffffffffu, d, 1) + __shfl_down_sync(0xffffffffu, d, 1);
        if (yy >= 2 && !(yy & 1)) {        // rows r0 + yy - 2, -1, yy: coarse row J = (r0 + yy - 2) / 2
            const int gJ = y0 / 2 + (r0 + yy - 2) / 2;
            if (xo && gI < nc && gJ < nc) {
                const double fd = R1 + (D0 + d);
                const double ed = R0 + rd;
                bc[(long long)gJ * pitch_c + gI] = ((4.0 * D1 + 2.0 * fd) + ed) * 0.0625;
            }
        }
        D0 = D1; R0 = R1; D1 = d; R1 = rd;
        qm = qc; rm = rc; qc = qn; rc = rn;
    }
}

template <int MODE, int FR_TY = 16>
__global__ void __launch_bounds__(NT) k_smooth2r(const __grid_constant__ CUtensorMap tu,
                                                 const __grid_constant__ CUtensorMap tb, double *__restrict__ out,
                                                 double *__restrict__ bc, int n, int pitch, int nc, int pitch_c,
                                                 SCoef c) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    using SR = SRT<FR_TY>;
    SmemSR<FR_TY> &S = *reinterpret_cast<SmemSR<FR_TY> *>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * FR_TX, y0 = blockIdx.y * FR_TY;
    if (tid == 0) {
        if (MODE != 1) tma_prefetch_desc(&tu);
        tma_prefetch_desc(&tb);
        mbar_init(&S.bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        mbar_expect_tx(&S.bar, ((MODE == 1 ? 0 : FR_UW * SR::UH) + FR_BW * SR::BH) * 8);
        if (MODE != 1) tma_load_2d(&S.u[0][0], &tu, x0 + FR_UOX, y0 + FR_UOY, &S.bar);
        tma_load_2d(&S.b[0][0], &tb, x0 + FR_BOX, y0 + FR_BOY, &S.bar);
    }
    mbar_wait(&S.bar, 0);
    const double *Bp = &S.b[0][0];
    // sweep 1: u -> t on [-2, 60] x [-2, 34] (MODE 1: from the zero iterate, u never read; sweep 2
    // writes every u'' point the defect reads, so the u buffer needs no zeros)
    fr_phase<0, FR_UW, FR_TW, FR_TY, MODE == 1>(&S.u[0][0], FR_UOX, FR_UOY, &S.t[0][0], FR_TOX, FR_TOY, Bp, -2, 63, -2,
                                                FR_TY + 5, x0, y0, n, c, nullptr, pitch);
    __syncthreads();
    // sweep 2: t -> u'' (into the u buffer) on [-1, 59] x [-1, 33]; the tile goes to global
    fr_phase<1, FR_TW, FR_UW, FR_TY>(&S.t[0][0], FR_TOX, FR_TOY, &S.u[0][0], FR_UOX, FR_UOY, Bp, -1, 61, -1, FR_TY + 3, x0, y0, n,
                              c, out, pitch);
    __syncthreads();
    // defect d = b - S u'' and full weighting in registers (no smem round trip): warp (chunk,
    // band) computes d on local columns [30*chunk, 30*chunk + 32) and rows 4*band .. 4*band + 4,
    // takes the x-pair sums d(x-1) + d(x+1) by shuffles and emits the coarse points of fine rows
    // 4*band + 1 and 4*band + 3 at its odd columns (chunk 0: 1..29, chunk 1: 31..57).
    fr_defect_fw(S, x0, y0, nc, pitch_c, c, bc);
}

}  // namespace f2d
