// kernels_fast3d.cuh -- tuned 3D kernels (sm_100a) for the levels n >= 31: 2.5D z-streaming with
// TMA-loaded xy planes (3D tensor maps, zero fill outside the domain = the Dirichlet data), a
// register ring in z per owned point and a 6-row register window in y, so every 19-point
// application costs 18 shared loads per 4 points.  Every value is produced by the canonical
// trees of DESIGN.md §4 in the same order as the generic kernels (bit-identical results):
//   r = q(x-1) + q(x+1);  f = r + (q(y-1) + q(y+1));  e = r(y-1) + r(y+1)
//   faces = f(z) + (q(z-1) + q(z+1));  edges = e(z) + (f(z-1) + f(z+1))
//   S u = (c0 u + c1 faces) + c2 edges;  Jacobi u + wd (b - S u)
//
// Thread layout shared by the streaming kernels: 8 warps, lane = column of a 32-wide region,
// warp w owns rows 4w..4w+3 of a 32-row region.
// TMA boxes must start at an even x (16-byte aligned global start of every row), so boxes that
// need an odd left halo start one column further left.
#pragma once
#include "common.cuh"
#include "tma.cuh"
#include <type_traits>

namespace f3d {

constexpr int NW = 8;            // warps per CTA
constexpr int NT = NW * 32;      // threads per CTA
constexpr int R = 4;             // rows per thread
constexpr int RW = 32;           // region width (one lane per column)
constexpr int RH = NW * R;       // region height

__host__ __device__ constexpr int a128(int b) { return (b + 127) / 128 * 128; }
// tiles per axis of the shifted tiling (tile t, region t + 2): the first tile emits t + 1 points
// (0 .. t), tile k >= 1 the points kt + 1 .. kt + t, and the region's last point where it is n - 1
__host__ __device__ constexpr int sh_tiles(int n, int t) { return n <= t + 2 ? 1 : (n - 2 + t - 1) / t; }

// In-plane partial sums of the R owned rows from a plane in shared memory (row stride `ld`):
// window rows row0 .. row0+R+1 (centre rows row0+1 .. row0+R), columns col0 .. col0+2 (centre
// col0+1).  q = centre value, f = face sum, e = edge sum, all in the canonical order.
template <bool WANT_E, int RR = R>
__device__ __forceinline__ void plane_partials(const double *__restrict__ P, int ld, int row0, int col0, double (&q)[RR],
                                               double (&f)[RR], double (&e)[RR]) {
    double v0[RR + 2], v1[RR + 2], v2[RR + 2];
#pragma unroll
    for (int k = 0; k < RR + 2; ++k) {
        const double *row = P + (row0 + k) * ld + col0;
        v0[k] = row[0];
        v1[k] = row[1];
        v2[k] = row[2];
    }
    double rr[RR + 2];
#pragma unroll
    for (int k = 0; k < RR + 2; ++k) rr[k] = v0[k] + v2[k];
#pragma unroll
    for (int r = 0; r < RR; ++r) {
        q[r] = v1[r + 1];
        f[r] = rr[r + 1] + (v1[r] + v1[r + 2]);
        if (WANT_E) e[r] = rr[r] + rr[r + 2];
    }
}

// ---------------------------------------------------------------------------------------------
// Fused two-sweep weighted Jacobi, one HBM pass (read u, b; write u''), DESIGN.md §6.7.
// Output tile 30 x 30 (x, y) x a z chunk [z0, z1).  Sweep 1 runs on the 32 x 32 region
// (tile + 1 halo) at plane p-1 while u plane p is ingested; its result t goes to a shared plane;
// sweep 2 runs on the tile at plane p-2 from t's register ring and the t plane's neighbours.
// u box 34 x 34 at (x0-2, y0-2); b box 34 x 32 at (x0-2, y0-1); t plane 34 x 34 (pad ring).
// ---------------------------------------------------------------------------------------------
constexpr int S_TX = RW - 2, S_TY = RH - 2;
constexpr int S_UW = RW + 2, S_UH = RH + 2;
constexpr int S_BW = RW + 2, S_BH = RH;
constexpr int S_TW = RW + 2, S_TH = RH + 2;
constexpr int S_NS = 6;          // TMA pipeline depth (planes in flight)
constexpr int S_UPL = a128(S_UW * S_UH * 8), S_BPL = a128(S_BW * S_BH * 8), S_TPL = a128(S_TW * S_TH * 8);
constexpr size_t S_SMEM = (size_t)S_NS * (S_UPL + S_BPL) + 2 * S_TPL + 8 * S_NS + 128;

// region-height-dependent sizes of the fused smoother (region RHR = SR x warps rows; the constants
// above are the 32-row case)
template <int RHR>
struct SS {
    static constexpr int TY = RHR - 2, UH = RHR + 2, BH = RHR, TH = RHR + 2;
    static constexpr int UPL = a128(S_UW * UH * 8), BPL = a128(S_BW * BH * 8), TPL = a128(S_TW * TH * 8);
    static constexpr size_t SMEM = (size_t)S_NS * (UPL + BPL) + 2 * TPL + 8 * S_NS + 128;
};

// Register state of one thread (SR owned points).  Rings are indexed by the iteration that
// produced the value (mod 3 for centre/face sums, mod 2 for edge sums and b), so after unrolling
// the z loop by 6 every index is a compile-time constant and no value is ever moved.
template <int SR>
struct SmoothRegs {
    double q[3][SR], f[3][SR], e[2][SR];      // u(p): centre, face, edge partials
    double tq[3][SR], tf[3][SR], te[2][SR];   // t(p-1) (first sweep), same partials
    double bb[2][SR];                         // b(p-1)
};

template <int SR>
struct SmoothCtx {
    const double *Us, *Bs;
    double *Ts;
    uint64_t *bar;
    double *optr;                  // output address of the owned column at plane z0 - 4, row ly0
    long long plane;
    int pitch, n, row0, lane, z0;
    unsigned inxy, oks;            // bit r: owned point r inside the domain (xy) / an output point
    double c0, c1, c2, wd;
};

template <int SR, int K, int RHR>   // K = it % 6 = it % S_NS (the z loop is unrolled by 6 from it = 0)
__device__ __forceinline__ void smooth_step(const SmoothCtx<SR> &C, SmoothRegs<SR> &G, int it, uint32_t phase) {
    using Z = SS<RHR>;
    static_assert(S_NS == 6, "stage index = K");
    constexpr int i3 = K % 3, m3 = (K + 2) % 3, mm3 = (K + 1) % 3;   // it, it-1, it-2 (mod 3)
    constexpr int i2 = K % 2, m2 = (K + 1) % 2;                       // it, it-1 (mod 2)
    constexpr int s = K;
    mbar_wait(&C.bar[s], phase);
    plane_partials<true, SR>(C.Us + s * (Z::UPL / 8), S_UW, C.row0, C.lane, G.q[i3], G.f[i3], G.e[i2]);
    double *T = C.Ts + i2 * (Z::TPL / 8);
    if (it >= 2) {   // sweep 1 at plane gz = p-1 on the 32 x 32 region
        const int gz = C.z0 - 3 + it;
        const unsigned in = ((unsigned)gz < (unsigned)C.n) ? C.inxy : 0u;
        const double *Bp = C.Bs + s * (Z::BPL / 8) + C.row0 * S_BW + C.lane + 1;
        double *Tp = T + (C.row0 + 1) * S_TW + C.lane + 1;
#pragma unroll
        for (int r = 0; r < SR; ++r) {
            const double faces = G.f[m3][r] + (G.q[mm3][r] + G.q[i3][r]);
            const double edges = G.e[m2][r] + (G.f[mm3][r] + G.f[i3][r]);
            const double su = (C.c0 * G.q[m3][r] + C.c1 * faces) + C.c2 * edges;
            const double bv = Bp[r * S_BW];
            const double t = G.q[m3][r] + C.wd * (bv - su);
            Tp[r * S_TW] = ((in >> r) & 1u) ? t : 0.0;
            G.bb[i2][r] = bv;
        }
    }
}

template <int SR, int K, int RHR>
__device__ __forceinline__ void smooth_step2(const SmoothCtx<SR> &C, SmoothRegs<SR> &G, int it) {
    using Z = SS<RHR>;
    constexpr int i3 = K % 3, m3 = (K + 2) % 3, mm3 = (K + 1) % 3;
    constexpr int i2 = K % 2, m2 = (K + 1) % 2;
    if (it < 2) return;
    const double *T = C.Ts + i2 * (Z::TPL / 8);
    plane_partials<true, SR>(T, S_TW, C.row0, C.lane, G.tq[i3], G.tf[i3], G.te[i2]);
    if (it >= 4) {   // sweep 2 at plane p-2 = z0 - 4 + it on the 30 x 30 tile
        double *op = C.optr + (long long)it * C.plane;
#pragma unroll
        for (int r = 0; r < SR; ++r) {
            const double faces = G.tf[m3][r] + (G.tq[mm3][r] + G.tq[i3][r]);
            const double edges = G.te[m2][r] + (G.tf[mm3][r] + G.tf[i3][r]);
            const double su = (C.c0 * G.tq[m3][r] + C.c1 * faces) + C.c2 * edges;
            const double o = G.tq[m3][r] + C.wd * (G.bb[m2][r] - su);
            if ((C.oks >> r) & 1u) *op = o;
            op += C.pitch;
        }
    }
}

// u box 34 x 34 at (x0-2, y0-2); b box 34 x 32 at (x0-2, y0-1); t plane 34 x 34 (pad ring).
// SR rows per thread, NWW warps (region SR * NWW rows).  MODE 0: u from memory; MODE 1: u == 0
// (first smoothing of a coarse correction: u is neither stored nor read, the u stages stay zero).
template <int SR, int MODE, int NWW = 32 / SR>
__global__ void __launch_bounds__(32 * NWW, 1) k_smooth2(const __grid_constant__ CUtensorMap tu,
                                                                const __grid_constant__ CUtensorMap tb,
                                                                double *__restrict__ out, int n, int pitch,
                                                                long long plane, SCoef c, int zc) {
    constexpr bool ZERO = MODE == 1;
    constexpr int RHR = SR * NWW;   // region rows
    using Z = SS<RHR>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);   // stays a shared pointer
    SmoothCtx<SR> C;
    C.Us = reinterpret_cast<const double *>(sm);
    C.Bs = reinterpret_cast<const double *>(sm + S_NS * Z::UPL);
    C.Ts = reinterpret_cast<double *>(sm + S_NS * (Z::UPL + Z::BPL));
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S_NS * (Z::UPL + Z::BPL) + 2 * Z::TPL);
    C.bar = bar;
    const int tid = threadIdx.x;
    C.lane = tid & 31;
    C.row0 = SR * (tid >> 5);
    const int x0 = blockIdx.x * S_TX, y0 = blockIdx.y * Z::TY;
    const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, n);
    const int nit = z1 - z0 + 4;
    C.z0 = z0; C.n = n; C.pitch = pitch; C.plane = plane;
    double *Usw = reinterpret_cast<double *>(sm), *Bsw = reinterpret_cast<double *>(sm + S_NS * Z::UPL);
    auto issue = [&](int it) {
        const int s = it % S_NS, p = z0 - 2 + it;
        mbar_expect_tx(&bar[s], ((ZERO ? 0 : S_UW * Z::UH) + S_BW * Z::BH) * 8);
        if (!ZERO) tma_load_3d(Usw + s * (Z::UPL / 8), &tu, x0 - 2, y0 - 2, p, &bar[s]);
        tma_load_3d(Bsw + s * (Z::BPL / 8), &tb, x0 - 2, y0 - 1, p - 1, &bar[s]);
    };
    if (tid == 0) {
        tma_prefetch_desc(&tu);
        tma_prefetch_desc(&tb);
        for (int s = 0; s < S_NS; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    if (ZERO)
        for (int s = 0; s < S_NS; ++s)
            for (int q = tid; q < S_UW * Z::UH; q += blockDim.x) Usw[s * (Z::UPL / 8) + q] = 0.0;
    __syncthreads();
    if (tid == 0)
        for (int it = 0; it < S_NS && it < nit; ++it) issue(it);

    C.c0 = c.c0; C.c1 = c.c1; C.c2 = c.c2; C.wd = c.wd;
    const int lx = C.lane - 1, ly0 = C.row0 - 1;        // region coordinates of the owned points
    const int gx = x0 + lx;
    const bool xin = gx >= 0 && gx < n;
    const bool xout = lx >= 0 && lx < S_TX && gx < n;
    C.inxy = 0u; C.oks = 0u;
#pragma unroll
    for (int r = 0; r < SR; ++r) {
        const int ly = ly0 + r, gy = y0 + ly;
        if (xin && gy >= 0 && gy < n) C.inxy |= 1u << r;
        if (xout && ly >= 0 && ly < Z::TY && gy < n) C.oks |= 1u << r;
    }
    C.optr = out + (long long)(z0 - 4) * plane + (long long)(y0 + ly0) * pitch + gx;
    SmoothRegs<SR> G;
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int r = 0; r < SR; ++r) G.bb[k][r] = 0.0;
#define ISDC_SMOOTH_STEP(K)                                            \
    {                                                                  \
        const int it = base + (K);                                     \
        if (it < nit) {                                                \
            smooth_step<SR, K, RHR>(C, G, it, phase);    \
            __syncthreads();                                           \
            if (tid == 0 && it + S_NS < nit) issue(it + S_NS);         \
            smooth_step2<SR, K, RHR>(C, G, it);                       \
        }                                                              \
    }
    for (int base = 0; base < nit; base += 6) {
        const uint32_t phase = (base / 6) & 1;
        ISDC_SMOOTH_STEP(0) ISDC_SMOOTH_STEP(1) ISDC_SMOOTH_STEP(2)
        ISDC_SMOOTH_STEP(3) ISDC_SMOOTH_STEP(4) ISDC_SMOOTH_STEP(5)
    }
#undef ISDC_SMOOTH_STEP
}

// ---------------------------------------------------------------------------------------------
// Warp-specialised fused two-sweep Jacobi: the tiles, trees and TMA boxes of
// k_smooth2<4, MODE, 8>, with sweep 1 and sweep 2 in separate groups of 8 warps (register rings of
// one sweep each, 16 warps per SM instead of 8) that run one plane apart and meet at one block
// barrier per plane.  MODE 0: u from memory; 1: u == 0 (nothing read); 2: u + P e first -- the
// trilinear prolongation + correction fused in (the sweep-1 group adds P e to each u plane in
// shared memory, in place, one plane ahead of its own partials; the two coarse planes of each fine
// plane arrive by TMA with its stage), so the fine post-smoothing moves 25 B/pt instead of 17 + 24.
// Stage j (plane p = z0 - 2 + j): u box 34 x 34 at (x0-2, y0-2, p), b box 34 x 32 at
// (x0-2, y0-1, p-1), MODE 2: coarse boxes 20 x 18 at (ex0, ey0) of planes za, za + 1.
// At iteration it sweep 1 handles stage it (t(p-1) -> T[it % 2]; MODE 2: first P e into stage
// it + 1), sweep 2 the t plane of stage it - 1 (output at p - 3 with b from stage it - 2).
// ---------------------------------------------------------------------------------------------
constexpr int WS_SR = 4, WS_GW = 8;                 // rows per thread, warps per sweep group
constexpr int WS_EW = 20, WS_EH = 18;               // coarse boxes (MODE 2)
constexpr int WS_EPL = a128(WS_EW * WS_EH * 8);
// SH (MODE 0 / 1): shifted tiling -- the region starts AT the tile origin (x0, y0) = 30 (bx, by)
// instead of one point before it, and the region's first / last point is an output where it is the
// domain's first / last point (its outer t neighbour is the Dirichlet zero of the t plane's pad
// ring, which needs no computing).  ceil((n - 2) / 30) tiles per axis instead of ceil(n / 30): 17
// instead of 18 at n = 511 (the 18th tile held one column).  Boxes (even x start): u 36 x 34 at
// (x0 - 2, y0 - 1), b 32 x 32 at (x0, y0).
constexpr int WS_UWS = RW + 4, WS_BWS = RW;
constexpr int WS_UPLS = a128(WS_UWS * S_UH * 8), WS_BPLS = a128(WS_BWS * S_BH * 8);
template <int MODE, int NSX = 0, bool SH = false>
struct WSCfg {
    // TMA stages (3 in use: it - 2 .. it; + 1 in MODE 2).  Default 6; the host picks NSX = 8 for the
    // shifted tiling with u from memory (one z chunk of 515 planes per tile at 511^3: 0.660 vs 0.694 ms
    // per fine launch; 10 stages: 0.688).  With the unshifted 18 x 18 x 5-chunk grid 8 and 10 stages
    // had measured slower (0.83 vs 0.79 ms)
    static constexpr int NS = NSX ? NSX : (MODE == 2 ? 7 : 6);
    static constexpr int NT = 32 * 2 * WS_GW;
    static constexpr int UPL = SH ? WS_UPLS : S_UPL, BPL = SH ? WS_BPLS : S_BPL, EPL = MODE == 2 ? 2 * WS_EPL : 0;
    static constexpr int UW = SH ? WS_UWS : S_UW, BW = SH ? WS_BWS : S_BW;
    static constexpr int SPL = UPL + BPL + EPL;     // one stage: u | b | e(za) | e(za+1)
    static constexpr size_t SMEM = (size_t)NS * SPL + 2 * S_TPL + 8 * NS + 128;
};

// MODE 2: u(p) += P e on the u box of one stage (in-domain points only), 2 x 2 fine blocks per
// thread (one double2 per box row), canonical nesting x, then y, then z, one multiply by
// 0.5^(#even axes) (the trees of k_prolong).
__device__ __forceinline__ void ws_prolong_plane(double *U, const double *Ea, const double *Eb, int p, int n, int x0,
                                                 int y0, int dlt, int ptid) {
    if ((unsigned)p >= (unsigned)n) return;
    const bool ze = !(p & 1);
    const double zw = ze ? 0.5 : 1.0;
    for (int q = ptid; q < 17 * 17; q += 32 * WS_GW) {
        const int a = q % 17, b = q / 17;           // fine box cols 2a, 2a+1; rows 2b, 2b+1
        const int gxe = x0 - 2 + 2 * a, gye = y0 - 2 + 2 * b;
        const bool ine = (unsigned)gxe < (unsigned)n, ino = (unsigned)(gxe + 1) < (unsigned)n;
        if (!ine && !ino) continue;
        const double *ra = Ea + b * WS_EW + a + dlt;
        double see = (ra[0] + ra[1]) + (ra[WS_EW] + ra[WS_EW + 1]);
        double soe = ra[1] + ra[WS_EW + 1];
        double seo = ra[WS_EW] + ra[WS_EW + 1];
        double soo = ra[WS_EW + 1];
        if (ze) {
            const double *rb = Eb + b * WS_EW + a + dlt;
            see = see + ((rb[0] + rb[1]) + (rb[WS_EW] + rb[WS_EW + 1]));
            soe = soe + (rb[1] + rb[WS_EW + 1]);
            seo = seo + (rb[WS_EW] + rb[WS_EW + 1]);
            soo = soo + rb[WS_EW + 1];
        }
        // weights (ye ? 0.5 : 1) * (ze ? 0.5 : 1), the even column * 0.5 (exact powers of two)
        const double w_e = 0.5 * zw, w_o = zw;      // even row, odd row
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int gy = gye + rr;
            if ((unsigned)gy >= (unsigned)n) continue;
            double2 *up = reinterpret_cast<double2 *>(U + (2 * b + rr) * S_UW + 2 * a);
            double2 v = *up;
            const double w = rr ? w_o : w_e;
            if (ine) v.x = v.x + (rr ? seo : see) * (w * 0.5);
            if (ino) v.y = v.y + (rr ? soo : soe) * w;
            *up = v;
        }
    }
}

template <int MODE, int NSX = 0, bool SH = false>
__global__ void __launch_bounds__(WSCfg<MODE, NSX, SH>::NT, 1) k_smooth2ws(const __grid_constant__ CUtensorMap tu,
                                                                 const __grid_constant__ CUtensorMap tb,
                                                                 const __grid_constant__ CUtensorMap te,
                                                                 double *__restrict__ out, int n, int pitch,
                                                                 long long plane, SCoef c, int zc) {
    using W = WSCfg<MODE, NSX, SH>;
    constexpr int NS = W::NS, SR = WS_SR;
    constexpr bool ZERO = MODE == 1, PRO = MODE == 2;
    static_assert(!(SH && PRO), "shifted tiling: MODE 0 / 1 only");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    double *St = reinterpret_cast<double *>(sm);
    double *Ts = reinterpret_cast<double *>(sm + NS * W::SPL);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + NS * W::SPL + 2 * S_TPL);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int x0 = blockIdx.x * S_TX, y0 = blockIdx.y * S_TY;
    const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, n);
    const int nit = z1 - z0 + 4;                    // stages: planes z0-2 .. z1+1
    const int niter = nit + 1;                      // sweep 2 trails the stages by one
    const int ex0 = ((x0 >> 1) - 2) & ~1, ey0 = (y0 >> 1) - 2;   // coarse box origin (even x: TMA rule)
    auto stage = [&](int j) { return St + (size_t)(j % NS) * (W::SPL / 8); };
    auto issue = [&](int j) {
        const int p = z0 - 2 + j;
        double *S = stage(j);
        uint64_t *bb = &bar[j % NS];
        mbar_expect_tx(bb, ((ZERO ? 0 : W::UW * S_UH) + W::BW * S_BH + (PRO ? 2 * WS_EW * WS_EH : 0)) * 8);
        if (!ZERO) tma_load_3d(S, &tu, x0 - 2, SH ? y0 - 1 : y0 - 2, p, bb);
        tma_load_3d(S + W::UPL / 8, &tb, SH ? x0 : x0 - 2, SH ? y0 : y0 - 1, p - 1, bb);
        if (PRO) {
            const int za = (p & 1) ? (p - 1) / 2 : p / 2 - 1;   // odd p: (p-1)/2; even p: p/2 - 1 and p/2
            tma_load_3d(S + (W::UPL + W::BPL) / 8, &te, ex0, ey0, za, bb);
            tma_load_3d(S + (W::UPL + W::BPL + WS_EPL) / 8, &te, ex0, ey0, za + 1, bb);
        }
    };
    if (tid == 0) {
        tma_prefetch_desc(&tu);
        tma_prefetch_desc(&tb);
        if (PRO) tma_prefetch_desc(&te);
        for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    if (SH)            // the t planes' pad ring is the Dirichlet zero read by the boundary outputs
        for (int q = tid; q < 2 * (S_TPL / 8); q += W::NT) Ts[q] = 0.0;
    __syncthreads();   // (MODE 1 reads no u: the zero-iterate sweep never touches the u stages)
    if (tid == 0)
        for (int j = 0; j < NS && j < nit; ++j) issue(j);

    const int role = w < WS_GW ? 0 : 1;             // sweep 1 | sweep 2
    const int row0 = SR * (w % WS_GW);
    const double c0 = c.c0, c1 = c.c1, c2 = c.c2, wd = c.wd;
    const int lx = SH ? lane : lane - 1, ly0 = SH ? row0 : row0 - 1;   // region coordinates of the owned points
    const int gx = x0 + lx;
    const bool xin = gx >= 0 && gx < n;
    // outputs: the region minus its one-point rim, plus the rim points on the domain boundary (SH)
    const bool xout = SH ? (gx < n && (lane >= 1 || gx == 0) && (lane <= S_TX || gx == n - 1))
                         : (lx >= 0 && lx < S_TX && gx < n);
    constexpr int UC0 = SH ? 1 : 0;                 // u box column of the owned point's left neighbour - lane
    constexpr int BC0 = SH ? 0 : 1;                 // b box column of the owned point - lane
    unsigned inxy = 0u, oks = 0u;
#pragma unroll
    for (int r = 0; r < SR; ++r) {
        const int ly = ly0 + r, gy = y0 + ly;
        if (xin && gy >= 0 && gy < n) inxy |= 1u << r;
        const bool yout = SH ? (gy < n && (ly >= 1 || gy == 0) && (ly <= S_TY || gy == n - 1))
                             : (ly >= 0 && ly < S_TY && gy < n);
        if (xout && yout) oks |= 1u << r;
    }
    double *optr = out + (long long)(z0 - 4) * plane + (long long)(y0 + ly0) * pitch + gx;
    // rings of one sweep (role 0: u partials; role 1: t partials), indexed by stage mod 3 / mod 2
    double q[3][SR], f[3][SR], e[2][SR];
    const int dlt = ((x0 >> 1) - 2) - ex0;
    auto prolong = [&](int j) {   // MODE 2, sweep-1 group: stage j's u plane += P e
        mbar_wait(&bar[j % NS], (j / NS) & 1);
        double *S = stage(j);
        ws_prolong_plane(S, S + (W::UPL + W::BPL) / 8, S + (W::UPL + W::BPL + WS_EPL) / 8, z0 - 2 + j, n, x0, y0,
                         dlt, tid);
    };
    if (PRO) {
        if (role == 0) prolong(0);
        __syncthreads();
    }

    if constexpr (!PRO) {
        // Decoupled groups (MODE 0 / 1): no block barrier per plane.  The t plane is double-buffered
        // between the groups with named barriers -- FULL[b] (sweep 1 arrives after writing T[b],
        // sweep 2 syncs before reading it) and EMPTY[b] (sweep 2 arrives after reading T[b], sweep 1
        // syncs before overwriting it) -- so the groups drift by up to two planes.  The sweep-2 group
        // refills the TMA stage it has finished (its b of stage j2 - 1), after a group-local barrier.
        constexpr int BAR_FULL = 1, BAR_EMPTY = 3, BAR_SW2 = 5;
        if (role == 0) {
            auto step1 = [&](auto Kc, int j) {
                constexpr int K = decltype(Kc)::value;      // j % 6
                constexpr int i3 = K % 3, m3 = (K + 2) % 3, mm3 = (K + 1) % 3, i2 = K % 2, m2 = (K + 1) % 2;
                mbar_wait(&bar[j % NS], (j / NS) & 1);
                const double *S = stage(j);
                if (!ZERO) plane_partials<true, SR>(S, W::UW, row0, lane + UC0, q[i3], f[i3], e[i2]);
                if (j >= 2) {   // sweep 1 at plane z0 - 3 + j on the 32 x 32 region -> T[j % 2]
                    const int gz = z0 - 3 + j;
                    const unsigned in = ((unsigned)gz < (unsigned)n) ? inxy : 0u;
                    const double *Bp = S + W::UPL / 8 + row0 * W::BW + lane + BC0;
                    double *Tp = Ts + i2 * (S_TPL / 8) + (row0 + 1) * S_TW + lane + 1;
                    double tv[SR];
#pragma unroll
                    for (int r = 0; r < SR; ++r) {
                        double t;
                        if (ZERO) {
                            // from the zero iterate: S 0 = +0 whatever the signs of c1, c2, so
                            // u' = 0 + wd (b - S 0) = 0.0 + wd b (the same bits, u never read)
                            t = 0.0 + wd * Bp[r * W::BW];
                        } else {
                            const double faces = f[m3][r] + (q[mm3][r] + q[i3][r]);
                            const double edges = e[m2][r] + (f[mm3][r] + f[i3][r]);
                            const double su = (c0 * q[m3][r] + c1 * faces) + c2 * edges;
                            t = q[m3][r] + wd * (Bp[r * W::BW] - su);
                        }
                        tv[r] = ((in >> r) & 1u) ? t : 0.0;
                    }
                    if (j >= 4) named_bar_sync(BAR_EMPTY + i2, W::NT);   // sweep 2 has read T[i2] of step j - 2
#pragma unroll
                    for (int r = 0; r < SR; ++r) Tp[r * S_TW] = tv[r];
                    named_bar_arrive(BAR_FULL + i2, W::NT);
                }
            };
            for (int base = 0; base < nit; base += 6) {
                if (base + 0 < nit) step1(std::integral_constant<int, 0>{}, base + 0);
                if (base + 1 < nit) step1(std::integral_constant<int, 1>{}, base + 1);
                if (base + 2 < nit) step1(std::integral_constant<int, 2>{}, base + 2);
                if (base + 3 < nit) step1(std::integral_constant<int, 3>{}, base + 3);
                if (base + 4 < nit) step1(std::integral_constant<int, 4>{}, base + 4);
                if (base + 5 < nit) step1(std::integral_constant<int, 5>{}, base + 5);
            }
        } else {
            auto step2 = [&](auto Kc, int j2) {
                constexpr int K = decltype(Kc)::value;      // j2 % 6
                constexpr int i3 = K % 3, m3 = (K + 2) % 3, mm3 = (K + 1) % 3, i2 = K % 2, m2 = (K + 1) % 2;
                if (j2 < 2) return;
                named_bar_sync(BAR_FULL + i2, W::NT);
                plane_partials<true, SR>(Ts + i2 * (S_TPL / 8), S_TW, row0, lane, q[i3], f[i3], e[i2]);
                if (j2 + 2 < nit) named_bar_arrive(BAR_EMPTY + i2, W::NT);   // T[i2] read (sweep 1 reuses it at j2 + 2)
                if (j2 >= 4) {   // sweep 2 at plane z0 - 4 + j2 on the 30 x 30 tile, b from stage j2 - 1
                    const double *Bp = stage(j2 - 1) + W::UPL / 8 + row0 * W::BW + lane + BC0;
                    double *op = optr + (long long)j2 * plane;
#pragma unroll
                    for (int r = 0; r < SR; ++r) {
                        const double faces = f[m3][r] + (q[mm3][r] + q[i3][r]);
                        const double edges = e[m2][r] + (f[mm3][r] + f[i3][r]);
                        const double su = (c0 * q[m3][r] + c1 * faces) + c2 * edges;
                        const double o = q[m3][r] + wd * (Bp[r * W::BW] - su);
                        if ((oks >> r) & 1u) *op = o;
                        op += pitch;
                    }
                }
                // stages <= j2 - 1 are finished by both groups (sweep 1 passed step j2): refill them
                named_bar_sync(BAR_SW2, 32 * WS_GW);
                if (w == WS_GW && lane == 0) {
                    for (int jr = (j2 == 2 ? 0 : j2 - 1); jr <= j2 - 1; ++jr)
                        if (jr + NS < nit) issue(jr + NS);
                }
            };
            for (int base = 0; base < nit; base += 6) {
                if (base + 0 < nit) step2(std::integral_constant<int, 0>{}, base + 0);
                if (base + 1 < nit) step2(std::integral_constant<int, 1>{}, base + 1);
                if (base + 2 < nit) step2(std::integral_constant<int, 2>{}, base + 2);
                if (base + 3 < nit) step2(std::integral_constant<int, 3>{}, base + 3);
                if (base + 4 < nit) step2(std::integral_constant<int, 4>{}, base + 4);
                if (base + 5 < nit) step2(std::integral_constant<int, 5>{}, base + 5);
            }
        }
        return;
    }

    auto step = [&](auto Kc, int it) {
        constexpr int K = decltype(Kc)::value;      // it % 6
        if (role == 0) {
            constexpr int i3 = K % 3, m3 = (K + 2) % 3, mm3 = (K + 1) % 3, i2 = K % 2, m2 = (K + 1) % 2;
            const int j = it;
            if (j < nit) {
                if (PRO) {
                    if (j + 1 < nit) prolong(j + 1);   // visible to the group after this plane's barrier
                } else {
                    mbar_wait(&bar[j % NS], (j / NS) & 1);
                }
                const double *S = stage(j);
                plane_partials<true, SR>(S, S_UW, row0, lane, q[i3], f[i3], e[i2]);
                if (j >= 2) {   // sweep 1 at plane z0 - 3 + j on the 32 x 32 region
                    const int gz = z0 - 3 + j;
                    const unsigned in = ((unsigned)gz < (unsigned)n) ? inxy : 0u;
                    const double *Bp = S + W::UPL / 8 + row0 * S_BW + lane + 1;
                    double *Tp = Ts + i2 * (S_TPL / 8) + (row0 + 1) * S_TW + lane + 1;
#pragma unroll
                    for (int r = 0; r < SR; ++r) {
                        const double faces = f[m3][r] + (q[mm3][r] + q[i3][r]);
                        const double edges = e[m2][r] + (f[mm3][r] + f[i3][r]);
                        const double su = (c0 * q[m3][r] + c1 * faces) + c2 * edges;
                        const double t = q[m3][r] + wd * (Bp[r * S_BW] - su);
                        Tp[r * S_TW] = ((in >> r) & 1u) ? t : 0.0;
                    }
                }
            }
        } else if (role == 1) {
            constexpr int KJ = (K + 5) % 6;         // j2 % 6
            constexpr int i3 = KJ % 3, m3 = (KJ + 2) % 3, mm3 = (KJ + 1) % 3, i2 = KJ % 2, m2 = (KJ + 1) % 2;
            const int j2 = it - 1;
            if (j2 >= 2 && j2 < nit) {
                plane_partials<true, SR>(Ts + i2 * (S_TPL / 8), S_TW, row0, lane, q[i3], f[i3], e[i2]);
                if (j2 >= 4) {   // sweep 2 at plane z0 - 4 + j2 on the 30 x 30 tile, b from stage j2 - 1
                    const double *Bp = stage(j2 - 1) + W::UPL / 8 + row0 * S_BW + lane + 1;
                    double *op = optr + (long long)j2 * plane;
#pragma unroll
                    for (int r = 0; r < SR; ++r) {
                        const double faces = f[m3][r] + (q[mm3][r] + q[i3][r]);
                        const double edges = e[m2][r] + (f[mm3][r] + f[i3][r]);
                        const double su = (c0 * q[m3][r] + c1 * faces) + c2 * edges;
                        const double o = q[m3][r] + wd * (Bp[r * S_BW] - su);
                        if ((oks >> r) & 1u) *op = o;
                        op += pitch;
                    }
                }
            }
        }
        __syncthreads();
        // stage it - 2 is free (sweep 2 read its b): refill it with stage it - 2 + NS
        if (tid == 0) {
            const int jr = it - 2;
            if (jr >= 0 && jr + NS < nit) issue(jr + NS);
        }
    };
    for (int base = 0; base < niter; base += 6) {
        if (base + 0 < niter) step(std::integral_constant<int, 0>{}, base + 0);
        if (base + 1 < niter) step(std::integral_constant<int, 1>{}, base + 1);
        if (base + 2 < niter) step(std::integral_constant<int, 2>{}, base + 2);
        if (base + 3 < niter) step(std::integral_constant<int, 3>{}, base + 3);
        if (base + 4 < niter) step(std::integral_constant<int, 4>{}, base + 4);
        if (base + 5 < niter) step(std::integral_constant<int, 5>{}, base + 5);
    }
}

// ---------------------------------------------------------------------------------------------
// Defect + full-weighting restriction, one HBM pass (read u, b; write b_c), DESIGN.md §6.8.
// Coarse tile 15 x 15 x a coarse z chunk [K0, K1).  Fine defect region 31 x 31 at
// (2 I0, 2 J0), streamed over fine planes 2 K0 .. 2 K1; d(z) goes to a shared plane, coarse
// threads take its in-plane partials (face / edge / centre) and combine three planes.
// u box 36 x 34 at (2 I0 - 2, 2 J0 - 1); b box 32 x 32 at (2 I0, 2 J0).
// ---------------------------------------------------------------------------------------------
constexpr int R_CX = 15, R_CY = 15;
constexpr int R_UW = RW + 4, R_UH = RH + 2;
constexpr int R_BW = RW, R_BH = RH;
constexpr int R_DW = RW, R_DH = RH;
constexpr int R_NS = 4;
constexpr int R_UPL = a128(R_UW * R_UH * 8), R_BPL = a128(R_BW * R_BH * 8), R_DPL = a128(R_DW * R_DH * 8);
constexpr size_t R_SMEM = (size_t)R_NS * (R_UPL + R_BPL) + 2 * R_DPL + 8 * R_NS + 128;

__global__ void __launch_bounds__(NT, 1) k_restrict(const __grid_constant__ CUtensorMap tu,
                                                    const __grid_constant__ CUtensorMap tb,
                                                    double *__restrict__ bc, int nf, int nc, int pitch_c,
                                                    long long plane_c, SCoef c, int kc) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);   // stays a shared pointer
    double *Us = reinterpret_cast<double *>(sm);
    double *Bs = reinterpret_cast<double *>(sm + R_NS * R_UPL);
    double *Ds = reinterpret_cast<double *>(sm + R_NS * (R_UPL + R_BPL));
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + R_NS * (R_UPL + R_BPL) + 2 * R_DPL);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int I0 = blockIdx.x * R_CX, J0 = blockIdx.y * R_CY;
    const int K0 = blockIdx.z * kc, K1 = min(K0 + kc, nc);
    const int fx0 = 2 * I0, fy0 = 2 * J0;
    const int nit = 2 * (K1 - K0) + 3;     // u planes 2K0-1 .. 2K1+1
    auto issue = [&](int it) {
        const int s = it % R_NS, p = 2 * K0 - 1 + it;
        mbar_expect_tx(&bar[s], (R_UW * R_UH + R_BW * R_BH) * 8);
        tma_load_3d(Us + s * (R_UPL / 8), &tu, fx0 - 2, fy0 - 1, p, &bar[s]);
        tma_load_3d(Bs + s * (R_BPL / 8), &tb, fx0, fy0, p - 1, &bar[s]);
    };
    if (tid == 0) {
        tma_prefetch_desc(&tu);
        tma_prefetch_desc(&tb);
        for (int s = 0; s < R_NS; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int it = 0; it < R_NS && it < nit; ++it) issue(it);

    const double c0 = c.c0, c1 = c.c1, c2 = c.c2;
    // coarse role: 16 x 16 thread grid over the 15 x 15 coarse tile (half-warp = one coarse row).
    // The defect plane is stored de-interleaved in x -- odd fine columns (the coarse points) at
    // [0, 16), even ones at [16, 32) -- so a coarse row's centre / left / right loads are unit
    // stride (2 shared wavefronts per warp load instead of the 4-6 of the stride-2 layout).
    const int ci = tid & 15, cj = tid >> 4;
    const bool crole = ci < R_CX && cj < R_CY;
    const int pcol = (lane & 1) ? (lane >> 1) : 16 + (lane >> 1);   // this lane's column in the d plane
    const int gI = I0 + ci, gJ = J0 + cj;
    const bool cout_ok = crole && gI < nc && gJ < nc;
    const int dy = 2 * cj + 1;
    double fdl = 0, edl = 0, dcl = 0, fdm = 0, edm = 0, dcm = 0;   // partials at planes 2K (lower), 2K+1 (mid)

    // register rings (plane it at slot it % 3 for q, f and it % 2 for e); the z loop is unrolled by
    // 6 so every slot index is a compile-time constant and no ring value is moved
    double qr[3][R], fr[3][R], er[2][R];
#pragma unroll
    for (int r = 0; r < R; ++r) { qr[0][r] = qr[1][r] = qr[2][r] = fr[0][r] = fr[1][r] = fr[2][r] = er[0][r] = er[1][r] = 0.0; }
    auto step = [&](auto Kc, int it) {
        constexpr int KK = decltype(Kc)::value;
        constexpr int i3 = KK % 3, m3 = (KK + 2) % 3, mm3 = (KK + 1) % 3, i2 = KK % 2, m2 = (KK + 1) % 2;
        const int s = it % R_NS;
        mbar_wait(&bar[s], (it / R_NS) & 1);
        plane_partials<true>(Us + s * (R_UPL / 8), R_UW, R * w, lane + 1, qr[i3], fr[i3], er[i2]);
        const bool dd = it >= 2;     // defect at fine plane p-1
        double *D = Ds + (KK & 1) * (R_DPL / 8);   // == it & 1 (the unrolled base is a multiple of 6)
        if (dd) {
            const double *Bp = Bs + s * (R_BPL / 8);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double faces = fr[m3][r] + (qr[mm3][r] + qr[i3][r]);
                const double edges = er[m2][r] + (fr[mm3][r] + fr[i3][r]);
                const double su = (c0 * qr[m3][r] + c1 * faces) + c2 * edges;
                D[(R * w + r) * R_DW + pcol] = Bp[(R * w + r) * R_BW + lane] - su;
            }
        }
        __syncthreads();
        if (tid == 0 && it + R_NS < nit) issue(it + R_NS);
        if (dd && crole) {
            const int j = it - 2;    // fine plane 2K0 + j
            // fine column dx = 2 ci + 1 sits at ci, its neighbours 2 ci and 2 ci + 2 at 16 + ci, 17 + ci
            const double *d0 = D + (dy - 1) * R_DW + ci, *d1 = d0 + R_DW, *d2 = d1 + R_DW;
            const double rd0 = d0[16] + d0[17], rd1 = d1[16] + d1[17], rd2 = d2[16] + d2[17];
            const double fd = rd1 + (d0[0] + d2[0]);
            const double ed = rd0 + rd2;
            const double dc = d1[0];
            if (j & 1) {
                fdm = fd; edm = ed; dcm = dc;
            } else {
                if (j >= 2) {
                    const double F = fdm + (dcl + dc);
                    const double E = edm + (fdl + fd);
                    const double C = edl + ed;
                    const int K = K0 + j / 2 - 1;
                    if (cout_ok) bc[(long long)K * plane_c + (long long)gJ * pitch_c + gI] =
                        ((8.0 * dcm + 4.0 * F) + (2.0 * E + C)) * 0.015625;
                }
                fdl = fd; edl = ed; dcl = dc;
            }
        }
    };
    for (int base = 0; base < nit; base += 6) {
        step(std::integral_constant<int, 0>{}, base);
        if (base + 1 < nit) step(std::integral_constant<int, 1>{}, base + 1);
        if (base + 2 < nit) step(std::integral_constant<int, 2>{}, base + 2);
        if (base + 3 < nit) step(std::integral_constant<int, 3>{}, base + 3);
        if (base + 4 < nit) step(std::integral_constant<int, 4>{}, base + 4);
        if (base + 5 < nit) step(std::integral_constant<int, 5>{}, base + 5);
    }
}

// ---------------------------------------------------------------------------------------------
// Trilinear prolongation + correction u += P e, two fine points (2t, 2t+1) per thread with
// 16-byte accesses on u; coarse values through the read-only path (L1/L2), DESIGN.md §6.9.
// Sums nest x, then y, then z; one multiply by 0.5^(#even axes).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_prolong(double *__restrict__ u, int nf, int pitch_f, long long plane_f,
                                                 const double *__restrict__ e, int nc, int pitch_c,
                                                 long long plane_c) {
    // two fine rows (y0, y0 + 1) per thread: both 16-byte u loads are issued before either update
    // (memory-level parallelism); the per-point expressions are unchanged
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int y0 = 2 * blockIdx.y, z = blockIdx.z;
    const int x = 2 * t;
    if (x >= nf) return;
    auto E = [&](int X, int Y, int Z) -> double {
        return (X >= 0 && X < nc && Y >= 0 && Y < nc && Z >= 0 && Z < nc)
                   ? __ldg(e + (long long)Z * plane_c + (long long)Y * pitch_c + X)
                   : 0.0;
    };
    const bool ze = !(z & 1);
    const int Za = ze ? z / 2 - 1 : (z - 1) / 2, Zb = z / 2;
    const bool pair = x + 1 < nf;
    double2 v[2];
    double *row[2];
    bool rin[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int y = y0 + q;
        rin[q] = y < nf;
        row[q] = u + (long long)z * plane_f + (long long)y * pitch_f;
        if (rin[q]) {
            if (pair) v[q] = *reinterpret_cast<const double2 *>(row[q] + x);
            else v[q].x = row[q][x];
        }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (!rin[q]) continue;
        const int y = y0 + q;
        const bool ye = !(y & 1);
        const int Ya = ye ? y / 2 - 1 : (y - 1) / 2, Yb = y / 2;
        auto sy = [&](int Z, double &se, double &so) {
            double sea = E(t - 1, Ya, Z) + E(t, Ya, Z), soa = E(t, Ya, Z);
            if (ye) {
                double seb = E(t - 1, Yb, Z) + E(t, Yb, Z), sob = E(t, Yb, Z);
                se = sea + seb; so = soa + sob;
            } else {
                se = sea; so = soa;
            }
        };
        double se, so;
        sy(Za, se, so);
        if (ze) {
            double se2, so2;
            sy(Zb, se2, so2);
            se = se + se2; so = so + so2;
        }
        double w = (ye ? 0.5 : 1.0) * (ze ? 0.5 : 1.0);
        double we = w * 0.5;   // the even column also averages in x
        if (pair) {
            v[q].x = v[q].x + se * we;
            v[q].y = v[q].y + so * w;
            *reinterpret_cast<double2 *>(row[q] + x) = v[q];
        } else {
            row[q][x] = v[q].x + se * we;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// B a (+|-) L c streaming kernel: the RHS of Eq. (5) (b = B v + L w) and the
// weighted SDC residual of one node (r~ = B p - L z, §4.5), DESIGN.md §6.10.  Per plane p, the K
// input fields arrive by TMA (34 x RH boxes at (x0-2, y0-1)); every thread forms the pointwise
// pair (a, c) at its RR points of the (30 + 2) x RH region, writes it to shared planes, then
// takes in-plane partials (a: centre + faces, c: centre + faces + edges) into register rings and
// emits the tile (30 x (RH-2)) at plane p-1.  f^E: 0 none, 1 u - u^3, 2 G cos t, 3 stored F
// fields (CD4 advection, computed once per new node field by k_fe_cd4).
// ---------------------------------------------------------------------------------------------
constexpr int BL_MAXF = 2 * ISDC_MAXM + 2;
constexpr int BL_MAXNM = 4;        // outputs (residual nodes) per pass
struct BLMaps {
    CUtensorMap m[BL_MAXF];
};
struct BLArgs {
    int K;                         // fields per plane
    int M;                         // nodes
    int mnode[BL_MAXNM];           // RHS: substep m (0-based); residual: the pass's nodes m (1..M-1)
    int iu0, iun, iuG, iF0, iFn;   // field slots: old/current u_j at iu0+j, u_m^{k+1} at iun, G at iuG,
                                   // stored F_j at iF0+j, F(u_m^{k+1}) at iFn
    // FE == 4 (RHS from fold fields, CD4): slots of u_{m+1}^old, F_m^old, WB_m, FA_m
    int iuo1, ifo, iwb, ifa;
    // residual passes may also store the RHS folds of the next sweep:
    // FA_q = fold_j (dt S_qj) F_j, WB_q = fold_j (nu dt S_qj) u_j, q = qnode[k], k < nfold
    int nfold, qnode[BL_MAXNM];
    double sa[BL_MAXNM][ISDC_MAXM], sb[BL_MAXNM][ISDC_MAXM];
    double fgm[BL_MAXNM];          // gamma_q: WB_q stores fold_j (nu dt S_qj) u_j - gamma_q u_{q+1}
    double *fa_out[BL_MAXNM], *wb_out[BL_MAXNM];
    const double *ct;              // device cos(t_j)
    double dtm, gm;                // RHS: dt*dtau_m, nu*dt*dtau_m
    double a[BL_MAXNM][ISDC_MAXM], beta[BL_MAXNM][ISDC_MAXM];   // RHS: dt*S_mj, nu*dt*S_mj;
                                                                // residual: dt*Q_mj, nu*dt*Q_mj
    BLConst bl;
    int n, pitch;
    long long plane;
    int zc;
    int sh;                        // shifted tiling (see WSCfg): the region starts at the tile origin, boundary
                                   // rim points are outputs, ceil((n - 2) / T) tiles per axis
    double *out;                   // RHS: b (pitched); residual: unused
    unsigned long long *slot[BL_MAXNM];   // max |out| per output (RHS: optional, residual: required)
};

template <int RR, int NWW = NW>
struct BLShape {
    static constexpr int RH = NWW * RR;                // region rows
    static constexpr int TX = RW - 2, TY = RH - 2;     // output tile
    static constexpr int FW = RW + 2, FH = RH;         // input box 34 x RH at (x0-2, y0-1)
    static constexpr int PW = RW + 2, PH = RH + 2;     // a / c planes with a pad ring
    static constexpr int FPL = a128(FW * FH * 8), PPL = a128(PW * PH * 8);
    static size_t smem(int K, int ns, int nm) {
        return (size_t)ns * K * FPL + 4 * (size_t)nm * PPL + 8 * 8 + 128;
    }
};

template <int RR>
struct BLRegs {
    double aq[3][RR], af[3][RR];               // a: centre, faces (by iteration mod 3)
    double cq[3][RR], cf[3][RR], ce[2][RR];    // c: centre, faces, edges
};

// pointwise (a, c) of output k at one point from the stage fields at smem offset `o`
// (DESIGN.md §4.4 RHS, §4.5 residual)
template <int FE, int MODE>
__device__ __forceinline__ void bl_point(const BLArgs &A, int k, const double *F, int fpl, int o, double &av,
                                         double &cv) {
    const int M = A.M, m = A.mnode[k];
    const double *a = A.a[k], *beta = A.beta[k];
    auto fld = [&](int slot) -> double { return F[slot * fpl + o]; };
    if (MODE == 0) {   // RHS substep m: a = v, c = w
        double acc = beta[0] * fld(A.iu0);
#pragma unroll
        for (int j = 1; j < ISDC_MAXM; ++j)
            if (j < M) acc = acc + beta[j] * fld(A.iu0 + j);
        cv = acc - A.gm * fld(A.iu0 + m + 1);
        const double un = fld(A.iun);
        if (FE == 0) {
            av = un;
        } else {
            double fa, fn, fo;
            if (FE == 1) {
                double uj = fld(A.iu0);
                fa = a[0] * (uj - (uj * uj) * uj);
#pragma unroll
                for (int j = 1; j < ISDC_MAXM; ++j)
                    if (j < M) { uj = fld(A.iu0 + j); fa = fa + a[j] * (uj - (uj * uj) * uj); }
                const double uo = fld(A.iu0 + m);
                fn = un - (un * un) * un;
                fo = uo - (uo * uo) * uo;
            } else if (FE == 2) {
                const double g = fld(A.iuG);
                fa = a[0] * (g * A.ct[0]);
#pragma unroll
                for (int j = 1; j < ISDC_MAXM; ++j)
                    if (j < M) fa = fa + a[j] * (g * A.ct[j]);
                fn = g * A.ct[m];
                fo = g * A.ct[m];
            } else {
                fa = a[0] * fld(A.iF0);
#pragma unroll
                for (int j = 1; j < ISDC_MAXM; ++j)
                    if (j < M) fa = fa + a[j] * fld(A.iF0 + j);
                fn = fld(A.iFn);
                fo = fld(A.iF0 + m);
            }
            av = (un + A.dtm * (fn - fo)) + fa;
        }
    } else if (MODE == 2) {   // RHS from stored folds (FE = CD4): the same expression trees
        cv = fld(A.iwb);          // = fold - gamma_m u_{m+1}^k, formed by the residual pass
        av = (fld(A.iun) + A.dtm * (fld(A.iFn) - fld(A.ifo))) + fld(A.ifa);
    } else {           // residual node m: a = p, c = z
        double diff = fld(A.iu0 + m) - fld(A.iu0);
        if (FE != 0) {
            double fa;
            if (FE == 1) {
                double uj = fld(A.iu0);
                fa = a[0] * (uj - (uj * uj) * uj);
#pragma unroll
                for (int j = 1; j < ISDC_MAXM; ++j)
                    if (j < M) { uj = fld(A.iu0 + j); fa = fa + a[j] * (uj - (uj * uj) * uj); }
            } else if (FE == 2) {
                const double g = fld(A.iuG);
                fa = a[0] * (g * A.ct[0]);
#pragma unroll
                for (int j = 1; j < ISDC_MAXM; ++j)
                    if (j < M) fa = fa + a[j] * (g * A.ct[j]);
            } else {
                fa = a[0] * fld(A.iF0);
#pragma unroll
                for (int j = 1; j < ISDC_MAXM; ++j)
                    if (j < M) fa = fa + a[j] * fld(A.iF0 + j);
            }
            diff = diff - fa;
        }
        av = diff;
        double acc = beta[0] * fld(A.iu0);
#pragma unroll
        for (int j = 1; j < ISDC_MAXM; ++j)
            if (j < M) acc = acc + beta[j] * fld(A.iu0 + j);
        cv = acc;
    }
}

// Residual pass at one point (MODE 1, f^E none or stored CD4): every node field u_j and F_j is read
// from the stage ONCE and streamed, in ascending j, into the left folds of all NM nodes and of the
// next sweep's RHS folds -- the same trees as bl_point + the fold code (each accumulator is
// c_0 x_0, then acc + c_j x_j for j = 1..M-1), with M loads per field instead of one per use.
template <int FE, int NM>
__device__ __forceinline__ void bl_resid_point(const BLArgs &A, const double *F, int fpl, int o, bool folds,
                                               double (&av)[NM], double (&cv)[NM], double (&fo)[NM],
                                               double (&wo)[NM]) {
    const int M = A.M;
    const double u0 = F[A.iu0 * fpl + o];
    const double f0 = (FE == 3) ? F[A.iF0 * fpl + o] : 0.0;
    double um[NM], fa[NM], uq1[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) {
        um[k] = u0;
        uq1[k] = u0;
        if (FE == 3) fa[k] = A.a[k][0] * f0;
        cv[k] = A.beta[k][0] * u0;
        if (FE == 3 && folds) { fo[k] = A.sa[k][0] * f0; wo[k] = A.sb[k][0] * u0; }
    }
#pragma unroll
    for (int j = 1; j < ISDC_MAXM; ++j) {
        if (j < M) {
            const double uj = F[(A.iu0 + j) * fpl + o];
            const double Fj = (FE == 3) ? F[(A.iF0 + j) * fpl + o] : 0.0;
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                if (j == A.mnode[k]) um[k] = uj;
                if (j == A.qnode[k] + 1) uq1[k] = uj;
                if (FE == 3) fa[k] = fa[k] + A.a[k][j] * Fj;
                cv[k] = cv[k] + A.beta[k][j] * uj;
                if (FE == 3 && folds) { fo[k] = fo[k] + A.sa[k][j] * Fj; wo[k] = wo[k] + A.sb[k][j] * uj; }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < NM; ++k) {
        double diff = um[k] - u0;
        if (FE == 3) diff = diff - fa[k];
        av[k] = diff;
        if (FE == 3 && folds) wo[k] = wo[k] - A.fgm[k] * uq1[k];   // the RHS's w = acc - gamma u_{m+1}
    }
}

// NM outputs per pass (RHS: 1; residual: nodes per pass).  Registers: 14 * RR * NM doubles of rings.
// NWW warps (region rows NWW * RR).
template <int FE, int MODE, int RR, int NM, int NWW = NW>
__global__ void __launch_bounds__(32 * NWW, 1) k_bl(const __grid_constant__ BLMaps maps, const BLArgs A, int ns) {
    using SH = BLShape<RR, NWW>;
    constexpr bool RHS = MODE != 1;   // MODE 0: RHS, 1: residual, 2: RHS from stored folds
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const int K = A.K;
    double *Fs = reinterpret_cast<double *>(sm);                                   // ns stages x K boxes
    double *Ps = reinterpret_cast<double *>(sm + (size_t)ns * K * SH::FPL);        // [buf][k][a|c]
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)ns * K * SH::FPL + 4 * NM * SH::PPL);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int n = A.n;
    const int x0 = blockIdx.x * SH::TX, y0 = blockIdx.y * SH::TY;
    const int z0 = blockIdx.z * A.zc, z1 = min(z0 + A.zc, n);
    const int nit = z1 - z0 + 2;              // ingest planes z0-1 .. z1
    const bool sh = A.sh != 0;
    auto issue = [&](int it) {
        const int s = it % ns, p = z0 - 1 + it;
        mbar_expect_tx(&bar[s], K * SH::FW * SH::FH * 8);
        for (int k = 0; k < K; ++k)
            tma_load_3d(Fs + ((size_t)s * K + k) * (SH::FPL / 8), &maps.m[k], sh ? x0 : x0 - 2, sh ? y0 : y0 - 1, p,
                        &bar[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < ns; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    if (sh)   // the pad ring of the (a, c) planes is the zero outside the domain read by the boundary outputs
        for (int q = tid; q < 4 * NM * (SH::PPL / 8); q += 32 * NWW) Ps[q] = 0.0;
    __syncthreads();
    if (tid == 0)
        for (int it = 0; it < ns && it < nit; ++it) issue(it);

    const int lx = sh ? lane : lane - 1, ly0 = sh ? RR * w : RR * w - 1;
    const int gx = x0 + lx;
    const bool xin = gx >= 0 && gx < n;
    const bool xout = sh ? (gx < n && (lane >= 1 || gx == 0) && (lane <= SH::TX || gx == n - 1))
                         : (lx >= 0 && lx < SH::TX && gx < n);
    unsigned inxy = 0u, oks = 0u;
#pragma unroll
    for (int r = 0; r < RR; ++r) {
        const int ly = ly0 + r, gy = y0 + ly;
        if (xin && gy >= 0 && gy < n) inxy |= 1u << r;
        const bool yout = sh ? (gy < n && (ly >= 1 || gy == 0) && (ly <= SH::TY || gy == n - 1))
                             : (ly >= 0 && ly < SH::TY && gy < n);
        if (xout && yout) oks |= 1u << r;
    }
    const BLConst c = A.bl;
    double vmax[NM];
    BLRegs<RR> G[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) vmax[k] = 0.0;
    double *orow = RHS ? A.out + (long long)(z0 - 2) * A.plane + (long long)(y0 + ly0) * A.pitch + gx : nullptr;
    auto step = [&](auto Kc, int it) {
        constexpr int Kk = decltype(Kc)::value;
        constexpr int i3 = Kk % 3, m3 = (Kk + 2) % 3, mm3 = (Kk + 1) % 3;
        constexpr int i2 = Kk % 2, m2 = (Kk + 1) % 2;
        const int s = it % ns, p = z0 - 1 + it;
        mbar_wait(&bar[s], (it / ns) & 1);
        const unsigned in = ((unsigned)p < (unsigned)n) ? inxy : 0u;
        const double *F = Fs + (size_t)s * K * (SH::FPL / 8);
        const int o0 = (RR * w) * SH::FW + lane + (sh ? 0 : 1);
        const int po = (RR * w + 1) * SH::PW + lane + 1;
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            if constexpr (MODE == 1 && (FE == 0 || FE == 3)) {
                // residual: one read of every stage field per point (bl_resid_point)
                double av[NM], cv[NM], fo[NM], wo[NM];
                const bool folds = FE == 3 && A.nfold > 0;
                if ((in >> r) & 1u) {
                    bl_resid_point<FE, NM>(A, F, SH::FPL / 8, o0 + r * SH::FW, folds, av, cv, fo, wo);
                } else {
#pragma unroll
                    for (int k = 0; k < NM; ++k) { av[k] = 0.0; cv[k] = 0.0; }
                }
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    double *Pa = Ps + ((i2 * NM + k) * 2) * (SH::PPL / 8);
                    Pa[po + r * SH::PW] = av[k];
                    Pa[SH::PPL / 8 + po + r * SH::PW] = cv[k];
                }
                if (folds && ((oks >> r) & 1u) && p >= z0 && p < z1) {
                    const long long gofs = (long long)p * A.plane + (long long)(y0 + ly0 + r) * A.pitch + gx;
#pragma unroll
                    for (int k = 0; k < NM; ++k) {
                        if (k >= A.nfold) break;
                        A.fa_out[k][gofs] = fo[k];
                        A.wb_out[k][gofs] = wo[k];
                    }
                }
                continue;
            }
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                double av = 0.0, cv = 0.0;
                if ((in >> r) & 1u) bl_point<FE, MODE>(A, k, F, SH::FPL / 8, o0 + r * SH::FW, av, cv);
                double *Pa = Ps + ((i2 * NM + k) * 2) * (SH::PPL / 8);
                Pa[po + r * SH::PW] = av;
                Pa[SH::PPL / 8 + po + r * SH::PW] = cv;
            }
        }
        __syncthreads();
        if (tid == 0 && it + ns < nit) issue(it + ns);
#pragma unroll
        for (int k = 0; k < NM; ++k) {
            const double *Pa = Ps + ((i2 * NM + k) * 2) * (SH::PPL / 8), *Pc = Pa + SH::PPL / 8;
            double dummy[RR];
            plane_partials<false, RR>(Pa, SH::PW, RR * w, lane, G[k].aq[i3], G[k].af[i3], dummy);
            plane_partials<true, RR>(Pc, SH::PW, RR * w, lane, G[k].cq[i3], G[k].cf[i3], G[k].ce[i2]);
        }
        if (it >= 2) {   // output plane p-1
            double *op = RHS ? orow + (long long)it * A.plane : nullptr;
#pragma unroll
            for (int r = 0; r < RR; ++r) {
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    const BLRegs<RR> &g = G[k];
                    const double fa_ = g.af[m3][r] + (g.aq[mm3][r] + g.aq[i3][r]);
                    const double fc_ = g.cf[m3][r] + (g.cq[mm3][r] + g.cq[i3][r]);
                    const double ec_ = g.ce[m2][r] + (g.cf[mm3][r] + g.cf[i3][r]);
                    const double Ba = c.kB0 * g.aq[m3][r] + c.kB1 * fa_;
                    const double Lc = (c.kL0 * g.cq[m3][r] + c.kL1 * fc_) + c.kL2 * ec_;
                    const double val = RHS ? Ba + Lc : Ba - Lc;
                    if ((oks >> r) & 1u) {
                        if (RHS) op[r * A.pitch] = val;
                        vmax[k] = amax(vmax[k], fabs(val));
                    }
                }
            }
        }
    };
    for (int base = 0; base < nit; base += 6) {
        if (base + 0 < nit) step(std::integral_constant<int, 0>{}, base + 0);
        if (base + 1 < nit) step(std::integral_constant<int, 1>{}, base + 1);
        if (base + 2 < nit) step(std::integral_constant<int, 2>{}, base + 2);
        if (base + 3 < nit) step(std::integral_constant<int, 3>{}, base + 3);
        if (base + 4 < nit) step(std::integral_constant<int, 4>{}, base + 4);
        if (base + 5 < nit) step(std::integral_constant<int, 5>{}, base + 5);
    }
#pragma unroll
    for (int k = 0; k < NM; ++k)
        if (A.slot[k]) { block_max_to(A.slot[k], vmax[k]); __syncthreads(); }
}

// ---------------------------------------------------------------------------------------------
// Weighted SDC residual of all four nodes of M = 5 (r~_m = B p_m - L z_m, m = 1..4)
// and, for stored-f^E CD4, the next sweep's RHS folds (FA_q, WB_q, q = 0..3, §6.12) in ONE z-stream
// pass: every node field u_j (and F_j) is read from HBM once per sweep instead of
// once per two-node pass.  Warp-specialised: R4_PW producer warps form the pointwise (p_m, z_m) of
// all four nodes and the folds from the TMA-staged planes (bl_resid_point: one shared load per input
// field and point), store them to double-buffered shared planes and the folds to global memory;
// 4 x R4_WG consumer warps -- one group per node -- take in-plane partials into register rings and
// emit |r~_m| at plane p-1 (the trees of k_bl MODE 1).  Producers run one plane ahead of the
// consumers; one block barrier per plane.  Region 32 x R4_RH (tile 30 x (R4_RH - 2) + halo 1).
// ---------------------------------------------------------------------------------------------
constexpr int R4_WG = 2, R4_RR = 4, R4_RH = R4_WG * R4_RR;   // consumer warps per node, rows per thread
constexpr int R4_PW = 8;                                     // producer warps (two per SM sub-partition)
constexpr int R4_PREG = 104, R4_CREG = 152;                  // setmaxnreg split (8 x 32 x (104 + 152) = 64 K)
constexpr int R4_NT = 32 * (4 * R4_WG + R4_PW);
struct R4Shape {
    static constexpr int RH = R4_RH, TX = RW - 2, TY = R4_RH - 2;
    static constexpr int FW = RW + 2, FH = R4_RH;              // input box 34 x RH at (x0-2, y0-1)
    static constexpr int PW = RW + 2, PH = R4_RH + 2;          // p / z planes with a pad ring
    static constexpr int FPL = a128(FW * FH * 8), PPL = a128(PW * PH * 8);
    static size_t smem(int K, int ns) { return (size_t)ns * K * FPL + 2 * 8 * (size_t)PPL + 8 * 8 + 128; }
};

// Pointwise part of the residual pass for M = 5 at one point, with every node index fixed at compile
// time (the trees of bl_resid_point: each accumulator is c_0 x_0, then acc + c_j x_j, j ascending).
// Node k = 0..3 is residual node m = k + 1; its fold is RHS node q = k (u_{q+1} = u_{k+1}).
template <int FE>
__device__ __forceinline__ void r4_point(const BLArgs &A, const double *F, int fpl, int o, bool folds, double (&av)[4],
                                         double (&cv)[4], double (&fo)[4], double (&wo)[4]) {
    double u[5], f[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) u[j] = F[(A.iu0 + j) * fpl + o];
    if (FE == 3) {
#pragma unroll
        for (int j = 0; j < 5; ++j) f[j] = F[(A.iF0 + j) * fpl + o];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        double c = A.beta[k][0] * u[0];
#pragma unroll
        for (int j = 1; j < 5; ++j) c = c + A.beta[k][j] * u[j];
        cv[k] = c;
        double diff = u[k + 1] - u[0];
        if (FE == 3) {
            double fa = A.a[k][0] * f[0];
#pragma unroll
            for (int j = 1; j < 5; ++j) fa = fa + A.a[k][j] * f[j];
            diff = diff - fa;
            if (folds) {
                double x = A.sa[k][0] * f[0], y = A.sb[k][0] * u[0];
#pragma unroll
                for (int j = 1; j < 5; ++j) { x = x + A.sa[k][j] * f[j]; y = y + A.sb[k][j] * u[j]; }
                fo[k] = x;
                wo[k] = y - A.fgm[k] * u[k + 1];
            }
        }
        av[k] = diff;
    }
}

template <int FE>
__global__ void __launch_bounds__(R4_NT, 1) k_resid4(const __grid_constant__ BLMaps maps, const BLArgs A, int ns) {
    using SH = R4Shape;
    constexpr int NM = 4, RR = R4_RR;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const int K = A.K;
    double *Fs = reinterpret_cast<double *>(sm);                                   // ns stages x K boxes
    double *Ps = reinterpret_cast<double *>(sm + (size_t)ns * K * SH::FPL);        // [buf][node][p|z]
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)ns * K * SH::FPL + 16 * SH::PPL);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int n = A.n;
    const int x0 = blockIdx.x * SH::TX, y0 = blockIdx.y * SH::TY;
    const int z0 = blockIdx.z * A.zc, z1 = min(z0 + A.zc, n);
    const int nit = z1 - z0 + 2;              // ingest planes z0-1 .. z1
    constexpr int PROD0 = 4 * R4_WG;          // first producer warp
    const bool producer = w >= PROD0;
    const bool sh = A.sh != 0;
    const int sh1 = sh ? 0 : 1;               // region coordinate -> tile-origin offset
    auto issue = [&](int it) {
        const int s = it % ns, p = z0 - 1 + it;
        mbar_expect_tx(&bar[s], K * SH::FW * SH::FH * 8);
        for (int k = 0; k < K; ++k)
            tma_load_3d(Fs + ((size_t)s * K + k) * (SH::FPL / 8), &maps.m[k], sh ? x0 : x0 - 2, sh ? y0 : y0 - 1, p,
                        &bar[s]);
    };
    const int ptid = tid - 32 * PROD0;        // producer thread index
    if (ptid == 0) {
        for (int s = 0; s < ns; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
        for (int s = 0; s < ns && s < nit; ++s) issue(s);
    }
    if (sh)   // zero pad ring of the p / z planes (read by the boundary outputs)
        for (int q = tid; q < 16 * (SH::PPL / 8); q += R4_NT) Ps[q] = 0.0;
    __syncthreads();
    const bool folds = FE == 3 && A.nfold > 0;
    // the two roles run separate loops (so the consumers' rings are not live in the producers' code)
    // that meet at one named barrier per plane
    if (producer) {
        // warp-specialised register split (sm_90+): the producer warpgroups give registers to the
        // consumer warpgroups, whose stencil rings (13 x R4_RR doubles per thread) need ~140
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(R4_PREG) : "memory");
        for (int it = 0; it < nit; ++it) {
            const int p = z0 - 1 + it, s = it % ns;
            mbar_wait(&bar[s], (it / ns) & 1);
            const double *F = Fs + (size_t)s * K * (SH::FPL / 8);
            double *Pb = Ps + (it & 1) * 8 * (SH::PPL / 8);
            const bool zin = (unsigned)p < (unsigned)n, zout = p >= z0 && p < z1;
            for (int q = ptid; q < RW * SH::RH; q += 32 * R4_PW) {
                const int col = q & 31, row = q >> 5;        // region column / row
                const int px = x0 - sh1 + col, py = y0 - sh1 + row;
                double av[NM], cv[NM], fo[NM], wo[NM];
                // the folds only at the tile's own points (they are stored, not stencilled)
                const bool own = sh ? (px < n && (col >= 1 || px == 0) && (col <= SH::TX || px == n - 1) && py < n &&
                                       (row >= 1 || py == 0) && (row <= SH::TY || py == n - 1))
                                    : (col >= 1 && col - 1 < SH::TX && px < n && row >= 1 && row - 1 < SH::TY && py < n);
                const bool fpt = folds && zout && own;
                if (zin && (unsigned)px < (unsigned)n && (unsigned)py < (unsigned)n) {
                    r4_point<FE>(A, F, SH::FPL / 8, row * SH::FW + col + sh1, fpt, av, cv, fo, wo);
                } else {
#pragma unroll
                    for (int k = 0; k < NM; ++k) { av[k] = 0.0; cv[k] = 0.0; }
                }
                const int po = (row + 1) * SH::PW + col + 1;
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    Pb[(2 * k) * (SH::PPL / 8) + po] = av[k];
                    Pb[(2 * k + 1) * (SH::PPL / 8) + po] = cv[k];
                }
                if (fpt) {
                    const long long gofs = (long long)p * A.plane + (long long)py * A.pitch + px;
#pragma unroll
                    for (int k = 0; k < NM; ++k) {
                        A.fa_out[k][gofs] = fo[k];
                        A.wb_out[k][gofs] = wo[k];
                    }
                }
            }
            named_bar_sync(1, R4_NT);
            if (ptid == 0 && it + ns < nit) issue(it + ns);   // the producers have consumed stage it % ns
        }
        return;
    }
    // consumer role: node kc = w / R4_WG, rows RR*wi .. RR*wi+RR-1 of the region
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(R4_CREG) : "memory");
    const int kc = w / R4_WG, wi = w % R4_WG;
    const int gx = x0 + lane - sh1;
    const bool xout = sh ? (gx < n && (lane >= 1 || gx == 0) && (lane <= SH::TX || gx == n - 1))
                         : (lane >= 1 && lane - 1 < SH::TX && gx < n);
    unsigned oks = 0u;
#pragma unroll
    for (int r = 0; r < RR; ++r) {
        const int ly = RR * wi + r - sh1, gy = y0 + ly;
        const bool yout = sh ? (gy < n && (ly >= 1 || gy == 0) && (ly <= SH::TY || gy == n - 1))
                             : (ly >= 0 && ly < SH::TY && gy < n);
        if (xout && yout) oks |= 1u << r;
    }
    const BLConst c = A.bl;
    double vmax = 0.0;
    double aq[3][RR], af[2][RR], cq[3][RR], cf[3][RR], ce[2][RR];
    auto step = [&](auto Kc, int it) {
        constexpr int Kk = decltype(Kc)::value;
        constexpr int i3 = Kk % 3, m3 = (Kk + 2) % 3, mm3 = (Kk + 1) % 3;
        constexpr int i2 = Kk % 2, m2 = (Kk + 1) % 2;
        named_bar_sync(1, R4_NT);
        const double *Pa = Ps + (i2 * 8 + 2 * kc) * (SH::PPL / 8), *Pc = Pa + SH::PPL / 8;
        double dummy[RR];
        plane_partials<false, RR>(Pa, SH::PW, RR * wi, lane, aq[i3], af[i2], dummy);
        plane_partials<true, RR>(Pc, SH::PW, RR * wi, lane, cq[i3], cf[i3], ce[i2]);
        if (it >= 2) {   // output plane p-1
#pragma unroll
            for (int r = 0; r < RR; ++r) {
                const double fa_ = af[m2][r] + (aq[mm3][r] + aq[i3][r]);
                const double fc_ = cf[m3][r] + (cq[mm3][r] + cq[i3][r]);
                const double ec_ = ce[m2][r] + (cf[mm3][r] + cf[i3][r]);
                const double Ba = c.kB0 * aq[m3][r] + c.kB1 * fa_;
                const double Lc = (c.kL0 * cq[m3][r] + c.kL1 * fc_) + c.kL2 * ec_;
                if ((oks >> r) & 1u) vmax = amax(vmax, fabs(Ba - Lc));
            }
        }
    };
    for (int base = 0; base < nit; base += 6) {
        if (base + 0 < nit) step(std::integral_constant<int, 0>{}, base + 0);
        if (base + 1 < nit) step(std::integral_constant<int, 1>{}, base + 1);
        if (base + 2 < nit) step(std::integral_constant<int, 2>{}, base + 2);
        if (base + 3 < nit) step(std::integral_constant<int, 3>{}, base + 3);
        if (base + 4 < nit) step(std::integral_constant<int, 4>{}, base + 4);
        if (base + 5 < nit) step(std::integral_constant<int, 5>{}, base + 5);
    }
    // one atomic per consumer warp into its node's slot
    const unsigned long long v = warp_max_u64((unsigned long long)__double_as_longlong(vmax));
    if (lane == 0 && v) atomicMax(A.slot[kc], v);
}

// ---------------------------------------------------------------------------------------------
// f^E = -a . grad u with CD4 differences and zero ghosts, stored once per new
// node field so that the RHS / residual kernels read it pointwise.  32 x 32 tile, z-streaming
// with a 5-plane ring of 36 x 36 boxes at (x0-2, y0-2).  DESIGN.md §6.11.
// ---------------------------------------------------------------------------------------------
constexpr int FE_W = RW + 4, FE_H = RH + 4;
constexpr int FE_NS = 8;   // ring: 3 planes in use (arrival .. centre) + 5 in flight
constexpr int FE_PL = a128(FE_W * FE_H * 8);
constexpr size_t FE_SMEM = (size_t)FE_NS * FE_PL + 8 * FE_NS + 128;

__global__ void __launch_bounds__(NT, 1) k_fe_cd4(const __grid_constant__ CUtensorMap tu, double *__restrict__ Fout,
                                                  int n, int pitch, long long plane, double kx, double ky,
                                                  double kz, int zc) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    double *Us = reinterpret_cast<double *>(sm);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)FE_NS * FE_PL);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int x0 = blockIdx.x * RW, y0 = blockIdx.y * RH;
    const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, n);
    const int nit = z1 - z0 + 4;              // planes z0-2 .. z1+1
    auto issue = [&](int it) {
        const int s = it % FE_NS;
        mbar_expect_tx(&bar[s], FE_W * FE_H * 8);
        tma_load_3d(Us + s * (FE_PL / 8), &tu, x0 - 2, y0 - 2, z0 - 2 + it, &bar[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < FE_NS; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int it = 0; it < FE_NS && it < nit; ++it) issue(it);
    const int gx = x0 + lane;
    // z neighbours from a register ring of the owned points (slot = plane index mod 5; the z loop is
    // unrolled by 5 so every slot is a compile-time constant): 4 shared loads per thread and plane
    // instead of 16, and a plane's slot is free two steps after its arrival (not four)
    double zr[5][R];
    auto step = [&](auto Kc, int it) {
        constexpr int K = decltype(Kc)::value;                                  // it % 5
        constexpr int km2 = (K + 1) % 5, km1 = (K + 2) % 5, kp1 = (K + 4) % 5;   // planes it-4, it-3, it-1
        mbar_wait(&bar[it % FE_NS], (it / FE_NS) & 1);
        const double *Pn = Us + (it % FE_NS) * (FE_PL / 8);
#pragma unroll
        for (int r = 0; r < R; ++r) zr[K][r] = Pn[(R * w + r + 2) * FE_W + lane + 2];
        if (it >= 4) {   // centre plane z = z0-2+it-2
            const int gz = z0 - 4 + it;
            const double *P0 = Us + ((it - 2) % FE_NS) * (FE_PL / 8);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int ly = R * w + r, gy = y0 + ly;
                const int o = (ly + 2) * FE_W + lane + 2;
                const double dx = (8.0 * (P0[o + 1] - P0[o - 1]) - (P0[o + 2] - P0[o - 2])) * kx;
                const double dy = (8.0 * (P0[o + FE_W] - P0[o - FE_W]) - (P0[o + 2 * FE_W] - P0[o - 2 * FE_W])) * ky;
                const double dz = (8.0 * (zr[kp1][r] - zr[km1][r]) - (zr[K][r] - zr[km2][r])) * kz;
                if (gx < n && gy < n) Fout[(long long)gz * plane + (long long)gy * pitch + gx] = -((dx + dy) + dz);
            }
        }
        __syncthreads();
        // plane it-2 has been the centre plane (or never is one): refill its slot with plane it-2+FE_NS
        if (tid == 0 && it >= 2 && it - 2 + FE_NS < nit) issue(it - 2 + FE_NS);
    };
    for (int base = 0; base < nit; base += 5) {
        step(std::integral_constant<int, 0>{}, base);
        if (base + 1 < nit) step(std::integral_constant<int, 1>{}, base + 1);
        if (base + 2 < nit) step(std::integral_constant<int, 2>{}, base + 2);
        if (base + 3 < nit) step(std::integral_constant<int, 3>{}, base + 3);
        if (base + 4 < nit) step(std::integral_constant<int, 4>{}, base + 4);
    }
}

}  // namespace f3d
