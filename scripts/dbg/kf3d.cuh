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
#pragma once
#include "../../paper_1401_7824_b200/csrc/common.cuh"
#include "../../paper_1401_7824_b200/csrc/tma.cuh"

namespace f3d {

constexpr int NW = 8;            // warps per CTA
constexpr int NT = NW * 32;      // threads per CTA
constexpr int R = 4;             // rows per thread
constexpr int RW = 32;           // region width (one lane per column)
constexpr int RH = NW * R;       // region height

__host__ __device__ constexpr int a128(int b) { return (b + 127) / 128 * 128; }

__device__ __forceinline__ unsigned char *align_smem(unsigned char *p) {
    return reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(p) + 127) & ~uintptr_t(127));
}

// In-plane partial sums of the R owned rows from a plane in shared memory (row stride `ld`):
// window rows row0 .. row0+R+1 (centre rows row0+1 .. row0+R), columns col0 .. col0+2 (centre
// col0+1).  q = centre value, f = face sum, e = edge sum, all in the canonical order.
template <bool WANT_E>
__device__ __forceinline__ void plane_partials(const double *__restrict__ P, int ld, int row0, int col0, double (&q)[R],
                                               double (&f)[R], double (&e)[R]) {
    double v0[R + 2], v1[R + 2], v2[R + 2];
#pragma unroll
    for (int k = 0; k < R + 2; ++k) {
        const double *row = P + (row0 + k) * ld + col0;
        v0[k] = row[0];
        v1[k] = row[1];
        v2[k] = row[2];
    }
    double rr[R + 2];
#pragma unroll
    for (int k = 0; k < R + 2; ++k) rr[k] = v0[k] + v2[k];
#pragma unroll
    for (int r = 0; r < R; ++r) {
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
// u box 34 x 34 at (x0-2, y0-2); b box 32 x 32 at (x0-1, y0-1); t plane 34 x 34 (pad ring).
// ---------------------------------------------------------------------------------------------
constexpr int S_TX = RW - 2, S_TY = RH - 2;
constexpr int S_UW = RW + 2, S_UH = RH + 2;
constexpr int S_BW = RW, S_BH = RH;
constexpr int S_TW = RW + 2, S_TH = RH + 2;
constexpr int S_NS = 4;
constexpr int S_UPL = a128(S_UW * S_UH * 8), S_BPL = a128(S_BW * S_BH * 8), S_TPL = a128(S_TW * S_TH * 8);
constexpr size_t S_SMEM = (size_t)S_NS * (S_UPL + S_BPL) + 2 * S_TPL + 8 * S_NS + 128;

__global__ void __launch_bounds__(NT, 1) k_smooth2(const __grid_constant__ CUtensorMap tu,
                                                   const __grid_constant__ CUtensorMap tb,
                                                   double *__restrict__ out, int n, int pitch, long long plane,
                                                   SCoef c, int zc) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *sm = align_smem(smem_raw);
    double *Us = reinterpret_cast<double *>(sm);
    double *Bs = reinterpret_cast<double *>(sm + S_NS * S_UPL);
    double *Ts = reinterpret_cast<double *>(sm + S_NS * (S_UPL + S_BPL));
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + S_NS * (S_UPL + S_BPL) + 2 * S_TPL);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int x0 = blockIdx.x * S_TX, y0 = blockIdx.y * S_TY;
    const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, n);
    const int nit = z1 - z0 + 4;
    auto issue = [&](int it) {
        const int s = it % S_NS, p = z0 - 2 + it;
        mbar_expect_tx(&bar[s], (S_BW * S_BH) * 8);

        tma_load_3d(Bs + s * (S_BPL / 8), &tb, x0 - 1, y0 - 1, p - 1, &bar[s]);
    };
    if (tid == 0) {
        tma_prefetch_desc(&tu);
        tma_prefetch_desc(&tb);
        for (int s = 0; s < S_NS; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int it = 0; it < S_NS && it < nit; ++it) issue(it);

    const double c0 = c.c0, c1 = c.c1, c2 = c.c2, wd = c.wd;
    const int lx = lane - 1, ly0 = R * w - 1;        // region coordinates of the owned points
    const int gx = x0 + lx;
    const bool xin = gx >= 0 && gx < n;
    const bool xout = lx >= 0 && lx < S_TX && gx < n;
    bool yin[R], yout[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int ly = ly0 + r, gy = y0 + ly;
        yin[r] = gy >= 0 && gy < n;
        yout[r] = ly >= 0 && ly < S_TY && gy < n;
    }
    double *optr = out + (long long)(y0 + ly0) * pitch + gx;
    // rings: u at planes p-2 (a), p-1 (b); t at planes p-3 (a), p-2 (b); b value of the previous sweep-1 plane
    double qa[R], qb[R], fa[R], fb[R], eb[R];
    double ta[R], tb_[R], fta[R], ftb[R], etb[R], bo[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        qa[r] = qb[r] = fa[r] = fb[r] = eb[r] = 0.0;
        ta[r] = tb_[r] = fta[r] = ftb[r] = etb[r] = bo[r] = 0.0;
    }
    for (int it = 0; it < nit; ++it) {
        const int s = it % S_NS, p = z0 - 2 + it;
        mbar_wait(&bar[s], (it / S_NS) & 1); if (it == 0) return;
        double qn[R], fn[R], en[R];
        plane_partials<true>(Us + s * (S_UPL / 8), S_UW, R * w, lane, qn, fn, en);
        double tn[R], bn[R];
        const bool s1 = it >= 2;
        double *T = Ts + (it & 1) * (S_TPL / 8);
        if (s1) {   // sweep 1 at plane p-1 on the 32 x 32 region
            const int gz = p - 1;
            const bool zin = gz >= 0 && gz < n;
            const double *Bp = Bs + s * (S_BPL / 8);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double faces = fb[r] + (qa[r] + qn[r]);
                const double edges = eb[r] + (fa[r] + fn[r]);
                const double su = (c0 * qb[r] + c1 * faces) + c2 * edges;
                const double bv = Bp[(R * w + r) * S_BW + lane];
                const double t = (xin && yin[r] && zin) ? qb[r] + wd * (bv - su) : 0.0;
                T[(R * w + r + 1) * S_TW + lane + 1] = t;
                tn[r] = t;
                bn[r] = bv;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) { qa[r] = qb[r]; qb[r] = qn[r]; fa[r] = fb[r]; fb[r] = fn[r]; eb[r] = en[r]; }
        __syncthreads();
        if (tid == 0 && it + S_NS < nit) issue(it + S_NS);
        if (s1) {
            double tq[R], ftn[R], etn[R];
            plane_partials<true>(T, S_TW, R * w, lane, tq, ftn, etn);
            if (it >= 4) {   // sweep 2 at plane p-2 on the 30 x 30 tile
                const int gz = p - 2;
                double *op = optr + (long long)gz * plane;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double faces = ftb[r] + (ta[r] + tn[r]);
                    const double edges = etb[r] + (fta[r] + ftn[r]);
                    const double su = (c0 * tb_[r] + c1 * faces) + c2 * edges;
                    const double o = tb_[r] + wd * (bo[r] - su);
                    if (xout && yout[r]) op[(long long)r * pitch] = o;
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                ta[r] = tb_[r]; tb_[r] = tn[r]; fta[r] = ftb[r]; ftb[r] = ftn[r]; etb[r] = etn[r]; bo[r] = bn[r];
            }
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Defect + full-weighting restriction, one HBM pass (read u, b; write b_c), DESIGN.md §6.8.
// Coarse tile 15 x 15 x a coarse z chunk [K0, K1).  Fine defect region 31 x 31 at
// (2 I0, 2 J0), streamed over fine planes 2 K0 .. 2 K1; d(z) goes to a shared plane, coarse
// threads take its in-plane partials (face / edge / centre) and combine three planes.
// u box 34 x 34 at (2 I0 - 1, 2 J0 - 1); b box 32 x 32 at (2 I0, 2 J0).
// ---------------------------------------------------------------------------------------------
constexpr int R_CX = 15, R_CY = 15;
constexpr int R_UW = RW + 2, R_UH = RH + 2;
constexpr int R_BW = RW, R_BH = RH;
constexpr int R_DW = RW, R_DH = RH;
constexpr int R_NS = 4;
constexpr int R_UPL = a128(R_UW * R_UH * 8), R_BPL = a128(R_BW * R_BH * 8), R_DPL = a128(R_DW * R_DH * 8);
constexpr size_t R_SMEM = (size_t)R_NS * (R_UPL + R_BPL) + 2 * R_DPL + 8 * R_NS + 128;

__global__ void __launch_bounds__(NT, 1) k_restrict(const __grid_constant__ CUtensorMap tu,
                                                    const __grid_constant__ CUtensorMap tb,
                                                    double *__restrict__ bc, int nf, int nc, int pitch_c,
                                                    long long plane_c, SCoef c, int kc) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *sm = align_smem(smem_raw);
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
        tma_load_3d(Us + s * (R_UPL / 8), &tu, fx0 - 1, fy0 - 1, p, &bar[s]);
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
    // coarse role
    const bool crole = tid < R_CX * R_CY;
    const int ci = tid % R_CX, cj = tid / R_CX;
    const int gI = I0 + ci, gJ = J0 + cj;
    const bool cout_ok = crole && gI < nc && gJ < nc;
    const int dx = 2 * ci + 1, dy = 2 * cj + 1;
    double fdl = 0, edl = 0, dcl = 0, fdm = 0, edm = 0, dcm = 0;   // partials at planes 2K (lower), 2K+1 (mid)

    double qa[R], qb[R], fa[R], fb[R], eb[R];
#pragma unroll
    for (int r = 0; r < R; ++r) qa[r] = qb[r] = fa[r] = fb[r] = eb[r] = 0.0;
    for (int it = 0; it < nit; ++it) {
        const int s = it % R_NS, p = 2 * K0 - 1 + it;
        mbar_wait(&bar[s], (it / R_NS) & 1);
        double qn[R], fn[R], en[R];
        plane_partials<true>(Us + s * (R_UPL / 8), R_UW, R * w, lane, qn, fn, en);
        const bool dd = it >= 2;     // defect at fine plane p-1
        double *D = Ds + (it & 1) * (R_DPL / 8);
        if (dd) {
            const double *Bp = Bs + s * (R_BPL / 8);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double faces = fb[r] + (qa[r] + qn[r]);
                const double edges = eb[r] + (fa[r] + fn[r]);
                const double su = (c0 * qb[r] + c1 * faces) + c2 * edges;
                D[(R * w + r) * R_DW + lane] = Bp[(R * w + r) * R_BW + lane] - su;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) { qa[r] = qb[r]; qb[r] = qn[r]; fa[r] = fb[r]; fb[r] = fn[r]; eb[r] = en[r]; }
        __syncthreads();
        if (tid == 0 && it + R_NS < nit) issue(it + R_NS);
        if (dd && crole) {
            const int j = it - 2;    // fine plane 2K0 + j
            const double *d0 = D + (dy - 1) * R_DW + dx, *d1 = d0 + R_DW, *d2 = d1 + R_DW;
            const double rd0 = d0[-1] + d0[1], rd1 = d1[-1] + d1[1], rd2 = d2[-1] + d2[1];
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
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y, z = blockIdx.z;
    const int x = 2 * t;
    if (x >= nf) return;
    auto E = [&](int X, int Y, int Z) -> double {
        return (X >= 0 && X < nc && Y >= 0 && Y < nc && Z >= 0 && Z < nc)
                   ? __ldg(e + (long long)Z * plane_c + (long long)Y * pitch_c + X)
                   : 0.0;
    };
    const bool ye = !(y & 1), ze = !(z & 1);
    const int Ya = ye ? y / 2 - 1 : (y - 1) / 2, Yb = y / 2;
    const int Za = ze ? z / 2 - 1 : (z - 1) / 2, Zb = z / 2;
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
    double *row = u + (long long)z * plane_f + (long long)y * pitch_f;
    if (x + 1 < nf) {
        double2 v = *reinterpret_cast<double2 *>(row + x);
        v.x = v.x + se * we;
        v.y = v.y + so * w;
        *reinterpret_cast<double2 *>(row + x) = v;
    } else {
        row[x] = row[x] + se * we;
    }
}

}  // namespace f3d
