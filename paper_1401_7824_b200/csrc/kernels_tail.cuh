// kernels_tail.cuh -- the coarse-level tail of the V-cycle in ONE single-CTA launch.
//
// All levels with n <= tail_n (2D: 63, 3D: 15) live in shared memory as dense arrays with a
// zero ring (the homogeneous Dirichlet data), and the whole down-up recursion -- weighted-Jacobi
// sweeps, defect + full weighting, exact 3^d solve, prolongation + correction -- runs between
// __syncthreads() barriers, replacing ~7 launches per level.  Arithmetic is the canonical trees
// of DESIGN.md §4, identical to the per-level kernels.  Every phase walks the level row by row
// (warp = row, lane = column) with row pointers, so a stencil costs 9 (2D) / 19 (3D) shared
// loads at immediate offsets and no index arithmetic.
#pragma once
#include "common.cuh"

constexpr int TAIL_MAX_LEVELS = 6;
constexpr int TAIL_THREADS = 1024;
constexpr int TAIL_WARPS = TAIL_THREADS / 32;

struct TailParams {
    int nlev;                       // levels handled (n0, (n0-1)/2, ..., 3)
    int n[TAIL_MAX_LEVELS];
    SCoef c[TAIL_MAX_LEVELS];
    int nu1, nu2;
    const double *Ginv;             // P x P inverse of the 3^d operator
    const double *b_in;             // pitched level-n0 right-hand side (global)
    const double *u_in;             // pitched initial iterate, or null for zero
    double *u_out;                  // pitched result
    int pitch;                      // pitch of b_in / u_in / u_out (n0 + 1)
    int fuse_dr;                    // 2D: defect formed inside the restriction phase
};

template <int D>
__host__ __device__ __forceinline__ int tail_padded(int n) {
    return D == 3 ? (n + 2) * (n + 2) * (n + 2) : (n + 2) * (n + 2);
}

// Row walk: for every interior row (j, k) of an n^D level, `body(rowoff, j, k)` is called by
// one warp, rowoff = padded offset of point (0, j, k); lanes then step through the columns.
template <int D, typename F>
__device__ __forceinline__ void tail_rows(int n, F body) {
    const int np = n + 2;
    const int rows = (D == 3) ? n * n : n;
    for (int q = threadIdx.x >> 5; q < rows; q += TAIL_WARPS) {
        const int j = (D == 3) ? q % n : q, k = (D == 3) ? q / n : 0;
        body(1 + np * ((j + 1) + (D == 3 ? np * (k + 1) : 0)), j, k);
    }
}

// out[o] = fn(o, i, j, k) for every interior point of an n^D level, with all of a thread's points
// (2D: up to 4 rows x 2 columns; 3D: 16 lanes per row, 2 rows per warp, up to 8 iterations)
// evaluated before any store, so the independent stencils overlap (ILP) and `out` may alias
// nothing that fn reads.  Covers 2D n <= 63 and 3D n <= 15 (the tail levels).
template <int D, typename F>
__device__ __forceinline__ void tail_map(int n, double *out, F fn) {
    constexpr int LPR = (D == 2) ? 32 : 16;            // lanes per row
    constexpr int RPW = 32 / LPR;                       // rows per warp per iteration
    constexpr int RM = (D == 2) ? 64 / TAIL_WARPS : 256 / (TAIL_WARPS * RPW), CM = (D == 2) ? 2 : 1;
    const int np = n + 2;
    const int rows = (D == 3) ? n * n : n;
    const int lane = threadIdx.x & 31, sub = lane / LPR, li = lane % LPR;
    const int q0 = (threadIdx.x >> 5) * RPW + sub;
    if (q0 >= rows || li >= n) return;   // idle warps / lanes of the small levels leave at once
    double v[RM][CM];
    int off[RM][CM];
    bool ok[RM][CM];
#pragma unroll
    for (int rr = 0; rr < RM; ++rr) {
        const int q = q0 + rr * TAIL_WARPS * RPW;
        const int j = (D == 3) ? q % n : q, k = (D == 3) ? q / n : 0;
        const int ro = 1 + np * ((j + 1) + (D == 3 ? np * (k + 1) : 0));
#pragma unroll
        for (int cc = 0; cc < CM; ++cc) {
            const int i = li + cc * LPR;
            ok[rr][cc] = q < rows && i < n;
            off[rr][cc] = ro + i;
            v[rr][cc] = ok[rr][cc] ? fn(ro + i, i, j, k) : 0.0;
        }
    }
#pragma unroll
    for (int rr = 0; rr < RM; ++rr)
#pragma unroll
        for (int cc = 0; cc < CM; ++cc)
            if (ok[rr][cc]) out[off[rr][cc]] = v[rr][cc];
}

// canonical S u at padded offset o: planes at +-pl (3D), rows at +-np
template <int D>
__device__ __forceinline__ double tail_S(const double *__restrict__ a, int o, int np, int pl, const SCoef &c) {
    const double rc = a[o - 1] + a[o + 1];
    const double rm = a[o - np - 1] + a[o - np + 1];
    const double rp = a[o + np - 1] + a[o + np + 1];
    const double f = rc + (a[o - np] + a[o + np]);
    const double e = rm + rp;
    if (D == 2) return (c.c0 * a[o] + c.c1 * f) + c.c2 * e;
    const int ol = o - pl, ou = o + pl;
    const double fl = (a[ol - 1] + a[ol + 1]) + (a[ol - np] + a[ol + np]);
    const double fu = (a[ou - 1] + a[ou + 1]) + (a[ou - np] + a[ou + np]);
    const double faces = f + (a[ol] + a[ou]);
    const double edges = e + (fl + fu);
    return (c.c0 * a[o] + c.c1 * faces) + c.c2 * edges;
}

// The phases are out-of-line functions: the tail runs each phase once per level and barrier, so
// straight-line (inlined, unrolled) code would miss the instruction cache on every phase.  Arrays
// are passed as offsets into the dynamic shared memory (tsm + offset stays a shared address).
extern __shared__ __align__(16) double tsm[];

// out = in + wd (b - S in)            (weighted Jacobi sweep)
template <int D>
__device__ __noinline__ void tail_ph_sweep(int oin, int oout, int ob, int n, SCoef c) {
    const double *in = tsm + oin, *B = tsm + ob;
    double *out = tsm + oout;
    const int np = n + 2, pl = np * np;
    tail_map<D>(n, out, [&](int o, int, int, int) { return in[o] + c.wd * (B[o] - tail_S<D>(in, o, np, pl, c)); });
}
// d = b - S u                          (defect)
template <int D>
__device__ __noinline__ void tail_ph_defect(int ou, int od, int ob, int n, SCoef c) {
    const double *u = tsm + ou, *B = tsm + ob;
    double *d = tsm + od;
    const int np = n + 2, pl = np * np;
    tail_map<D>(n, d, [&](int o, int, int, int) { return B[o] - tail_S<D>(u, o, np, pl, c); });
}
// b_c = R d                            (full weighting: coarse I <-> fine 2I+1)
template <int D>
__device__ __noinline__ void tail_ph_restrict(int od, int obc, int n, int nc) {
    const double *d = tsm + od;
    double *Bc = tsm + obc;
    const int np = n + 2, pl = np * np;
    tail_map<D>(nc, Bc, [&](int, int I, int J, int K) {
        const int o = 1 + np * ((2 * J + 2) + (D == 3 ? np * (2 * K + 2) : 0)) + 2 * I + 1;
        const double rm = d[o - np - 1] + d[o - np + 1];
        const double rc = d[o - 1] + d[o + 1];
        const double rp = d[o + np - 1] + d[o + np + 1];
        const double f = rc + (d[o - np] + d[o + np]);
        const double e = rm + rp;
        if (D == 2) return ((4.0 * d[o] + 2.0 * f) + e) * 0.0625;
        const int ol = o - pl, ou = o + pl;
        const double fl = (d[ol - 1] + d[ol + 1]) + (d[ol - np] + d[ol + np]);
        const double fu = (d[ou - 1] + d[ou + 1]) + (d[ou - np] + d[ou + np]);
        const double el = (d[ol - np - 1] + d[ol - np + 1]) + (d[ol + np - 1] + d[ol + np + 1]);
        const double eu = (d[ou - np - 1] + d[ou - np + 1]) + (d[ou + np - 1] + d[ou + np + 1]);
        const double faces = f + (d[ol] + d[ou]);
        const double edges = e + (fl + fu);
        const double co = el + eu;
        return ((8.0 * d[o] + 4.0 * faces) + (2.0 * edges + co)) * 0.015625;
    });
}
// b_c = R (b - S u) with the defect formed on the fly at the 9 fine points of each coarse point
// (2D; the same tail_S / restriction trees as tail_ph_defect + tail_ph_restrict, one barrier less)
__device__ __noinline__ void tail_ph_defect_restrict2(int ou, int ob, int obc, int n, int nc, SCoef c) {
    const double *u = tsm + ou, *B = tsm + ob;
    double *Bc = tsm + obc;
    const int np = n + 2;
    tail_map<2>(nc, Bc, [&](int, int I, int J, int) {
        const int o = 1 + np * (2 * J + 2) + 2 * I + 1;
        auto d = [&](int q) { return B[q] - tail_S<2>(u, q, np, 0, c); };
        const double dmm = d(o - np - 1), dmp = d(o - np + 1), dpm = d(o + np - 1), dpp = d(o + np + 1);
        const double dcm = d(o - 1), dcp = d(o + 1), dmc = d(o - np), dpc = d(o + np), dcc = d(o);
        const double rm = dmm + dmp;
        const double rc = dcm + dcp;
        const double rp = dpm + dpp;
        const double f = rc + (dmc + dpc);
        const double e = rm + rp;
        return ((4.0 * dcc + 2.0 * f) + e) * 0.0625;
    });
}

// u += P e                             (sums nest x, then y, then z; one multiply by 0.5^#even)
template <int D>
__device__ __noinline__ void tail_ph_prolong(int oe, int ou, int n, int nc) {
    const double *e = tsm + oe;
    double *u = tsm + ou;
    const int npc = nc + 2, plc = npc * npc;
    tail_map<D>(n, u, [&](int o, int i, int j, int k) {
        const bool ye = !(j & 1), ze = (D == 3) && !(k & 1), xe = !(i & 1);
        // padded coarse offsets (coarse index -1 -> the zero ring)
        const int Ya = ye ? j / 2 - 1 : (j - 1) / 2, Yb = j / 2;
        const int Za = (D == 3) ? (ze ? k / 2 - 1 : (k - 1) / 2) : 0, Zb = (D == 3) ? k / 2 : 0;
        const int xa = (xe ? i / 2 - 1 : (i - 1) / 2) + 1, xb = i / 2 + 1;
        const int rya = npc * (Ya + 1), ryb = npc * (Yb + 1);
        const int pza = (D == 3) ? plc * (Za + 1) : 0, pzb = (D == 3) ? plc * (Zb + 1) : 0;
        double w = 1.0;
        if (xe) w *= 0.5;
        if (ye) w *= 0.5;
        if (ze) w *= 0.5;
        auto sx = [&](int off) { return xe ? e[off + xa] + e[off + xb] : e[off + xa]; };
        auto sy = [&](int pz) { return ye ? sx(pz + rya) + sx(pz + ryb) : sx(pz + rya); };
        const double sz = ze ? sy(pza) + sy(pzb) : sy(pza);
        return u[o] + sz * w;
    });
}

template <int D>
__global__ void __launch_bounds__(TAIL_THREADS, 1) k_tail(TailParams P) {
    const int L = P.nlev;
    const int lane = threadIdx.x & 31;
    __shared__ int offs[TAIL_MAX_LEVELS], szs[TAIL_MAX_LEVELS];
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int l = 0; l < L; ++l) { offs[l] = tot; szs[l] = tail_padded<D>(P.n[l]); tot += 3 * szs[l]; }
    }
    {
        int tot = 0;
        for (int l = 0; l < L; ++l) tot += 3 * tail_padded<D>(P.n[l]);
        // zero everything once: the rings stay zero for the whole kernel
        for (int q = threadIdx.x; q < tot; q += TAIL_THREADS) tsm[q] = 0.0;
    }
    __syncthreads();
    // buffer w in {0,1} = iterate ping-pong, 2 = right-hand side
    auto ofs = [&](int l, int w) { return offs[l] + w * szs[l]; };
    {
        const int n = P.n[0];
        double *U = tsm + ofs(0, 0), *B = tsm + ofs(0, 2);
        tail_rows<D>(n, [&](int ro, int j, int k) {
            const long long g = (long long)P.pitch * (j + (D == 3 ? (long long)n * k : 0));
            for (int i = lane; i < n; i += 32) {
                B[ro + i] = P.b_in[g + i];
                if (P.u_in) U[ro + i] = P.u_in[g + i];
            }
        });
    }
    __syncthreads();
    unsigned cur = 0;   // bit l: iterate of level l is in buffer 1
    auto smooth = [&](int l, int sweeps) {
        for (int s = 0; s < sweeps; ++s) {
            const int w = (cur >> l) & 1;
            tail_ph_sweep<D>(ofs(l, w), ofs(l, 1 - w), ofs(l, 2), P.n[l], P.c[l]);
            cur ^= 1u << l;
            __syncthreads();
        }
    };
    // ---------------- down
    for (int l = 0; l < L - 1; ++l) {
        smooth(l, P.nu1);
        const int w = (cur >> l) & 1;
        if (D == 2 && P.fuse_dr) {
            tail_ph_defect_restrict2(ofs(l, w), ofs(l, 2), ofs(l + 1, 2), P.n[l], P.n[l + 1], P.c[l]);
        } else {
            tail_ph_defect<D>(ofs(l, w), ofs(l, 1 - w), ofs(l, 2), P.n[l], P.c[l]);
            __syncthreads();
            tail_ph_restrict<D>(ofs(l, 1 - w), ofs(l + 1, 2), P.n[l], P.n[l + 1]);
        }
        __syncthreads();
        // the next level starts from a zero iterate (its buffers are zero except where written;
        // buffer 0 of level l+1 has never been written at this point of the down sweep)
    }
    // ---------------- coarsest: exact solve u = Ginv b, ascending-j accumulation
    {
        constexpr int Pc = D == 3 ? 27 : 9;
        const int l = L - 1;
        double *u = tsm + ofs(l, 0);
        const double *B = tsm + ofs(l, 2);
        if (threadIdx.x < Pc) {
            const int t = threadIdx.x;
            auto po = [&](int q) {   // padded offset of unknown q (x fastest) on the 5^D array
                return (q % 3 + 1) + 5 * (((q / 3) % 3 + 1) + (D == 3 ? 5 * (q / 9 + 1) : 0));
            };
            double acc = P.Ginv[t * Pc] * B[po(0)];
            for (int jj = 1; jj < Pc; ++jj) acc = acc + P.Ginv[t * Pc + jj] * B[po(jj)];
            u[po(t)] = acc;
        }
        cur &= ~(1u << l);
        __syncthreads();
    }
    // ---------------- up
    for (int l = L - 2; l >= 0; --l) {
        tail_ph_prolong<D>(ofs(l + 1, (cur >> (l + 1)) & 1), ofs(l, (cur >> l) & 1), P.n[l], P.n[l + 1]);
        __syncthreads();
        smooth(l, P.nu2);
    }
    // ---------------- write the level-0 result
    {
        const int n = P.n[0];
        const double *u = tsm + ofs(0, cur & 1);
        tail_rows<D>(n, [&](int ro, int j, int k) {
            const long long g = (long long)P.pitch * (j + (D == 3 ? (long long)n * k : 0));
            for (int i = lane; i < n; i += 32) P.u_out[g + i] = u[ro + i];
        });
    }
}

template <int D>
inline size_t tail_smem_bytes(const TailParams &P) {
    size_t s = 0;
    for (int l = 0; l < P.nlev; ++l) s += 3 * (size_t)tail_padded<D>(P.n[l]);
    return s * sizeof(double);
}
