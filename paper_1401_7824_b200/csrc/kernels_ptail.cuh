// kernels_ptail.cuh -- the coarse-level tail of a PERIODIC V-cycle in one single-CTA launch (NEXT f3).
//
// Periodic grids (n = 2^p points, wrap-around neighbours) cannot use the Dirichlet tail's zero
// ring (kernels_tail.cuh), so this kernel keeps every level with n <= 64 (2D) / 16 (3D) as a dense
// n^D array in shared memory and runs the whole down-up recursion between __syncthreads()
// barriers: nu1 weighted-Jacobi sweeps, defect + full weighting, the exact 4^D solve, prolongation
// + correction, nu2 sweeps.  3D evaluates every point with the SAME device functions as the
// per-level kernels (apply_S, fw_defect, prolong_val of common.cuh / kernels_generic.cuh) on
// GridDesc views of the shared arrays; 2D writes the same canonical trees out on shared-memory
// offsets with power-of-two wrap masks (the defect is formed once per fine point, then weighted).
// Either way the result is bit-identical to launching the per-level kernels -- the tail only
// removes ~6 launches per level from these launch-latency-bound small problems.
#pragma once
#include "kernels_generic.cuh"

constexpr int PTAIL_MAX_LEVELS = 6;
constexpr int PTAIL_THREADS = 1024;

struct PTailParams {
    int nlev;                        // levels handled: n0, n0/2, ..., 4
    int n[PTAIL_MAX_LEVELS];
    SCoef c[PTAIL_MAX_LEVELS];
    int nu1, nu2;
    const double *Ginv;              // P x P inverse of the 4^D operator
    const double *b_in;              // level-n0 right-hand side (global, pitch n0)
    const double *u_in;              // initial iterate, or null for zero
    double *u_out;                   // result
};

template <int D>
__host__ __device__ inline size_t ptail_smem_bytes(const PTailParams &P) {
    size_t pts = 0;
    for (int l = 0; l < P.nlev; ++l) pts += (size_t)P.n[l] * P.n[l] * (D == 3 ? P.n[l] : 1);
    return 3 * pts * sizeof(double);
}

template <int D>
__device__ __forceinline__ GridDesc ptail_grid(int n) {
    GridDesc g;
    g.n = n;
    g.pitch = n;
    g.plane = (D == 3) ? (long long)n * n : 0;
    g.per = 1;
    return g;
}

// body(p, i, j, k) for every point of an n^D level (n a power of two), block-strided
template <int D, typename F>
__device__ __forceinline__ void ptail_points(int n, F body) {
    const int lg = __ffs(n) - 1;
    const int pts = (D == 3) ? n * n * n : n * n;
    for (int p = threadIdx.x; p < pts; p += PTAIL_THREADS) {
        const int i = p & (n - 1), j = (p >> lg) & (n - 1), k = (D == 3) ? (p >> (2 * lg)) : 0;
        body(p, i, j, k);
    }
}

// 2D: the S-tree of apply_S at point (i, j) of a periodic n x n shared array at offset ou
__device__ __forceinline__ double ptail_S2(const SCoef &c, const double *sm, int ou, int n, int i, int j) {
    const int msk = n - 1, lg = __ffs(n) - 1;
    const int im = (i - 1) & msk, ip = (i + 1) & msk;
    const int r0 = ou + (((j - 1) & msk) << lg), r1 = ou + (j << lg), r2 = ou + (((j + 1) & msk) << lg);
    const double rm = sm[r0 + im] + sm[r0 + ip];
    const double rc = sm[r1 + im] + sm[r1 + ip];
    const double rp = sm[r2 + im] + sm[r2 + ip];
    const double faces = rc + (sm[r0 + i] + sm[r2 + i]);
    const double edges = rm + rp;
    return (c.c0 * sm[r1 + i] + c.c1 * faces) + c.c2 * edges;
}
template <int D>
__device__ __noinline__ void ptail_jacobi(const SCoef c, const GridDesc g, double *out, const double *u,
                                          const double *b) {
    if (D == 2) {
        // 2D: the canonical trees of apply_S written out on shared-memory offsets with power-of-two
        // wrap masks (same operations in the same order as tr_r / tr_f / tr_e, so the same bits)
        extern __shared__ double sm[];
        const int n = g.n, msk = n - 1, lg = __ffs(n) - 1;
        const int ou = (int)(u - sm), ob = (int)(b - sm), oo = (int)(out - sm);
        for (int p = threadIdx.x; p < n * n; p += PTAIL_THREADS)
            sm[oo + p] = sm[ou + p] + c.wd * (sm[ob + p] - ptail_S2(c, sm, ou, n, p & msk, p >> lg));
    } else {
        ptail_points<D>(g.n, [&](int p, int i, int j, int k) { out[p] = u[p] + c.wd * (b[p] - apply_S<D>(c, u, g, i, j, k)); });
    }
    __syncthreads();
}

// d = b - S u at every point (defect_at's value)
__device__ __noinline__ void ptail_defect2(const SCoef c, int n, double *d, const double *u, const double *b) {
    extern __shared__ double sm[];
    const int msk = n - 1, lg = __ffs(n) - 1;
    const int ou = (int)(u - sm), ob = (int)(b - sm), od = (int)(d - sm);
    for (int p = threadIdx.x; p < n * n; p += PTAIL_THREADS)
        sm[od + p] = sm[ob + p] - ptail_S2(c, sm, ou, n, p & msk, p >> lg);
    __syncthreads();
}
// full weighting of a stored defect (fw_defect's tree): coarse (I, J) <-> fine (2I, 2J); zero uc
__device__ __noinline__ void ptail_fw2(int nc, double *bc, double *uc, const double *d) {
    extern __shared__ double sm[];
    const int nf = 2 * nc, mf = nf - 1, lgf = __ffs(nf) - 1, lgc = __ffs(nc) - 1;
    const int od = (int)(d - sm), obc = (int)(bc - sm), ouc = (int)(uc - sm);
    for (int p = threadIdx.x; p < nc * nc; p += PTAIL_THREADS) {
        const int x = 2 * (p & (nc - 1)), y = 2 * (p >> lgc);
        const int xm = (x - 1) & mf, xp = (x + 1) & mf;
        const int r0 = od + (((y - 1) & mf) << lgf), r1 = od + (y << lgf), r2 = od + (((y + 1) & mf) << lgf);
        const double rd0 = sm[r0 + xm] + sm[r0 + xp], rd1 = sm[r1 + xm] + sm[r1 + xp], rd2 = sm[r2 + xm] + sm[r2 + xp];
        const double fd = rd1 + (sm[r0 + x] + sm[r2 + x]);
        const double ed = rd0 + rd2;
        sm[obc + p] = ((4.0 * sm[r1 + x] + 2.0 * fd) + ed) * 0.0625;
        sm[ouc + p] = 0.0;
    }
}
// u += P e (prolong_val's tree): an odd fine index pairs coarse (x-1)/2 and (x+1)/2 mod nc
__device__ __noinline__ void ptail_prolong2(int n, double *u, const double *e) {
    extern __shared__ double sm[];
    const int nc = n / 2, mc = nc - 1, lg = __ffs(n) - 1, lgc = lg - 1;
    const int ou = (int)(u - sm), oe = (int)(e - sm);
    for (int p = threadIdx.x; p < n * n; p += PTAIL_THREADS) {
        const int i = p & (n - 1), j = p >> lg;
        const bool xe = i & 1, ye = j & 1;
        const int xa = i >> 1, xb = (xa + 1) & mc, ya = j >> 1, yb = (ya + 1) & mc;
        double w = 1.0;
        if (xe) w *= 0.5;
        if (ye) w *= 0.5;
        double sx = sm[oe + (ya << lgc) + xa];
        if (xe) sx = sx + sm[oe + (ya << lgc) + xb];
        double sy = sx;
        if (ye) {
            double sx2 = sm[oe + (yb << lgc) + xa];
            if (xe) sx2 = sx2 + sm[oe + (yb << lgc) + xb];
            sy = sy + sx2;
        }
        sm[ou + p] = sm[ou + p] + sy * w;
    }
}

template <int D>
__global__ void __launch_bounds__(PTAIL_THREADS, 1) k_ptail(PTailParams P) {
    extern __shared__ double sm[];
    double *U[PTAIL_MAX_LEVELS], *B[PTAIL_MAX_LEVELS], *T[PTAIL_MAX_LEVELS];
    {
        size_t off = 0;
        for (int l = 0; l < P.nlev; ++l) {
            const size_t pts = (size_t)P.n[l] * P.n[l] * (D == 3 ? P.n[l] : 1);
            U[l] = sm + off; off += pts;
            B[l] = sm + off; off += pts;
            T[l] = sm + off; off += pts;
        }
    }
    const int L = P.nlev - 1;
    ptail_points<D>(P.n[0], [&](int p, int, int, int) {
        B[0][p] = P.b_in[p];
        U[0][p] = P.u_in ? P.u_in[p] : 0.0;
    });
    __syncthreads();
    // down: pre-smoothing, defect + full weighting into the next level's b, zero correction there
    for (int l = 0; l < L; ++l) {
        const GridDesc g = ptail_grid<D>(P.n[l]);
        for (int s = 0; s < P.nu1; ++s) {
            ptail_jacobi<D>(P.c[l], g, T[l], U[l], B[l]);
            double *t = U[l]; U[l] = T[l]; T[l] = t;
        }
        const GridDesc gc = ptail_grid<D>(P.n[l + 1]);
        const SCoef c = P.c[l];
        double *u = U[l], *b = B[l], *bc = B[l + 1], *uc = U[l + 1];
        if (D == 2) {
            ptail_defect2(c, g.n, T[l], u, b);          // d = b - S u once per fine point, into T
            ptail_fw2(gc.n, bc, uc, T[l]);
        } else {
            ptail_points<D>(gc.n, [&](int p, int I, int J, int K) {
                bc[p] = fw_defect<D>(c, u, b, g, I, J, K);
                uc[p] = 0.0;
            });
        }
        __syncthreads();
    }
    // coarsest (n = 4): exact solve u = Ginv b, left fold over ascending j
    {
        const int Pc = (D == 3) ? 64 : 16;
        const double *b = B[L];
        double *u = U[L];
        if ((int)threadIdx.x < Pc) {
            const int t = threadIdx.x;
            double acc = P.Ginv[t * Pc] * b[0];
            for (int jj = 1; jj < Pc; ++jj) acc = acc + P.Ginv[t * Pc + jj] * b[jj];
            u[t] = acc;
        }
        __syncthreads();
    }
    // up: prolongation + correction, post-smoothing
    for (int l = L - 1; l >= 0; --l) {
        const GridDesc g = ptail_grid<D>(P.n[l]), gc = ptail_grid<D>(P.n[l + 1]);
        double *u = U[l];
        const double *e = U[l + 1];
        if (D == 2) ptail_prolong2(g.n, u, e);
        else ptail_points<D>(g.n, [&](int p, int i, int j, int k) { u[p] = u[p] + prolong_val<D>(e, gc, g, i, j, k); });
        __syncthreads();
        for (int s = 0; s < P.nu2; ++s) {
            ptail_jacobi<D>(P.c[l], g, T[l], U[l], B[l]);
            double *t = U[l]; U[l] = T[l]; T[l] = t;
        }
    }
    ptail_points<D>(P.n[0], [&](int p, int, int, int) { P.u_out[p] = U[0][p]; });
}
