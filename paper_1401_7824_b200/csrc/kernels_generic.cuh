// kernels_generic.cuh -- one-point-per-thread kernels for every step of the ISDC hot path, 2D and
// 3D, reading the canonical trees straight from global memory (L1/L2 absorb the neighbour reuse).
// They serve the coarse levels, the RHS/residual, and the reference for the tuned fine-level
// kernels (kernels_fast2d.cuh / kernels_fast3d.cuh), which must produce the same bits.
#pragma once
#include "common.cuh"

struct VWParams {                 // RHS of Eq. (5) for substep m
    const double *uold[ISDC_MAXM];
    const double *unew_m;
    int M, m;
    double dtm, gm;               // dt*dtau_m, nu*dtm
    double a[ISDC_MAXM];          // dt*S_{m,j}
    double beta[ISDC_MAXM];       // (nu*dt)*S_{m,j}
    const double *ct;             // device: cos(t_n + dt*tau_j), j = 0..M-1 (Burgers: alpha of uold_j)
    const double *ctn;            // the same for unew_m (&ct[m]; Burgers: alpha of unew_m)
    const double *F[ISDC_MAXM];   // stored f^E(uold_j), or F[0] == null: evaluate f^E here
    const double *Fn;             // stored f^E(unew_m)
    FeDesc fe;
    GridDesc g;
};

struct PZParams {                 // residual of node m
    const double *u[ISDC_MAXM];
    int M, m;
    double qa[ISDC_MAXM];         // dt*Q_{m,j}
    double qb[ISDC_MAXM];         // (nu*dt)*Q_{m,j}
    const double *ct;             // device: cos(t_n + dt*tau_j) (Burgers: alpha of u_j)
    const double *F[ISDC_MAXM];   // stored f^E(u_j), or F[0] == null: evaluate f^E here
    FeDesc fe;
    GridDesc g;
};

#define POINT_INDEX_OR_RETURN(g)                                   \
    int i = blockIdx.x * blockDim.x + threadIdx.x;                 \
    int j = blockIdx.y * blockDim.y + threadIdx.y;                 \
    int k = (D == 3) ? (int)blockIdx.z : 0;                        \
    bool inside = (i < (g).n && j < (g).n);

// weighted Jacobi sweep, out of place: out = u + wd*(b - S u)
template <int D>
__global__ void k_jacobi(double *__restrict__ out, const double *__restrict__ u, const double *__restrict__ b,
                         GridDesc g, SCoef c) {
    POINT_INDEX_OR_RETURN(g)
    if (!inside) return;
    long long p = gidx(g, i, j, k);
    out[p] = u[p] + c.wd * (b[p] - apply_S<D>(c, u, g, i, j, k));
}

// ||b - S u||_inf into *slot (uint64 bits of a non-negative double)
template <int D>
__global__ void k_defect_norm(const double *__restrict__ u, const double *__restrict__ b, GridDesc g, SCoef c,
                              unsigned long long *slot) {
    POINT_INDEX_OR_RETURN(g)
    double v = 0.0;
    if (inside) v = fabs(b[gidx(g, i, j, k)] - apply_S<D>(c, u, g, i, j, k));
    block_max_to(slot, v);
}

// ||q||_inf into *slot
template <int D>
__global__ void k_norm(const double *__restrict__ q, GridDesc g, unsigned long long *slot) {
    POINT_INDEX_OR_RETURN(g)
    double v = 0.0;
    if (inside) v = fabs(q[gidx(g, i, j, k)]);
    block_max_to(slot, v);
}

// defect at a fine point
template <int D>
__device__ __forceinline__ double defect_at(const SCoef &c, const double *u, const double *b, const GridDesc &g,
                                            int i, int j, int k) {
    if (g.per) {   // periodic: the fine neighbours of coarse point 0 wrap around
        i = wrapn(i, g.n); j = wrapn(j, g.n);
        if (D == 3) k = wrapn(k, g.n);
    }
    return b[gidx(g, i, j, k)] - apply_S<D>(c, u, g, i, j, k);
}

// full weighting of the fine defect d = b - S u: coarse (I,J,K) <-> fine (2I+1, 2J+1, 2K+1);
// periodic grids: fine (2I, 2J, 2K).  The value at one coarse point (shared with the periodic tail).
template <int D>
__device__ __forceinline__ double fw_defect(const SCoef &c, const double *u, const double *b, const GridDesc &gf,
                                            int I, int J, int K) {
    const int o = gf.per ? 0 : 1;
    int x = 2 * I + o, y = 2 * J + o, z = (D == 3) ? 2 * K + o : 0;
    if (D == 2) {
        double d[3][3];
#pragma unroll
        for (int b_ = 0; b_ < 3; ++b_)
#pragma unroll
            for (int a_ = 0; a_ < 3; ++a_) d[b_][a_] = defect_at<D>(c, u, b, gf, x - 1 + a_, y - 1 + b_, 0);
        double rd0 = d[0][0] + d[0][2], rd1 = d[1][0] + d[1][2], rd2 = d[2][0] + d[2][2];
        double fd = rd1 + (d[0][1] + d[2][1]);
        double ed = rd0 + rd2;
        return ((4.0 * d[1][1] + 2.0 * fd) + ed) * 0.0625;
    } else {
        double fd[3], ed[3], dc[3];
#pragma unroll
        for (int c_ = 0; c_ < 3; ++c_) {
            double d[3][3];
#pragma unroll
            for (int b_ = 0; b_ < 3; ++b_)
#pragma unroll
                for (int a_ = 0; a_ < 3; ++a_) d[b_][a_] = defect_at<D>(c, u, b, gf, x - 1 + a_, y - 1 + b_, z - 1 + c_);
            double rd0 = d[0][0] + d[0][2], rd1 = d[1][0] + d[1][2], rd2 = d[2][0] + d[2][2];
            fd[c_] = rd1 + (d[0][1] + d[2][1]);
            ed[c_] = rd0 + rd2;
            dc[c_] = d[1][1];
        }
        double F = fd[1] + (dc[0] + dc[2]);
        double E = ed[1] + (fd[0] + fd[2]);
        double C = ed[0] + ed[2];
        return ((8.0 * dc[1] + 4.0 * F) + (2.0 * E + C)) * 0.015625;
    }
}
template <int D>
__global__ void k_restrict_defect(double *__restrict__ bc, GridDesc gc, const double *__restrict__ u,
                                  const double *__restrict__ b, GridDesc gf, SCoef c) {
    int I = blockIdx.x * blockDim.x + threadIdx.x;
    int J = blockIdx.y * blockDim.y + threadIdx.y;
    int K = (D == 3) ? (int)blockIdx.z : 0;
    if (I >= gc.n || J >= gc.n) return;
    bc[gidx(gc, I, J, K)] = fw_defect<D>(c, u, b, gf, I, J, K);
}

// bi/trilinear prolongation + correction u += P e.  Per axis, Dirichlet: an even
// fine index takes the coarse pair (x/2-1, x/2), an odd one (x-1)/2; periodic: an odd fine index
// takes the pair ((x-1)/2, (x+1)/2 mod nc), an even one x/2.
__device__ __forceinline__ bool prolong_axis(int x, bool per, int &a, int &b) {
    // pair iff (x + per) is even; first member (x - 1 + per) >> 1 (arithmetic shift: -1 at x = 0)
    bool pair = ((x + (per ? 1 : 0)) & 1) == 0;
    a = (x - (per ? 0 : 1)) >> 1;
    b = a + 1;
    if (!pair) a = b = (per ? x >> 1 : (x - 1) >> 1);
    return pair;
}
// the correction (P e)(i,j,k) at one fine point (shared with the periodic tail)
template <int D>
__device__ __forceinline__ double prolong_val(const double *e, const GridDesc &gc, const GridDesc &gf, int i, int j,
                                              int k) {
    int xa, xb, ya, yb, za = 0, zb = 0;
    const bool per = gf.per != 0;
    bool xe = prolong_axis(i, per, xa, xb), ye = prolong_axis(j, per, ya, yb);
    bool ze = (D == 3) && prolong_axis(k, per, za, zb);
    double w = 1.0;
    if (xe) w *= 0.5;
    if (ye) w *= 0.5;
    if (ze) w *= 0.5;
    double sz = 0.0;
    for (int cz = 0; cz < ((D == 3 && ze) ? 2 : 1); ++cz) {
        int Z = cz ? zb : za;
        double sy = 0.0;
        for (int cy = 0; cy < (ye ? 2 : 1); ++cy) {
            int Y = cy ? yb : ya;
            double sx = ldz<D>(e, gc, xa, Y, Z);
            if (xe) sx = sx + ldz<D>(e, gc, xb, Y, Z);
            sy = cy ? sy + sx : sx;
        }
        sz = cz ? sz + sy : sy;
    }
    return sz * w;
}
template <int D>
__global__ void k_prolong_add(double *__restrict__ u, GridDesc gf, const double *__restrict__ e, GridDesc gc) {
    POINT_INDEX_OR_RETURN(gf)
    if (!inside) return;
    long long p = gidx(gf, i, j, k);
    u[p] = u[p] + prolong_val<D>(e, gc, gf, i, j, k);
}

// coarsest level (n = 3; periodic n = 4): u = Ginv b, accumulated over ascending j
template <int D>
__global__ void k_coarse_solve(double *__restrict__ u, const double *__restrict__ b, GridDesc g,
                               const double *__restrict__ Ginv) {
    const int n = g.n, P = (D == 3) ? n * n * n : n * n;
    __shared__ double bs[64];
    int t = threadIdx.x;
    if (t < P) bs[t] = b[gidx(g, t % n, (t / n) % n, D == 3 ? t / (n * n) : 0)];
    __syncthreads();
    if (t < P) {
        double acc = Ginv[t * P] * bs[0];
        for (int jj = 1; jj < P; ++jj) acc = acc + Ginv[t * P + jj] * bs[jj];
        u[gidx(g, t % n, (t / n) % n, D == 3 ? t / (n * n) : 0)] = acc;
    }
}

// RHS pass 1: v and w of Eq. (5), pointwise (CD4 reads radius 2)
template <int D>
__global__ void k_vw(double *__restrict__ V, double *__restrict__ W, VWParams P) {
    const GridDesc &g = P.g;
    POINT_INDEX_OR_RETURN(g)
    if (!inside) return;
    long long p = gidx(g, i, j, k);
    double acc = P.beta[0] * P.uold[0][p];
    for (int jj = 1; jj < P.M; ++jj) acc = acc + P.beta[jj] * P.uold[jj][p];
    W[p] = acc - P.gm * P.uold[P.m + 1][p];
    if (P.fe.kind == 0) {
        V[p] = P.unew_m[p];
    } else if (P.F[0]) {            // the same tree on stored f^E values
        double fa = P.a[0] * P.F[0][p];
        for (int jj = 1; jj < P.M; ++jj) fa = fa + P.a[jj] * P.F[jj][p];
        V[p] = (P.unew_m[p] + P.dtm * (P.Fn[p] - P.F[P.m][p])) + fa;
    } else {
        double fa = P.a[0] * fe_at<D>(P.fe, P.uold[0], g, i, j, k, P.ct[0]);
        for (int jj = 1; jj < P.M; ++jj) fa = fa + P.a[jj] * fe_at<D>(P.fe, P.uold[jj], g, i, j, k, P.ct[jj]);
        double fn = fe_at<D>(P.fe, P.unew_m, g, i, j, k, *P.ctn);
        double fo = fe_at<D>(P.fe, P.uold[P.m], g, i, j, k, P.ct[P.m]);
        V[p] = (P.unew_m[p] + P.dtm * (fn - fo)) + fa;
    }
}

// RHS pass 2: b = B v + L w; optional ||b||_inf into *slot
template <int D>
__global__ void k_bvw(double *__restrict__ Bout, const double *__restrict__ V, const double *__restrict__ W,
                      GridDesc g, BLConst c, unsigned long long *slot) {
    POINT_INDEX_OR_RETURN(g)
    double val = 0.0;
    if (inside) {
        val = apply_B<D>(c, V, g, i, j, k) + apply_L<D>(c, W, g, i, j, k);
        Bout[gidx(g, i, j, k)] = val;
    }
    if (slot) block_max_to(slot, fabs(val));
}

// residual pass 1 for node m: p = (u_m - u_0) - sum qa_j fE(u_j),  z = sum qb_j u_j
template <int D>
__global__ void k_pz(double *__restrict__ Pf, double *__restrict__ Zf, PZParams P) {
    const GridDesc &g = P.g;
    POINT_INDEX_OR_RETURN(g)
    if (!inside) return;
    long long p = gidx(g, i, j, k);
    double diff = P.u[P.m][p] - P.u[0][p];
    if (P.fe.kind != 0 && P.F[0]) {
        double fa = P.qa[0] * P.F[0][p];
        for (int jj = 1; jj < P.M; ++jj) fa = fa + P.qa[jj] * P.F[jj][p];
        diff = diff - fa;
    } else if (P.fe.kind != 0) {
        double fa = P.qa[0] * fe_at<D>(P.fe, P.u[0], g, i, j, k, P.ct[0]);
        for (int jj = 1; jj < P.M; ++jj) fa = fa + P.qa[jj] * fe_at<D>(P.fe, P.u[jj], g, i, j, k, P.ct[jj]);
        diff = diff - fa;
    }
    Pf[p] = diff;
    double acc = P.qb[0] * P.u[0][p];
    for (int jj = 1; jj < P.M; ++jj) acc = acc + P.qb[jj] * P.u[jj][p];
    Zf[p] = acc;
}

// residual pass 2: r = B p - L z, ||r||_inf into *slot
template <int D>
__global__ void k_resid(const double *__restrict__ Pf, const double *__restrict__ Zf, GridDesc g, BLConst c,
                        unsigned long long *slot, double *__restrict__ out) {
    POINT_INDEX_OR_RETURN(g)
    double val = 0.0;
    if (inside) {
        val = apply_B<D>(c, Pf, g, i, j, k) - apply_L<D>(c, Zf, g, i, j, k);
        if (out) out[gidx(g, i, j, k)] = val;   // r~ field (unweighted residual)
    }
    block_max_to(slot, fabs(val));
}

// f^E(u) into a stored field (generic; Burgers: aux = the alpha slot of u, else cos t unused)
template <int D>
__global__ void k_fe(double *__restrict__ F, const double *__restrict__ u, GridDesc g, FeDesc fe,
                     const unsigned long long *aux) {
    POINT_INDEX_OR_RETURN(g)
    if (!inside) return;
    const double a = __longlong_as_double((long long)*aux);
    F[gidx(g, i, j, k)] = fe_at<D>(fe, u, g, i, j, k, a);
}
