// kernels_mlsdc.cuh -- the transfers and the FAS correction of two-level MLSDC with ISDC sweeps
// (NEXT f4; "SDC sweeps in a multigrid-like way on multiple levels ... connected through
// an FAS correction term"; reading R32).  One point per thread; these run once per node
// per MLSDC iteration (the sweeps themselves use the tuned kernels).  Canonical trees of DESIGN.md
// §4.7, the same as the oracle's (bit-identical).  Dirichlet grids: coarse I <-> fine 2I+1.
#pragma once
#include "common.cuh"

// injection: coarse (I,J,K) <- fine (2I+1, 2J+1, 2K+1)
template <int D>
__global__ void k_inject(double *__restrict__ uc, GridDesc gc, const double *__restrict__ uf, GridDesc gf) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y * blockDim.y + threadIdx.y;
    const int K = (D == 3) ? (int)blockIdx.z : 0;
    if (I >= gc.n || J >= gc.n) return;
    uc[gidx(gc, I, J, K)] = uf[gidx(gf, 2 * I + 1, 2 * J + 1, D == 3 ? 2 * K + 1 : 0)];
}

// full weighting of a fine field r at coarse (I,J,K) (the restriction tree of DESIGN.md §4.2)
template <int D>
__device__ __forceinline__ double fw_field(const double *r, const GridDesc &gf, int I, int J, int K) {
    const int x = 2 * I + 1, y = 2 * J + 1, z = (D == 3) ? 2 * K + 1 : 0;
    if (D == 2) {
        double d[3][3];
#pragma unroll
        for (int b_ = 0; b_ < 3; ++b_)
#pragma unroll
            for (int a_ = 0; a_ < 3; ++a_) d[b_][a_] = ldz<D>(r, gf, x - 1 + a_, y - 1 + b_, 0);
        const double rd0 = d[0][0] + d[0][2], rd1 = d[1][0] + d[1][2], rd2 = d[2][0] + d[2][2];
        const double fd = rd1 + (d[0][1] + d[2][1]);
        const double ed = rd0 + rd2;
        return ((4.0 * d[1][1] + 2.0 * fd) + ed) * 0.0625;
    } else {
        double fd[3], ed[3], dc[3];
#pragma unroll
        for (int c_ = 0; c_ < 3; ++c_) {
            double d[3][3];
#pragma unroll
            for (int b_ = 0; b_ < 3; ++b_)
#pragma unroll
                for (int a_ = 0; a_ < 3; ++a_) d[b_][a_] = ldz<D>(r, gf, x - 1 + a_, y - 1 + b_, z - 1 + c_);
            const double rd0 = d[0][0] + d[0][2], rd1 = d[1][0] + d[1][2], rd2 = d[2][0] + d[2][2];
            fd[c_] = rd1 + (d[0][1] + d[2][1]);
            ed[c_] = rd0 + rd2;
            dc[c_] = d[1][1];
        }
        const double F = fd[1] + (dc[0] + dc[2]);
        const double E = ed[1] + (fd[0] + fd[2]);
        const double C = ed[0] + ed[2];
        return ((8.0 * dc[1] + 4.0 * F) + (2.0 * E + C)) * 0.015625;
    }
}

// FAS correction of node m: fas = r~_H(R_i u)_m - R_fw r~_h,m
template <int D>
__global__ void k_fas(double *__restrict__ fas, GridDesc gc, const double *__restrict__ rH,
                      const double *__restrict__ rh, GridDesc gf) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y * blockDim.y + threadIdx.y;
    const int K = (D == 3) ? (int)blockIdx.z : 0;
    if (I >= gc.n || J >= gc.n) return;
    const long long p = gidx(gc, I, J, K);
    fas[p] = rH[p] - fw_field<D>(rh, gf, I, J, K);
}

// coarse RHS of substep m: b = b + (fas_{m+1} - fas_m), fas_0 = 0 (f0 == nullptr)
template <int D>
__global__ void k_add_fas(double *__restrict__ b, GridDesc g, const double *__restrict__ f1,
                          const double *__restrict__ f0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = (D == 3) ? (int)blockIdx.z : 0;
    if (i >= g.n || j >= g.n) return;
    const long long p = gidx(g, i, j, k);
    b[p] = b[p] + (f1[p] - (f0 ? f0[p] : 0.0));
}

// e = a - b (the coarse correction U_j - Ubar_j)
template <int D>
__global__ void k_sub(double *__restrict__ e, GridDesc g, const double *__restrict__ a, const double *__restrict__ b) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = (D == 3) ? (int)blockIdx.z : 0;
    if (i >= g.n || j >= g.n) return;
    const long long p = gidx(g, i, j, k);
    e[p] = a[p] - b[p];
}

// 4th-order interpolation P4 along one axis: a fine odd index 2I+1 takes the coarse
// value I; a fine even index x between coarse a = x/2-1 and b = x/2 takes the cubic midpoint
// (9*(c(a) + c(b)) - (c(a-1) + c(b+1))) * 0.0625, c(-1) = c(nc) = 0, c(-2) = -c(0), c(nc+1) = -c(nc-1).
__device__ __forceinline__ double p4_c(const double *row, long long stride, int nc, int i) {
    if (i >= 0 && i < nc) return row[(long long)i * stride];
    if (i == -1 || i == nc) return 0.0;
    if (i == -2) return -row[0];
    return -row[(long long)(nc - 1) * stride];
}
__device__ __forceinline__ double p4_interp(const double *row, long long stride, int nc, int x) {
    if (x & 1) return row[(long long)((x - 1) / 2) * stride];
    const int a = x / 2 - 1, b = x / 2;
    return (9.0 * (p4_c(row, stride, nc, a) + p4_c(row, stride, nc, b)) -
            (p4_c(row, stride, nc, a - 1) + p4_c(row, stride, nc, b + 1))) * 0.0625;
}

// pass x: T1[(K*nc + J)*nf + x] = P4_x of the coarse row (J, K) of e (pitched, gc)
template <int D>
__global__ void k_p4x(double *__restrict__ T1, const double *__restrict__ e, GridDesc gc, int nf) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y * blockDim.y + threadIdx.y;
    const int K = (D == 3) ? (int)blockIdx.z : 0;
    const int nc = gc.n;
    if (x >= nf || J >= nc) return;
    T1[((long long)K * nc + J) * nf + x] = p4_interp(e + gidx(gc, 0, J, K), 1, nc, x);
}
// pass y: 2D adds into u (pitched, gf); 3D writes T2[(K*nf + y)*nf + x]
template <int D>
__global__ void k_p4y(double *__restrict__ out, const double *__restrict__ T1, int nc, GridDesc gf) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
    const int K = (D == 3) ? (int)blockIdx.z : 0;
    const int nf = gf.n;
    if (x >= nf || y >= nf) return;
    const double v = p4_interp(T1 + (long long)K * nc * nf + x, nf, nc, y);
    if (D == 2) {
        const long long p = gidx(gf, x, y, 0);
        out[p] = out[p] + v;
    } else {
        out[((long long)K * nf + y) * nf + x] = v;
    }
}
// pass z (3D): u = u + P4_z of T2
__global__ void k_p4z(double *__restrict__ u, const double *__restrict__ T2, int nc, GridDesc gf) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
    const int z = blockIdx.z;
    const int nf = gf.n;
    if (x >= nf || y >= nf) return;
    const double v = p4_interp(T2 + (long long)y * nf + x, (long long)nf * nf, nc, z);
    const long long p = gidx(gf, x, y, z);
    u[p] = u[p] + v;
}
