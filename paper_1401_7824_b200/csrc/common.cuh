// common.cuh -- shared device definitions of libisdc (grid descriptors, coefficient structs,
// canonical stencil trees, max-norm reduction).  See DESIGN.md §4 for the canonical arithmetic.
//
// Compiled with --fmad=false: every a*b+c is a rounded multiply followed by a rounded add,
// exactly as in the CPU oracle (-ffp-contract=off), so results are bit-identical.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define ISDC_MAXM 8

// A pitched interior-only field on one level: point (i,j,k) at i + pitch*j + plane*k,
// pitch = n+1 (a power of two), plane = n*pitch (3D).  Values outside 0..n-1 are the
// homogeneous Dirichlet data (zero) and are never stored.  Periodic grids (per = 1, NEXT f3):
// n = 2^p points, pitch = n, indices wrap modulo n (stencil offsets never exceed n).
struct GridDesc {
    int n;
    int pitch;
    long long plane;
    int per;
};

// Node-system coefficients on one level:
//   S u = (c0*u + c1*faces) + c2*edges,  Jacobi: u + wd*(b - S u)
struct SCoef {
    double c0, c1, c2, wd;
};

// Compact pair constants: B q = kB0 q + kB1 faces;  L q = (kL0 q + kL1 faces) + kL2 edges
struct BLConst {
    double kB0, kB1, kL0, kL1, kL2;
};

// f^E description
struct FeDesc {
    int kind;            // 0 none, 1 cubic, 2 forcing, 3 advection CD4, 4 Burgers WENO5 (periodic)
    double kx, ky, kz;   // CD4: a_a * N / 12
    double kh;           // Burgers: 1/h
    const double *G;     // forcing profile (pitched), or null
};

__device__ __forceinline__ long long gidx(const GridDesc &g, int i, int j, int k) {
    return (long long)i + (long long)g.pitch * j + g.plane * k;
}

__device__ __forceinline__ int wrapn(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

template <int D>
__device__ __forceinline__ double ldz(const double *__restrict__ q, const GridDesc &g, int i, int j, int k) {
    if (g.per) {
        i = wrapn(i, g.n); j = wrapn(j, g.n);
        if (D == 3) k = wrapn(k, g.n);
    }
    if (i < 0 || j < 0 || i >= g.n || j >= g.n) return 0.0;
    if (D == 3 && (k < 0 || k >= g.n)) return 0.0;
    return q[gidx(g, i, j, D == 3 ? k : 0)];
}

// ---- canonical trees, evaluated from global memory (generic/reference kernels) -------------
template <int D>
__device__ __forceinline__ double tr_r(const double *q, const GridDesc &g, int i, int j, int k) {
    return ldz<D>(q, g, i - 1, j, k) + ldz<D>(q, g, i + 1, j, k);
}
template <int D>
__device__ __forceinline__ double tr_f(const double *q, const GridDesc &g, int i, int j, int k) {
    return tr_r<D>(q, g, i, j, k) + (ldz<D>(q, g, i, j - 1, k) + ldz<D>(q, g, i, j + 1, k));
}
template <int D>
__device__ __forceinline__ double tr_e(const double *q, const GridDesc &g, int i, int j, int k) {
    return tr_r<D>(q, g, i, j - 1, k) + tr_r<D>(q, g, i, j + 1, k);
}
template <int D>
__device__ __forceinline__ double tr_faces(const double *q, const GridDesc &g, int i, int j, int k) {
    if (D == 2) return tr_f<D>(q, g, i, j, k);
    return tr_f<D>(q, g, i, j, k) + (ldz<D>(q, g, i, j, k - 1) + ldz<D>(q, g, i, j, k + 1));
}
template <int D>
__device__ __forceinline__ double tr_edges(const double *q, const GridDesc &g, int i, int j, int k) {
    if (D == 2) return tr_e<D>(q, g, i, j, k);
    return tr_e<D>(q, g, i, j, k) + (tr_f<D>(q, g, i, j, k - 1) + tr_f<D>(q, g, i, j, k + 1));
}
template <int D>
__device__ __forceinline__ double apply_S(const SCoef &c, const double *u, const GridDesc &g, int i, int j, int k) {
    return (c.c0 * ldz<D>(u, g, i, j, k) + c.c1 * tr_faces<D>(u, g, i, j, k)) + c.c2 * tr_edges<D>(u, g, i, j, k);
}
template <int D>
__device__ __forceinline__ double apply_B(const BLConst &c, const double *q, const GridDesc &g, int i, int j, int k) {
    return c.kB0 * ldz<D>(q, g, i, j, k) + c.kB1 * tr_faces<D>(q, g, i, j, k);
}
template <int D>
__device__ __forceinline__ double apply_L(const BLConst &c, const double *q, const GridDesc &g, int i, int j, int k) {
    return (c.kL0 * ldz<D>(q, g, i, j, k) + c.kL1 * tr_faces<D>(q, g, i, j, k)) + c.kL2 * tr_edges<D>(q, g, i, j, k);
}

// WENO5-JS face value between v2 and v3 (reading R31): the canonical tree
__device__ __noinline__ double weno5(double v0, double v1, double v2, double v3, double v4) {
    const double eps = 1e-6, c13 = 13.0 / 12.0;
    double p0 = ((2.0 * v0 - 7.0 * v1) + 11.0 * v2) / 6.0;
    double p1 = ((5.0 * v2 - v1) + 2.0 * v3) / 6.0;
    double p2 = ((2.0 * v2 + 5.0 * v3) - v4) / 6.0;
    double s0 = (v0 - 2.0 * v1) + v2, t0 = (v0 - 4.0 * v1) + 3.0 * v2;
    double s1 = (v1 - 2.0 * v2) + v3, t1 = v1 - v3;
    double s2 = (v2 - 2.0 * v3) + v4, t2 = (3.0 * v2 - 4.0 * v3) + v4;
    double b0 = c13 * (s0 * s0) + 0.25 * (t0 * t0);
    double b1 = c13 * (s1 * s1) + 0.25 * (t1 * t1);
    double b2 = c13 * (s2 * s2) + 0.25 * (t2 * t2);
    double e0 = eps + b0, e1 = eps + b1, e2 = eps + b2;
    double a0 = 0.1 / (e0 * e0), a1 = 0.6 / (e1 * e1), a2 = 0.3 / (e2 * e2);
    return ((a0 * p0 + a1 * p1) + a2 * p2) / ((a0 + a1) + a2);
}
// Lax-Friedrichs split flux of u^2/2: (q +- alpha*u)*0.5, q = (u*u)*0.5
__device__ __forceinline__ double split_flux(double x, double alpha, bool plus) {
    double q = (x * x) * 0.5, a = alpha * x;
    return plus ? (q + a) * 0.5 : (q - a) * 0.5;
}
// numerical flux through the face between s and s+1 along axis (di,dj,dk)
template <int D>
__device__ __forceinline__ double burgers_face(const double *u, const GridDesc &g, int i, int j, int k, int di, int dj,
                                               int dk, double alpha) {
    double fp[5], fm[5];
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        int o = s - 2, q = 3 - s;
        fp[s] = split_flux(ldz<D>(u, g, i + o * di, j + o * dj, k + o * dk), alpha, true);
        fm[s] = split_flux(ldz<D>(u, g, i + q * di, j + q * dj, k + q * dk), alpha, false);
    }
    return weno5(fp[0], fp[1], fp[2], fp[3], fp[4]) + weno5(fm[0], fm[1], fm[2], fm[3], fm[4]);
}

// f^E at a point; aux = cos(t_j) for the forcing kind, alpha = max|u| for Burgers
template <int D>
__device__ __forceinline__ double fe_at(const FeDesc &fe, const double *u, const GridDesc &g, int i, int j, int k,
                                        double ct) {
    if (fe.kind == 4) {
        double gx = burgers_face<D>(u, g, i, j, k, 1, 0, 0, ct) - burgers_face<D>(u, g, i - 1, j, k, 1, 0, 0, ct);
        double gy = burgers_face<D>(u, g, i, j, k, 0, 1, 0, ct) - burgers_face<D>(u, g, i, j - 1, k, 0, 1, 0, ct);
        double sum = gx + gy;
        if (D == 3)
            sum = sum + (burgers_face<D>(u, g, i, j, k, 0, 0, 1, ct) - burgers_face<D>(u, g, i, j, k - 1, 0, 0, 1, ct));
        return -(sum * fe.kh);
    }
    if (fe.kind == 1) {
        double x = u[gidx(g, i, j, k)];
        return x - (x * x) * x;
    }
    if (fe.kind == 2) return fe.G[gidx(g, i, j, k)] * ct;
    // CD4 advection, zero ghosts beyond the boundary
    double dx = (8.0 * (ldz<D>(u, g, i + 1, j, k) - ldz<D>(u, g, i - 1, j, k)) -
                 (ldz<D>(u, g, i + 2, j, k) - ldz<D>(u, g, i - 2, j, k))) * fe.kx;
    double dy = (8.0 * (ldz<D>(u, g, i, j + 1, k) - ldz<D>(u, g, i, j - 1, k)) -
                 (ldz<D>(u, g, i, j + 2, k) - ldz<D>(u, g, i, j - 2, k))) * fe.ky;
    if (D == 2) return -(dx + dy);
    double dz = (8.0 * (ldz<D>(u, g, i, j, k + 1) - ldz<D>(u, g, i, j, k - 1)) -
                 (ldz<D>(u, g, i, j, k + 2) - ldz<D>(u, g, i, j, k - 2))) * fe.kz;
    return -((dx + dy) + dz);
}

// ---- named barrier over `count` threads (warp-specialised kernels: the roles reach it from
// different code locations; count is a multiple of 32)
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- max-norm reduction: non-negative doubles ordered as uint64; NaN bits exceed +Inf ---------
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}
// running max of absolute values that keeps NaN (bits of a positive NaN exceed +Inf)
__device__ __forceinline__ double amax(double acc, double absval) {
    unsigned long long a = (unsigned long long)__double_as_longlong(acc);
    unsigned long long b = (unsigned long long)__double_as_longlong(absval);
    return __longlong_as_double((long long)(a > b ? a : b));
}
// every thread of the block must call; one atomicMax per block into *slot
__device__ __forceinline__ void block_max_to(unsigned long long *slot, double absval) {
    __shared__ unsigned long long red_s[32];
    unsigned long long v = (unsigned long long)__double_as_longlong(absval);
    v = warp_max_u64(v);
    int lane = threadIdx.x & 31;
    int wid = (threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z)) >> 5;
    int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    int nw = (blockDim.x * blockDim.y * blockDim.z + 31) >> 5;
    (void)lane;
    if ((tid & 31) == 0) red_s[wid] = v;
    __syncthreads();
    if (tid < 32) {
        unsigned long long w = tid < nw ? red_s[tid] : 0ull;
        w = warp_max_u64(w);
        if (tid == 0 && w) atomicMax(slot, w);
    }
}
