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
// homogeneous Dirichlet data (zero) and are never stored.
struct GridDesc {
    int n;
    int pitch;
    long long plane;
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
    int kind;            // 0 none, 1 cubic, 2 forcing, 3 advection CD4
    double kx, ky, kz;   // CD4: a_a * N / 12
    const double *G;     // forcing profile (pitched), or null
};

__device__ __forceinline__ long long gidx(const GridDesc &g, int i, int j, int k) {
    return (long long)i + (long long)g.pitch * j + g.plane * k;
}

template <int D>
__device__ __forceinline__ double ldz(const double *__restrict__ q, const GridDesc &g, int i, int j, int k) {
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

// f^E at a point; ct = cos(t_j) for the forcing kind
template <int D>
__device__ __forceinline__ double fe_at(const FeDesc &fe, const double *u, const GridDesc &g, int i, int j, int k,
                                        double ct) {
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

// ---- programmatic dependent launch (sm_90+): kernels are launched with programmatic stream
// serialization, so a kernel may start while its predecessor drains.  Every kernel calls
// pdl_launch() at entry (lets its own successor launch early) and pdl_wait() before its first
// global-memory access (waits for the predecessor's completion and memory flush); only shared
// memory / parameter work may precede pdl_wait().
__device__ __forceinline__ void pdl_launch() {}   // implicit trigger at CTA exit (an early trigger measured slower: waiting successor CTAs hold SM resources)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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
