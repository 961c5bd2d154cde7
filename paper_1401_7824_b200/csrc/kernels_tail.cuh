// kernels_tail.cuh -- the coarse-level tail of the V-cycle in ONE single-CTA launch.
//
// All levels with n <= tail_n (2D: 63, 3D: 15) live in shared memory as dense arrays with a
// zero ring (the homogeneous Dirichlet data), and the whole down-up recursion -- weighted-Jacobi
// sweeps, defect + full weighting, exact 3^d solve, prolongation + correction -- runs between
// __syncthreads() barriers, replacing ~7 launches per level.  Arithmetic is the canonical trees
// of DESIGN.md §4, identical to the per-level kernels.
#pragma once
#include "common.cuh"

constexpr int TAIL_MAX_LEVELS = 6;
constexpr int TAIL_THREADS = 1024;

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
};

// a zero-ringed level array in shared memory
template <int D>
struct PL {
    double *p;
    int n, np;
    __device__ __forceinline__ int idx(int i, int j, int k) const {
        return (i + 1) + np * ((j + 1) + (D == 3 ? np * (k + 1) : 0));
    }
    __device__ __forceinline__ double at(int i, int j, int k) const { return p[idx(i, j, k)]; }
    __device__ __forceinline__ double r(int i, int j, int k) const { return at(i - 1, j, k) + at(i + 1, j, k); }
    __device__ __forceinline__ double f(int i, int j, int k) const {
        return r(i, j, k) + (at(i, j - 1, k) + at(i, j + 1, k));
    }
    __device__ __forceinline__ double e(int i, int j, int k) const { return r(i, j - 1, k) + r(i, j + 1, k); }
    __device__ __forceinline__ double faces(int i, int j, int k) const {
        if (D == 2) return f(i, j, k);
        return f(i, j, k) + (at(i, j, k - 1) + at(i, j, k + 1));
    }
    __device__ __forceinline__ double edges(int i, int j, int k) const {
        if (D == 2) return e(i, j, k);
        return e(i, j, k) + (f(i, j, k - 1) + f(i, j, k + 1));
    }
    __device__ __forceinline__ double S(const SCoef &c, int i, int j, int k) const {
        return (c.c0 * at(i, j, k) + c.c1 * faces(i, j, k)) + c.c2 * edges(i, j, k);
    }
};

template <int D>
__host__ __device__ __forceinline__ int tail_padded(int n) {
    return D == 3 ? (n + 2) * (n + 2) * (n + 2) : (n + 2) * (n + 2);
}

// loop over the interior points of an n^D level assigned to this thread
#define TAIL_FOR(D, n, ...)                                                                    \
    do {                                                                                        \
        if (D == 2) {                                                                           \
            for (int j_ = threadIdx.x >> 5; j_ < (n); j_ += 32)                                 \
                for (int i_ = threadIdx.x & 31; i_ < (n); i_ += 32) {                           \
                    const int i = i_, j = j_, k = 0;                                            \
                    __VA_ARGS__                                                                 \
                }                                                                               \
        } else {                                                                                \
            for (int k_ = threadIdx.x >> 7; k_ < (n); k_ += 8)                                  \
                for (int j_ = (threadIdx.x >> 4) & 7; j_ < (n); j_ += 8)                        \
                    for (int i_ = threadIdx.x & 15; i_ < (n); i_ += 16) {                       \
                        const int i = i_, j = j_, k = k_;                                       \
                        __VA_ARGS__                                                             \
                    }                                                                           \
        }                                                                                       \
    } while (0)

template <int D>
__global__ void __launch_bounds__(TAIL_THREADS) k_tail(TailParams P) {
    extern __shared__ __align__(16) double tsm[];
    const int L = P.nlev;
    // zero everything once: the rings stay zero for the whole kernel
    {
        int tot = 0;
        for (int l = 0; l < L; ++l) tot += 3 * tail_padded<D>(P.n[l]);
        for (int q = threadIdx.x; q < tot; q += TAIL_THREADS) tsm[q] = 0.0;
    }
    auto level_base = [&](int l) -> double * {
        double *p = tsm;
        for (int q = 0; q < l; ++q) p += 3 * tail_padded<D>(P.n[q]);
        return p;
    };
    // buffer w in {0,1} = iterate ping-pong, 2 = right-hand side
    auto lv = [&](int l, int w) -> PL<D> {
        PL<D> a;
        a.n = P.n[l];
        a.np = a.n + 2;
        a.p = level_base(l) + w * tail_padded<D>(a.n);
        return a;
    };
    __syncthreads();
    {
        PL<D> U = lv(0, 0), B = lv(0, 2);
        const int n = U.n;
        TAIL_FOR(D, n, {
            long long gi = (long long)i + (long long)P.pitch * (j + (D == 3 ? (long long)n * k : 0));
            B.p[B.idx(i, j, k)] = P.b_in[gi];
            if (P.u_in) U.p[U.idx(i, j, k)] = P.u_in[gi];
        });
    }
    __syncthreads();
    unsigned cur = 0;   // bit l: iterate of level l is in buffer 1
    auto smooth = [&](int l, int sweeps) {
        const SCoef c = P.c[l];
        PL<D> B = lv(l, 2);
        for (int s = 0; s < sweeps; ++s) {
            int w = (cur >> l) & 1;
            PL<D> in = lv(l, w), out = lv(l, 1 - w);
            const int n = in.n;
            TAIL_FOR(D, n, {
                int q = in.idx(i, j, k);
                out.p[q] = in.p[q] + c.wd * (B.p[q] - in.S(c, i, j, k));
            });
            cur ^= 1u << l;
            __syncthreads();
        }
    };
    // ---------------- down
    for (int l = 0; l < L - 1; ++l) {
        smooth(l, P.nu1);
        int w = (cur >> l) & 1;
        PL<D> u = lv(l, w), d = lv(l, 1 - w), B = lv(l, 2), Bc = lv(l + 1, 2);
        const SCoef c = P.c[l];
        const int n = u.n, nc = Bc.n;
        TAIL_FOR(D, n, {
            int q = u.idx(i, j, k);
            d.p[q] = B.p[q] - u.S(c, i, j, k);
        });
        __syncthreads();
        TAIL_FOR(D, nc, {
            const int x = 2 * i + 1, y = 2 * j + 1, z = D == 3 ? 2 * k + 1 : 0;
            double v;
            if (D == 2) {
                v = ((4.0 * d.at(x, y, 0) + 2.0 * d.f(x, y, 0)) + d.e(x, y, 0)) * 0.0625;
            } else {
                double co = d.e(x, y, z - 1) + d.e(x, y, z + 1);
                v = ((8.0 * d.at(x, y, z) + 4.0 * d.faces(x, y, z)) + (2.0 * d.edges(x, y, z) + co)) * 0.015625;
            }
            Bc.p[Bc.idx(i, j, k)] = v;
        });
        __syncthreads();
        // the next level starts from a zero iterate (its buffers are zero except where written;
        // buffer 0 of level l+1 has never been written at this point of the down sweep)
    }
    // ---------------- coarsest: exact solve u = Ginv b, ascending-j accumulation
    {
        constexpr int Pc = D == 3 ? 27 : 9;
        const int l = L - 1;
        PL<D> u = lv(l, 0), B = lv(l, 2);
        if (threadIdx.x < Pc) {
            const int t = threadIdx.x;
            auto bb = [&](int q) { return B.at(q % 3, (q / 3) % 3, D == 3 ? q / 9 : 0); };
            double acc = P.Ginv[t * Pc] * bb(0);
            for (int jj = 1; jj < Pc; ++jj) acc = acc + P.Ginv[t * Pc + jj] * bb(jj);
            u.p[u.idx(t % 3, (t / 3) % 3, D == 3 ? t / 9 : 0)] = acc;
        }
        cur &= ~(1u << l);
        __syncthreads();
    }
    // ---------------- up
    for (int l = L - 2; l >= 0; --l) {
        PL<D> e = lv(l + 1, (cur >> (l + 1)) & 1), u = lv(l, (cur >> l) & 1);
        const int n = u.n;
        TAIL_FOR(D, n, {
            int xa, xb, ya, yb, za = 0, zb = 0;
            bool xe = !(i & 1), ye = !(j & 1), ze = (D == 3) && !(k & 1);
            double w = 1.0;
            if (xe) { xa = i / 2 - 1; xb = i / 2; w *= 0.5; } else { xa = xb = (i - 1) / 2; }
            if (ye) { ya = j / 2 - 1; yb = j / 2; w *= 0.5; } else { ya = yb = (j - 1) / 2; }
            if (D == 3) {
                if (ze) { za = k / 2 - 1; zb = k / 2; w *= 0.5; } else { za = zb = (k - 1) / 2; }
            }
            double sz = 0.0;
            for (int cz = 0; cz < ((D == 3 && ze) ? 2 : 1); ++cz) {
                int Z = cz ? zb : za;
                double sy = 0.0;
                for (int cy = 0; cy < (ye ? 2 : 1); ++cy) {
                    int Y = cy ? yb : ya;
                    double sx = e.at(xa, Y, Z);
                    if (xe) sx = sx + e.at(xb, Y, Z);
                    sy = cy ? sy + sx : sx;
                }
                sz = cz ? sz + sy : sy;
            }
            int q = u.idx(i, j, k);
            u.p[q] = u.p[q] + sz * w;
        });
        __syncthreads();
        smooth(l, P.nu2);
    }
    // ---------------- write the level-0 result
    {
        PL<D> u = lv(0, cur & 1);
        const int n = u.n;
        TAIL_FOR(D, n, {
            long long gi = (long long)i + (long long)P.pitch * (j + (D == 3 ? (long long)n * k : 0));
            P.u_out[gi] = u.at(i, j, k);
        });
    }
}

template <int D>
inline size_t tail_smem_bytes(const TailParams &P) {
    size_t s = 0;
    for (int l = 0; l < P.nlev; ++l) s += 3 * (size_t)tail_padded<D>(P.n[l]);
    return s * sizeof(double);
}
