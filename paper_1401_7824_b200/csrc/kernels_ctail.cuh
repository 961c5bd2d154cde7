// kernels_ctail.cuh -- the coarse-level tail of the V-cycle as ONE thread-block-cluster launch
// (the north star's "coarse-level tail that runs the small grids in one
// persistent/cluster launch").  A cluster of CT_CS = 16 CTAs (one per SM, 1024 threads each) holds
// every level from n0 (2D: 255, 3D: 31) down to 3 in distributed shared memory:
//   * distributed levels (n >= 15, n + 1 = 16 B): CTA r owns rows (2D) / planes (3D)
//     [r B, r B + B) of each array, stored as a padded block with one ghost row / plane on each
//     side (zero at the domain boundary); after every phase that writes a stencilled array the
//     CTAs pass a cluster barrier and copy their neighbours' edge rows into their ghosts (DSMEM);
//   * local levels (n <= 7): CTA 0 alone, full padded arrays, __syncthreads between phases (the
//     other CTAs wait at the next cluster barrier).  The last distributed level's defect is
//     gathered into CTA 0 for the restriction; CTA 0's coarse result is copied to every CTA for
//     the prolongation.
// Restriction between distributed levels is local: with B_f = 2 B_c a coarse row J of CTA r needs
// the fine rows 2J .. 2J + 2, i.e. its own block and its upper ghost; the prolongation needs the
// coarse block and its lower ghost.  Every value is formed by the canonical trees of DESIGN.md §4
// -- the expressions of kernels_tail.cuh (k_tail), on the same operands -- so the result is
// bit-identical to the per-level kernels and the single-CTA tail.
#pragma once
#include "common.cuh"
#include <cooperative_groups.h>

constexpr int CT_CS = 16;                 // CTAs per cluster (non-portable size)
constexpr int CT_THREADS = 1024;
constexpr int CT_WARPS = CT_THREADS / 32;
constexpr int CT_MAX_LEVELS = 8;

struct CTailParams {
    int nlev;                    // levels n0, (n0-1)/2, ..., 3
    int ndist;                   // levels 0 .. ndist-1 are distributed (n >= 15), the rest local
    int n[CT_MAX_LEVELS];
    SCoef c[CT_MAX_LEVELS];
    int nu1, nu2;
    const double *Ginv;          // P x P inverse of the 3^d operator
    const double *b_in;          // pitched level-n0 right-hand side (global)
    const double *u_in;          // pitched initial iterate, or null for zero
    double *u_out;               // pitched result
    int pitch;
};

// An array of one level as seen by this CTA: element (i, j[, k]) of the level, with the
// distributed index q = j (2D) / k (3D) in [r0 - 1, r0 + B], lives at
//   2D: (q - r0 + 1) np + i + 1            3D: ((q - r0 + 1) np + j + 1) np + i + 1
// np = n + 2.  A full local array is the case r0 = 0, B = n.
struct CtArr {
    double *p;
    int r0;
};

template <int D>
__host__ __device__ __forceinline__ int ct_rowsize(int n) { return D == 3 ? (n + 2) * (n + 2) : (n + 2); }

template <int D>
__device__ __forceinline__ int ct_off(int n, int r0, int i, int j, int k) {
    const int np = n + 2;
    return D == 2 ? (j - r0 + 1) * np + i + 1 : ((k - r0 + 1) * np + j + 1) * np + i + 1;
}

// canonical S u at offset o (the tree of tail_S)
template <int D>
__device__ __forceinline__ double ct_S(const double *__restrict__ a, int o, int np, const SCoef &c) {
    const double rc = a[o - 1] + a[o + 1];
    const double rm = a[o - np - 1] + a[o - np + 1];
    const double rp = a[o + np - 1] + a[o + np + 1];
    const double f = rc + (a[o - np] + a[o + np]);
    const double e = rm + rp;
    if (D == 2) return (c.c0 * a[o] + c.c1 * f) + c.c2 * e;
    const int pl = np * np, ol = o - pl, ou = o + pl;
    const double fl = (a[ol - 1] + a[ol + 1]) + (a[ol - np] + a[ol + np]);
    const double fu = (a[ou - 1] + a[ou + 1]) + (a[ou - np] + a[ou + np]);
    const double faces = f + (a[ol] + a[ou]);
    const double edges = e + (fl + fu);
    return (c.c0 * a[o] + c.c1 * faces) + c.c2 * edges;
}

// out(o) = fn(o, i, j, k) over the points of rows/planes q in [q0, q1) of an n^D level held with
// origin r0: tasks = (q, row, 32-column chunk) spread over the warps, lanes over the columns.
// `out` is never read by fn (ping-pong), so every point is stored as soon as it is formed.
template <int D, typename F>
__device__ __forceinline__ void ct_map(int n, int r0, int q0, int q1, double *__restrict__ out, F fn) {
    if (q1 <= q0) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int chunks = (n + 31) >> 5;
    const int rows = (D == 3) ? n : 1;                   // rows per plane (3D)
    const int tasks = (q1 - q0) * rows * chunks;
    for (int t = w; t < tasks; t += CT_WARPS) {
        const int ch = t % chunks, qr = t / chunks;
        const int j = (D == 3) ? qr % rows : q0 + qr;
        const int k = (D == 3) ? q0 + qr / rows : 0;
        const int i = ch * 32 + lane;
        if (i < n) {
            const int o = ct_off<D>(n, r0, i, j, k);
            out[o] = fn(o, i, j, k);
        }
    }
}

// ------------------------------------------------------------------------------ phases
template <int D>
__device__ __noinline__ void ct_sweep(const double *in, double *out, const double *B, int n, int r0, int q0, int q1,
                                      SCoef c) {
    const int np = n + 2;
    ct_map<D>(n, r0, q0, q1, out, [&](int o, int, int, int) { return in[o] + c.wd * (B[o] - ct_S<D>(in, o, np, c)); });
}
template <int D>
__device__ __noinline__ void ct_defect(const double *u, double *d, const double *B, int n, int r0, int q0, int q1,
                                       SCoef c) {
    const int np = n + 2;
    ct_map<D>(n, r0, q0, q1, d, [&](int o, int, int, int) { return B[o] - ct_S<D>(u, o, np, c); });
}
// b_c = R d on the coarse rows [Q0, Q1) (coarse origin rc0); d has fine origin rf0 and holds the fine
// rows 2 Q0 .. 2 Q1 (the tree of tail_ph_restrict)
template <int D>
__device__ __noinline__ void ct_restrict(const double *d, int rf0, double *Bc, int rc0, int n, int nc, int Q0, int Q1) {
    const int np = n + 2;
    ct_map<D>(nc, rc0, Q0, Q1, Bc, [&](int, int I, int J, int K) {
        const int o = ct_off<D>(n, rf0, 2 * I + 1, 2 * J + 1, 2 * K + 1);
        const double rm = d[o - np - 1] + d[o - np + 1];
        const double rc = d[o - 1] + d[o + 1];
        const double rp = d[o + np - 1] + d[o + np + 1];
        const double f = rc + (d[o - np] + d[o + np]);
        const double e = rm + rp;
        if (D == 2) return ((4.0 * d[o] + 2.0 * f) + e) * 0.0625;
        const int pl = np * np, ol = o - pl, ou = o + pl;
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
// u += P e on the fine rows [q0, q1) (the tree of tail_ph_prolong); e has coarse origin rc0 and
// holds the coarse rows the fine rows need (including index -1 = the zero ring / ghost)
template <int D>
__device__ __noinline__ void ct_prolong(const double *e, int rc0, double *u, int rf0, int n, int nc, int q0, int q1) {
    const int npc = nc + 2;
    ct_map<D>(n, rf0, q0, q1, u, [&](int o, int i, int j, int k) {
        const bool ye = !(j & 1), ze = (D == 3) && !(k & 1), xe = !(i & 1);
        const int Ya = ye ? j / 2 - 1 : (j - 1) / 2, Yb = j / 2;
        const int Za = (D == 3) ? (ze ? k / 2 - 1 : (k - 1) / 2) : 0, Zb = (D == 3) ? k / 2 : 0;
        const int xa = (xe ? i / 2 - 1 : (i - 1) / 2) + 1, xb = i / 2 + 1;
        // row offsets of the coarse rows / planes in e (distributed index Y in 2D, Z in 3D)
        int rya, ryb, pza = 0, pzb = 0;
        if (D == 2) {
            rya = npc * (Ya - rc0 + 1); ryb = npc * (Yb - rc0 + 1);
        } else {
            rya = npc * (Ya + 1); ryb = npc * (Yb + 1);
            pza = npc * npc * (Za - rc0 + 1); pzb = npc * npc * (Zb - rc0 + 1);
        }
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

// Cluster barrier, then this CTA's ghost rows / planes of array A (level n, block B, origin r0)
// from its neighbours' edge rows; local barrier so the next phase sees them.
template <int D>
__device__ __forceinline__ void ct_exchange(cooperative_groups::cluster_group &cl, double *A, int n, int B, int r0) {
    cl.sync();
    const int rank = (int)cl.block_rank();
    const int rs = ct_rowsize<D>(n);
    if (rank > 0 && r0 - 1 >= 0) {             // ghost below <- rank - 1's last row (its local row B)
        const double *src = cl.map_shared_rank(A, rank - 1) + (size_t)B * rs;
        for (int q = threadIdx.x; q < rs; q += CT_THREADS) A[q] = src[q];
    }
    if (rank + 1 < CT_CS && r0 + B < n) {      // ghost above <- rank + 1's first row (its local row 1)
        const double *src = cl.map_shared_rank(A, rank + 1) + (size_t)rs;
        double *dst = A + (size_t)(B + 1) * rs;
        for (int q = threadIdx.x; q < rs; q += CT_THREADS) dst[q] = src[q];
    }
    __syncthreads();
}

template <int D>
__host__ __device__ inline int ct_level_doubles(int n, bool dist) {
    const int B = dist ? (n + 1) / CT_CS : n;
    return (B + 2) * ct_rowsize<D>(n);
}

// shared-memory plan: per level 3 arrays (iterate ping-pong 0/1, right-hand side 2), then the
// gather array of the last distributed level (full padded, CTA 0)
template <int D>
__host__ __device__ inline size_t ct_smem_doubles(const CTailParams &P, int *offs) {
    size_t tot = 0;
    for (int l = 0; l < P.nlev; ++l) {
        if (offs) offs[l] = (int)tot;
        tot += 3 * (size_t)ct_level_doubles<D>(P.n[l], l < P.ndist);
    }
    if (offs) offs[P.nlev] = (int)tot;
    tot += (size_t)ct_level_doubles<D>(P.n[P.ndist - 1], false);
    return tot;
}

template <int D>
__global__ void __launch_bounds__(CT_THREADS, 1) k_ctail(CTailParams P) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double csm[];
    const int rank = (int)cl.block_rank();
    const int L = P.nlev, LD = P.ndist;
    __shared__ int offs[CT_MAX_LEVELS + 1];
    if (threadIdx.x == 0) ct_smem_doubles<D>(P, offs);
    const size_t tot = ct_smem_doubles<D>(P, nullptr);
    for (size_t q = threadIdx.x; q < tot; q += CT_THREADS) csm[q] = 0.0;   // rings and ghosts stay zero
    __syncthreads();
    auto nB = [&](int l) { return l < LD ? (P.n[l] + 1) / CT_CS : P.n[l]; };
    auto r0 = [&](int l) { return l < LD ? rank * nB(l) : 0; };
    auto q1 = [&](int l) { return min(r0(l) + nB(l), P.n[l]); };             // owned rows [r0, q1)
    auto arr = [&](int l, int w) { return csm + offs[l] + (size_t)w * ct_level_doubles<D>(P.n[l], l < LD); };
    // ---- load b (own rows) and u (own rows + ghosts) of level 0
    {
        const int n = P.n[0], R0 = r0(0);
        double *Bb = arr(0, 2), *U = arr(0, 0);
        const int lo = P.u_in ? R0 - 1 : R0, hi = P.u_in ? q1(0) + 1 : q1(0);
        const int rows = (D == 3) ? n : 1;
        const int chunks = (n + 31) >> 5;
        for (int q = max(lo, 0); q < min(hi, n); ++q)
            for (int t = threadIdx.x >> 5; t < rows * chunks; t += CT_WARPS) {
                const int i = (t % chunks) * 32 + (threadIdx.x & 31), jr = t / chunks;
                if (i >= n) continue;
                const int j = (D == 3) ? jr : q, k = (D == 3) ? q : 0;
                const long long g = (long long)P.pitch * (j + (D == 3 ? (long long)n * k : 0)) + i;
                const int o = ct_off<D>(n, R0, i, j, k);
                if (q >= R0 && q < q1(0)) Bb[o] = P.b_in[g];
                if (P.u_in) U[o] = P.u_in[g];
            }
    }
    __syncthreads();
    unsigned cur = 0;   // bit l: the iterate of level l is in buffer 1
    auto sweeps = [&](int l, int count) {
        for (int s = 0; s < count; ++s) {
            const int w = (cur >> l) & 1;
            if (l < LD) {
                ct_sweep<D>(arr(l, w), arr(l, 1 - w), arr(l, 2), P.n[l], r0(l), r0(l), q1(l), P.c[l]);
                cur ^= 1u << l;
                ct_exchange<D>(cl, arr(l, 1 - w), P.n[l], nB(l), r0(l));
            } else {
                if (rank == 0) ct_sweep<D>(arr(l, w), arr(l, 1 - w), arr(l, 2), P.n[l], 0, 0, P.n[l], P.c[l]);
                cur ^= 1u << l;
                __syncthreads();
            }
        }
    };
    // ---------------- down
    for (int l = 0; l < L - 1; ++l) {
        sweeps(l, P.nu1);
        const int w = (cur >> l) & 1;
        const int n = P.n[l], nc = P.n[l + 1];
        if (l < LD) {
            // defect d = b - S u into buffer 1 - w (own rows), ghosts exchanged
            ct_defect<D>(arr(l, w), arr(l, 1 - w), arr(l, 2), n, r0(l), r0(l), q1(l), P.c[l]);
            ct_exchange<D>(cl, arr(l, 1 - w), n, nB(l), r0(l));
            if (l + 1 < LD) {
                ct_restrict<D>(arr(l, 1 - w), r0(l), arr(l + 1, 2), r0(l + 1), n, nc, r0(l + 1), q1(l + 1));
                __syncthreads();
            } else {
                // last distributed level: CTA 0 gathers the whole defect, then restricts locally
                if (rank == 0) {
                    double *G = csm + offs[L];
                    const int rs = ct_rowsize<D>(n), Bq = nB(l);
                    for (int q = 0; q < n; ++q) {
                        const int owner = q / Bq;
                        const double *src = cl.map_shared_rank(arr(l, 1 - w), owner) + (size_t)(q - owner * Bq + 1) * rs;
                        double *dst = G + (size_t)(q + 1) * rs;
                        for (int t = threadIdx.x; t < rs; t += CT_THREADS) dst[t] = src[t];
                    }
                    __syncthreads();
                    ct_restrict<D>(G, 0, arr(l + 1, 2), 0, n, nc, 0, nc);
                }
                __syncthreads();
            }
        } else {
            if (rank == 0) {
                ct_defect<D>(arr(l, w), arr(l, 1 - w), arr(l, 2), n, 0, 0, n, P.c[l]);
                __syncthreads();
                ct_restrict<D>(arr(l, 1 - w), 0, arr(l + 1, 2), 0, n, nc, 0, nc);
            }
            __syncthreads();
        }
    }
    // ---------------- coarsest (local, CTA 0): u = Ginv b, ascending-j accumulation
    {
        constexpr int Pc = D == 3 ? 27 : 9;
        const int l = L - 1;
        if (rank == 0 && threadIdx.x < Pc) {
            double *u = arr(l, 0);
            const double *Bq = arr(l, 2);
            const int t = threadIdx.x;
            auto po = [&](int q) { return (q % 3 + 1) + 5 * (((q / 3) % 3 + 1) + (D == 3 ? 5 * (q / 9 + 1) : 0)); };
            double acc = P.Ginv[t * Pc] * Bq[po(0)];
            for (int jj = 1; jj < Pc; ++jj) acc = acc + P.Ginv[t * Pc + jj] * Bq[po(jj)];
            u[po(t)] = acc;
        }
        cur &= ~(1u << l);
        __syncthreads();
    }
    // ---------------- up
    for (int l = L - 2; l >= 0; --l) {
        const int n = P.n[l], nc = P.n[l + 1];
        const double *E = arr(l + 1, (cur >> (l + 1)) & 1);
        double *U = arr(l, (cur >> l) & 1);
        if (l < LD) {
            if (l + 1 < LD) {
                ct_prolong<D>(E, r0(l + 1), U, r0(l), n, nc, r0(l), q1(l));
            } else {
                // the coarse result lives in CTA 0: every CTA copies it (full padded array) first
                cl.sync();
                double *C = csm + offs[L];
                const double *src = cl.map_shared_rank(E, 0);
                const int cnt = ct_level_doubles<D>(nc, false);
                for (int t = threadIdx.x; t < cnt; t += CT_THREADS) C[t] = src[t];
                __syncthreads();
                ct_prolong<D>(C, 0, U, r0(l), n, nc, r0(l), q1(l));
            }
            ct_exchange<D>(cl, U, n, nB(l), r0(l));
        } else {
            if (rank == 0) ct_prolong<D>(E, 0, U, 0, n, nc, 0, n);
            __syncthreads();
        }
        sweeps(l, P.nu2);
    }
    // ---------------- write the level-0 result (own rows)
    {
        const int n = P.n[0], R0 = r0(0);
        const double *U = arr(0, cur & 1);
        const int rows = (D == 3) ? n : 1;
        const int chunks = (n + 31) >> 5;
        for (int q = R0; q < q1(0); ++q)
            for (int t = threadIdx.x >> 5; t < rows * chunks; t += CT_WARPS) {
                const int i = (t % chunks) * 32 + (threadIdx.x & 31), jr = t / chunks;
                if (i >= n) continue;
                const int j = (D == 3) ? jr : q, k = (D == 3) ? q : 0;
                const long long g = (long long)P.pitch * (j + (D == 3 ? (long long)n * k : 0)) + i;
                P.u_out[g] = U[ct_off<D>(n, R0, i, j, k)];
            }
    }
    cl.sync();   // no CTA exits while another may still read its shared memory
}
