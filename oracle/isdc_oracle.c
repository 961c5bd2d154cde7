/*
 * isdc_oracle.c -- plain, slow, obviously-correct CPU oracle for the ISDC hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_1401_7824_b200/csrc); both follow the paper and the
 * canonical expression trees written out in DESIGN.md §4 ("canonical arithmetic").
 *
 * Paper: Speck, Ruprecht, Minion, Emmett, Krause, "Inexact spectral deferred corrections"
 * (arXiv:1401.7824), /root/reference/PAPER.md.  Citation key P:n = PAPER.md line n.
 *
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC ... -lquadmath
 * (no FMA contraction: every a*b+c below is a rounded multiply followed by a rounded add).
 *
 * Layout: dense fp64 arrays, n^d points, x fastest: idx = i + n*(j + n*k).
 * Boundary kinds (g_per, set per call by ora_set_bc / from ora_problem.bc):
 *   Dirichlet (default): n = 2^p - 1 interior points of [0,1]^d, h = 1/(n+1); every value outside
 *     0..n-1 reads as 0 (homogeneous data).
 *   Periodic (NEXT f3, Burgers P:106-112): n = 2^p points x_i = -1 + i h of [-1,1)^d, h = 2/n;
 *     indices wrap modulo n ("periodic boundary conditions"; reading R31).
 *
 * Pins (tests/test_oracle_*.py): every function below is pinned by a closed form, an invariant,
 * a special case or brute force, except where a header comment says "parity unpinned".
 */
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __float128 qf;

int ora_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
/* Thread count of the OpenMP loops (timing only: every loop is over independent grid points or an
 * exact max, so the results do not depend on it). */
void ora_set_num_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* ------------------------------------------------------------------------------------------ */
/* Quadrature tables (Eq. 2).  Gauss-Lobatto nodes on [0,1]; Q_{m,j} = int_0^{tau_m}  */
/* l_j(s) ds, S_{m,j} = int_{tau_m}^{tau_{m+1}} l_j(s) ds (node-to-node weights s_{m,j}).      */
/* Everything in binary128, rounded once to binary64 at the end.                               */
/* ------------------------------------------------------------------------------------------ */

/* Legendre P_n(x) and P_n'(x) by the three-term recurrence (k+1)P_{k+1} = (2k+1)xP_k - kP_{k-1}. */
static void legendre_pd(int n, qf x, qf *p, qf *dp) {
    qf p0 = 1, p1 = x;
    if (n == 0) { *p = 1; *dp = 0; return; }
    for (int k = 1; k < n; ++k) {
        qf p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
        p0 = p1; p1 = p2;
    }
    *p = p1;
    /* (1 - x^2) P_n' = n (P_{n-1} - x P_n), valid for |x| < 1 (interior Lobatto nodes). */
    *dp = n * (p0 - x * p1) / (1 - x * x);
}

/* Gauss-Lobatto nodes on [-1,1]: +-1 and the roots of P'_{M-1}; Newton on P'_{M-1} with
 * P'' from the Legendre ODE (1-x^2)P'' - 2xP' + n(n+1)P = 0. */
static int lobatto_q(int M, qf *x) {
    if (M < 2 || M > 16) return -1;
    int n = M - 1;
    x[0] = -1; x[M - 1] = 1;
    for (int k = 1; k < M - 1; ++k) {
        qf xi = -cosq(M_PIq * k / n);
        for (int it = 0; it < 100; ++it) {
            qf p, dp;
            legendre_pd(n, xi, &p, &dp);
            qf d2p = (2 * xi * dp - n * (n + 1) * p) / (1 - xi * xi);
            qf dx = dp / d2p;
            xi -= dx;
            if (fabsq(dx) < 1e-33Q) break;
        }
        x[k] = xi;
    }
    return 0;
}

/* Q_{m,j} = int_0^{tau_m} l_j, by exact integration of the monomial expansion of l_j. */
static void q_matrix_q(int M, const qf *tau, qf *Q) {
    for (int j = 0; j < M; ++j) {
        qf c[32];
        memset(c, 0, sizeof c);
        c[0] = 1;
        int deg = 0;
        for (int k = 0; k < M; ++k) {
            if (k == j) continue;
            qf den = tau[j] - tau[k];
            /* c(s) <- c(s) * (s - tau_k) / den */
            for (int p = deg + 1; p >= 1; --p) c[p] = (c[p - 1] - tau[k] * c[p]) / den;
            c[0] = (-tau[k] * c[0]) / den;
            ++deg;
        }
        for (int m = 0; m < M; ++m) {
            qf acc = 0, tp = tau[m];
            for (int p = 0; p <= deg; ++p) { acc += c[p] * tp / (p + 1); tp *= tau[m]; }
            Q[m * M + j] = acc;
        }
    }
}

/* tau[M], Q[M*M], S[(M-1)*M], dtau[M-1] (all binary64, each rounded once from binary128). */
int ora_tables(int M, double *tau, double *Q, double *S, double *dtau) {
    qf x[32], t[32], Qq[32 * 32];
    if (lobatto_q(M, x)) return -1;
    for (int m = 0; m < M; ++m) t[m] = (x[m] + 1) / 2;
    t[0] = 0; t[M - 1] = 1;
    q_matrix_q(M, t, Qq);
    for (int m = 0; m < M; ++m) tau[m] = (double)t[m];
    for (int i = 0; i < M * M; ++i) Q[i] = (double)Qq[i];
    for (int m = 0; m + 1 < M; ++m) {
        dtau[m] = (double)(t[m + 1] - t[m]);
        for (int j = 0; j < M; ++j) S[m * M + j] = (double)(Qq[(m + 1) * M + j] - Qq[m * M + j]);
    }
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Grid access                                                                                 */
/* ------------------------------------------------------------------------------------------ */
static int g_per = 0;    /* 1: periodic grid (see the header); read-only inside parallel regions */
void ora_set_bc(int periodic) { g_per = periodic ? 1 : 0; }
int ora_get_bc(void) { return g_per; }

/* one wrap suffices: stencil offsets are at most 3 and n >= 4 */
static inline int wrap(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }
/* 1/h: Dirichlet N = n+1; periodic n/2 (both exact powers of two) */
static inline double inv_h(int n) { return g_per ? (double)n * 0.5 : (double)(n + 1); }
/* next coarser level and the coarsest one (exact dense solve) */
static inline int coarser(int n) { return g_per ? n / 2 : (n - 1) / 2; }
static inline int coarsest(void) { return g_per ? 4 : 3; }

static inline double at(const double *u, int d, int n, int i, int j, int k) {
    if (g_per) {
        i = wrap(i, n); j = wrap(j, n);
        if (d == 3) k = wrap(k, n);
    }
    if (i < 0 || j < 0 || i >= n || j >= n) return 0.0;
    if (d == 3) {
        if (k < 0 || k >= n) return 0.0;
        return u[(size_t)i + (size_t)n * ((size_t)j + (size_t)n * (size_t)k)];
    }
    return u[(size_t)i + (size_t)n * (size_t)j];
}
static inline size_t npts(int d, int n) { return d == 3 ? (size_t)n * n * n : (size_t)n * n; }

/* In-plane partial sums of the canonical trees:
 *   r(i,j,k) = q(i-1,j,k) + q(i+1,j,k)
 *   f(i,j,k) = r(i,j,k) + (q(i,j-1,k) + q(i,j+1,k))      in-plane face sum (4 terms)
 *   e(i,j,k) = r(i,j-1,k) + r(i,j+1,k)                    in-plane diagonal sum (4 terms)
 * 3D adds   F = f(k) + (q(k-1) + q(k+1))                  6 faces
 *           E = e(k) + (f(k-1) + f(k+1))                  12 edges
 * A row/plane outside the domain contributes exact zeros. */
static inline double r_(const double *q, int d, int n, int i, int j, int k) {
    return at(q, d, n, i - 1, j, k) + at(q, d, n, i + 1, j, k);
}
static inline double f_(const double *q, int d, int n, int i, int j, int k) {
    return r_(q, d, n, i, j, k) + (at(q, d, n, i, j - 1, k) + at(q, d, n, i, j + 1, k));
}
static inline double e_(const double *q, int d, int n, int i, int j, int k) {
    return r_(q, d, n, i, j - 1, k) + r_(q, d, n, i, j + 1, k);
}
/* faces (2D: 4, 3D: 6) and edges/corners-of-the-9-point (2D: 4 diagonals, 3D: 12 edges) */
static inline double faces(const double *q, int d, int n, int i, int j, int k) {
    if (d == 2) return f_(q, d, n, i, j, 0);
    return f_(q, d, n, i, j, k) + (at(q, d, n, i, j, k - 1) + at(q, d, n, i, j, k + 1));
}
static inline double edges(const double *q, int d, int n, int i, int j, int k) {
    if (d == 2) return e_(q, d, n, i, j, 0);
    return e_(q, d, n, i, j, k) + (f_(q, d, n, i, j, k - 1) + f_(q, d, n, i, j, k + 1));
}

/* ------------------------------------------------------------------------------------------ */
/* Compact (Mehrstellen) pair, P:68-72 and SPEC S:144 (2D); 3D: standard 19-point pair.        */
/*   2D: L_h = 1/(6h^2)[1 4 1; 4 -20 4; 1 4 1],  B_h = 1/12[0 1 0; 1 8 1; 0 1 0]               */
/*   3D: L_h = 1/(6h^2)(centre -24, faces 2, edges 1),  B_h = 1/12(centre 6, faces 1)          */
/* Constants (host, binary64, in this order): N = 1/h (inv_h), N2 = N*N;                     */
/*   2D kB0 = 8/12, kB1 = 1/12, kL0 = (-20*N2)/6, kL1 = (4*N2)/6, kL2 = N2/6                   */
/*   3D kB0 = 6/12, kB1 = 1/12, kL0 = (-24*N2)/6, kL1 = (2*N2)/6, kL2 = N2/6                   */
/*   B q = kB0*q + kB1*faces;   L q = (kL0*q + kL1*faces) + kL2*edges                          */
/* ------------------------------------------------------------------------------------------ */
typedef struct { double kB0, kB1, kL0, kL1, kL2; } bl_consts;

static bl_consts make_bl(int d, int n) {
    bl_consts c;
    double N = inv_h(n), N2 = N * N;
    if (d == 2) {
        c.kB0 = 8.0 / 12.0; c.kB1 = 1.0 / 12.0;
        c.kL0 = (-20.0 * N2) / 6.0; c.kL1 = (4.0 * N2) / 6.0; c.kL2 = N2 / 6.0;
    } else {
        c.kB0 = 6.0 / 12.0; c.kB1 = 1.0 / 12.0;
        c.kL0 = (-24.0 * N2) / 6.0; c.kL1 = (2.0 * N2) / 6.0; c.kL2 = N2 / 6.0;
    }
    return c;
}
static inline double B_at(const bl_consts *c, const double *q, int d, int n, int i, int j, int k) {
    return c->kB0 * at(q, d, n, i, j, k) + c->kB1 * faces(q, d, n, i, j, k);
}
static inline double L_at(const bl_consts *c, const double *q, int d, int n, int i, int j, int k) {
    return (c->kL0 * at(q, d, n, i, j, k) + c->kL1 * faces(q, d, n, i, j, k)) +
           c->kL2 * edges(q, d, n, i, j, k);
}

#define FOR_POINTS(d, n)                                                        \
    _Pragma("omp parallel for collapse(2) schedule(static)")                    \
    for (int kk = 0; kk < ((d) == 3 ? (n) : 1); ++kk)                          \
        for (int jj = 0; jj < (n); ++jj)                                        \
            for (int ii = 0; ii < (n); ++ii)
#define IDX(d, n) ((size_t)ii + (size_t)(n) * ((size_t)jj + (size_t)(n) * (size_t)kk))

void ora_apply_B(int d, int n, const double *q, double *out) {
    bl_consts c = make_bl(d, n);
    FOR_POINTS(d, n) out[IDX(d, n)] = B_at(&c, q, d, n, ii, jj, kk);
}
void ora_apply_L(int d, int n, const double *q, double *out) {
    bl_consts c = make_bl(d, n);
    FOR_POINTS(d, n) out[IDX(d, n)] = L_at(&c, q, d, n, ii, jj, kk);
}

/* ------------------------------------------------------------------------------------------ */
/* Node-system operator S_l = B_h - gamma L_h on level l ("W - dt_m A", A = nu L_h),      */
/* rediscretised with h_l = 1/N_l (N_l = inv_h).  g = gamma*(N_l*N_l) (N_l^2 a power of two).  */
/*   2D: c0 = (8 + 40g)/12, c1 = (1 - 8g)/12, c2 = (-2g)/12                                    */
/*   3D: c0 = (6 + 48g)/12, c1 = (1 - 4g)/12, c2 = (-2g)/12                                    */
/*   S u = (c0*u + c1*faces) + c2*edges ;  weighted Jacobi: u + wd*(b - S u), wd = omega/c0    */
/* ------------------------------------------------------------------------------------------ */
typedef struct { double c0, c1, c2, wd; } s_coef;

static s_coef make_s(int d, int n, double gamma, double omega) {
    s_coef s;
    double N = inv_h(n);
    double g = gamma * (N * N);
    if (d == 2) {
        s.c0 = (8.0 + 40.0 * g) / 12.0; s.c1 = (1.0 - 8.0 * g) / 12.0; s.c2 = (-2.0 * g) / 12.0;
    } else {
        s.c0 = (6.0 + 48.0 * g) / 12.0; s.c1 = (1.0 - 4.0 * g) / 12.0; s.c2 = (-2.0 * g) / 12.0;
    }
    s.wd = omega / s.c0;
    return s;
}
static inline double S_at(const s_coef *s, const double *u, int d, int n, int i, int j, int k) {
    return (s->c0 * at(u, d, n, i, j, k) + s->c1 * faces(u, d, n, i, j, k)) +
           s->c2 * edges(u, d, n, i, j, k);
}

void ora_level_coefs(int d, int n, double gamma, double omega, double *c4) {
    s_coef s = make_s(d, n, gamma, omega);
    c4[0] = s.c0; c4[1] = s.c1; c4[2] = s.c2; c4[3] = s.wd;
}

void ora_apply_S(int d, int n, double gamma, const double *u, double *out) {
    s_coef s = make_s(d, n, gamma, 0.8);
    FOR_POINTS(d, n) out[IDX(d, n)] = S_at(&s, u, d, n, ii, jj, kk);
}

/* one weighted-Jacobi sweep, out of place */
static void jacobi(const s_coef *s, int d, int n, const double *b, const double *u, double *out) {
    FOR_POINTS(d, n) {
        size_t p = IDX(d, n);
        out[p] = u[p] + s->wd * (b[p] - S_at(s, u, d, n, ii, jj, kk));
    }
}
void ora_jacobi(int d, int n, double gamma, double omega, int sweeps, const double *b, double *u) {
    s_coef s = make_s(d, n, gamma, omega);
    size_t P = npts(d, n);
    double *t = malloc(P * sizeof(double));
    for (int it = 0; it < sweeps; ++it) {
        jacobi(&s, d, n, b, u, t);
        memcpy(u, t, P * sizeof(double));
    }
    free(t);
}

static void defect(const s_coef *s, int d, int n, const double *b, const double *u, double *r) {
    FOR_POINTS(d, n) {
        size_t p = IDX(d, n);
        r[p] = b[p] - S_at(s, u, d, n, ii, jj, kk);
    }
}
static double maxabs(const double *a, size_t P) {
    double m = 0.0;
#pragma omp parallel for reduction(max : m)
    for (size_t p = 0; p < P; ++p) {
        double v = fabs(a[p]);
        if (isnan(v)) v = INFINITY;  /* non-finite values surface as Inf */
        if (v > m) m = v;
    }
    return m;
}
double ora_defect_norm(int d, int n, double gamma, const double *b, const double *u) {
    s_coef s = make_s(d, n, gamma, 0.8);
    size_t P = npts(d, n);
    double *r = malloc(P * sizeof(double));
    defect(&s, d, n, b, u, r);
    double m = maxabs(r, P);
    free(r);
    return m;
}

/* Full-weighting restriction: coarse (I,J[,K]) <-> fine 2I+1
 * (Dirichlet) or fine 2I (periodic, the coarse grid keeps the even points of x_i = -1 + i h).
 *   2D: bc = ((4*d + 2*faces) + edges) * 0.0625
 *   3D: bc = ((8*d + 4*faces) + (2*edges + corners)) * 0.015625,
 *       corners = e(k-1) + e(k+1)  (8 corners of the 27-point cube)                           */
void ora_restrict(int d, int nf, const double *df, double *bc) {
    int nc = coarser(nf), o = g_per ? 0 : 1;
    FOR_POINTS(d, nc) {
        int x = 2 * ii + o, y = 2 * jj + o, z = (d == 3) ? 2 * kk + o : 0;
        double c = at(df, d, nf, x, y, z);
        double fa = faces(df, d, nf, x, y, z), ed = edges(df, d, nf, x, y, z);
        double v;
        if (d == 2) {
            v = ((4.0 * c + 2.0 * fa) + ed) * 0.0625;
        } else {
            double co = e_(df, d, nf, x, y, z - 1) + e_(df, d, nf, x, y, z + 1);
            v = ((8.0 * c + 4.0 * fa) + (2.0 * ed + co)) * 0.015625;
        }
        bc[IDX(d, nc)] = v;
    }
}

/* Bi/trilinear prolongation + correction: u += P e.  Per axis (Dirichlet): odd fine index x ->
 * coarse (x-1)/2 (weight 1); even x -> coarse pair (x/2-1, x/2) summed (a + b), weight 1/2.
 * Periodic: even x -> coarse x/2; odd x -> pair ((x-1)/2, (x+1)/2 mod nc), weight 1/2.  Pairs are
 * summed x innermost, then y, then z; the sum is scaled once by 0.5^(#paired axes).          */
static void prolong_axis(int x, int *xs, int *nx, double *w) {
    if (g_per) {
        if (x & 1) { xs[0] = (x - 1) / 2; xs[1] = (x + 1) / 2; *nx = 2; *w *= 0.5; }
        else { xs[0] = x / 2; *nx = 1; }
    } else {
        if (x & 1) { xs[0] = (x - 1) / 2; *nx = 1; }
        else { xs[0] = x / 2 - 1; xs[1] = x / 2; *nx = 2; *w *= 0.5; }
    }
}
void ora_prolong_add(int d, int nc, const double *ec, double *uf) {
    int nf = g_per ? 2 * nc : 2 * nc + 1;
    FOR_POINTS(d, nf) {
        int xs[2], ys[2], zs[2], nx, ny, nz;
        double w = 1.0;
        prolong_axis(ii, xs, &nx, &w);
        prolong_axis(jj, ys, &ny, &w);
        if (d == 2) { zs[0] = 0; nz = 1; }
        else prolong_axis(kk, zs, &nz, &w);
        double sz = 0.0;
        for (int c = 0; c < nz; ++c) {
            double sy = 0.0;
            for (int b = 0; b < ny; ++b) {
                double sx = at(ec, d, nc, xs[0], ys[b], zs[c]);
                if (nx == 2) sx = sx + at(ec, d, nc, xs[1], ys[b], zs[c]);
                sy = (b == 0) ? sx : sy + sx;
            }
            sz = (c == 0) ? sy : sz + sy;
        }
        size_t p = IDX(d, nf);
        uf[p] = uf[p] + sz * w;
    }
}

/* Coarsest level (Dirichlet n = 3; periodic n = 4): exact solve with the inverse of the P x P
 * matrix of S (P = n^d), built from the binary64 coefficients (c0,c1,c2) and inverted by
 * Gauss-Jordan elimination with partial pivoting in binary128, rounded once (DESIGN.md reading
 * R12; periodic: neighbour distances taken modulo n).  e_i = sum_j Ginv_ij b_j, accumulated left
 * to right over ascending j starting from Ginv_i0*b_0. */
#define ORA_PMAX 64
int ora_coarse_inverse(int d, double gamma, double omega, double *Ginv) {
    int n = coarsest(), P = (d == 3) ? n * n * n : n * n;
    s_coef s = make_s(d, n, gamma, omega);
    qf (*A)[2 * ORA_PMAX] = malloc(sizeof(qf) * ORA_PMAX * 2 * ORA_PMAX);
    for (int r = 0; r < P; ++r) for (int c = 0; c < 2 * P; ++c) A[r][c] = 0;
    for (int r = 0; r < P; ++r) {
        int ri = r % n, rj = (r / n) % n, rk = r / (n * n);
        for (int c = 0; c < P; ++c) {
            int ci = c % n, cj = (c / n) % n, ck = c / (n * n);
            int di = abs(ri - ci), dj = abs(rj - cj), dk = abs(rk - ck);
            if (g_per) { if (n - di < di) di = n - di; if (n - dj < dj) dj = n - dj; if (n - dk < dk) dk = n - dk; }
            if (di > 1 || dj > 1 || dk > 1) continue;
            int nd = di + dj + dk;
            double v = (nd == 0) ? s.c0 : (nd == 1) ? s.c1 : (nd == 2) ? s.c2 : 0.0;
            A[r][c] = (qf)v;
        }
        A[r][P + r] = 1;
    }
    for (int c = 0; c < P; ++c) {
        int piv = c;
        for (int r = c + 1; r < P; ++r) if (fabsq(A[r][c]) > fabsq(A[piv][c])) piv = r;
        if (A[piv][c] == 0) { free(A); return -1; }
        if (piv != c) for (int k = 0; k < 2 * P; ++k) { qf t = A[c][k]; A[c][k] = A[piv][k]; A[piv][k] = t; }
        qf inv = 1 / A[c][c];
        for (int k = 0; k < 2 * P; ++k) A[c][k] *= inv;
        for (int r = 0; r < P; ++r) {
            if (r == c || A[r][c] == 0) continue;
            qf f = A[r][c];
            for (int k = 0; k < 2 * P; ++k) A[r][k] -= f * A[c][k];
        }
    }
    for (int r = 0; r < P; ++r) for (int c = 0; c < P; ++c) Ginv[r * P + c] = (double)A[r][P + c];
    free(A);
    return 0;
}
static void coarse_apply(int P, const double *Ginv, const double *b, double *e) {
    for (int i = 0; i < P; ++i) {
        double acc = Ginv[i * P] * b[0];
        for (int j = 1; j < P; ++j) acc = acc + Ginv[i * P + j] * b[j];
        e[i] = acc;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Geometric multigrid V(nu1,nu2) cycle on S_l ("V-cycles"; components per B:configs[1] */
/* and DESIGN.md R11-R14): nu1 weighted-Jacobi sweeps; d = b - S u; b_c = R d; e_c = V(0,b_c)  */
/* on level l+1 (correction scheme, zero initial guess, same gamma); u += P e_c; nu2 sweeps.   */
/* On the coarsest level (n = 3, periodic 4) the cycle is the exact solve.                   */
/* ------------------------------------------------------------------------------------------ */
static void vcycle_rec(int d, int n, double gamma, int nu1, int nu2, double omega,
                       const double *b, double *u) {
    size_t P = npts(d, n);
    if (n == coarsest()) {
        /* one-entry cache of the coarse inverse (the oracle is single-threaded at this level) */
        static double Ginv[ORA_PMAX * ORA_PMAX], cg = -1.0, co = -1.0;
        static int cd = 0, cp = -1;
        if (cd != d || cg != gamma || co != omega || cp != g_per) {
            ora_coarse_inverse(d, gamma, omega, Ginv);
            cd = d; cg = gamma; co = omega; cp = g_per;
        }
        coarse_apply((int)P, Ginv, b, u);
        return;
    }
    s_coef s = make_s(d, n, gamma, omega);
    double *t = malloc(P * sizeof(double));
    for (int it = 0; it < nu1; ++it) { jacobi(&s, d, n, b, u, t); memcpy(u, t, P * sizeof(double)); }
    defect(&s, d, n, b, u, t);
    int nc = coarser(n);
    size_t Pc = npts(d, nc);
    double *bc = malloc(Pc * sizeof(double)), *ec = calloc(Pc, sizeof(double));
    ora_restrict(d, n, t, bc);
    vcycle_rec(d, nc, gamma, nu1, nu2, omega, bc, ec);
    ora_prolong_add(d, nc, ec, u);
    for (int it = 0; it < nu2; ++it) { jacobi(&s, d, n, b, u, t); memcpy(u, t, P * sizeof(double)); }
    free(t); free(bc); free(ec);
}
void ora_vcycle(int d, int n, double gamma, int nu1, int nu2, double omega, const double *b, double *u) {
    vcycle_rec(d, n, gamma, nu1, nu2, omega, b, u);
}

/* ------------------------------------------------------------------------------------------ */
/* Explicit part f^E (Eq. 4; kinds from B:configs; R20-R22)                 */
/*   NONE: not evaluated (all f^E terms are dropped);  CUBIC: u - (u*u)*u;                     */
/*   FORCING: G*ct (ct = cos(t_j), host scalar);                                               */
/*   ADVECTION (CD4, zero ghosts): dx = (8*(u(x+1)-u(x-1)) - (u(x+2)-u(x-2)))*kx, kx=(a_x*N)/12,*/
/*   f = -((dx + dy) + dz)   (2D: -(dx + dy))                                                   */
/*   BURGERS (periodic; "5th order WENO"; reading R31): f = -(u u_x + u u_y)    */
/*     in conservation form -sum_a d_a(u^2/2), WENO5-JS reconstruction of Lax-Friedrichs split  */
/*     fluxes (below).                                                                         */
/* ------------------------------------------------------------------------------------------ */
enum { FE_NONE = 0, FE_CUBIC = 1, FE_FORCING = 2, FE_ADVECTION = 3, FE_BURGERS = 4 };

/* WENO5 reconstruction (Jiang & Shu 1996; restated, reading R31) of the value at the face between
 * v2 and v3 from the five cell values v0..v4 (upwind side v0..v2):
 *   candidate stencils  p0 = (2v0 - 7v1 + 11v2)/6,  p1 = (-v1 + 5v2 + 2v3)/6,  p2 = (2v2 + 5v3 - v4)/6
 *   smoothness          b_k = 13/12 s_k^2 + 1/4 t_k^2   with
 *                       s0 = v0 - 2v1 + v2, t0 = v0 - 4v1 + 3v2;  s1 = v1 - 2v2 + v3, t1 = v1 - v3;
 *                       s2 = v2 - 2v3 + v4, t2 = 3v2 - 4v3 + v4
 *   weights             a_k = d_k / (eps + b_k)^2,  d = (0.1, 0.6, 0.3),  eps = 1e-6
 *   value               (a0 p0 + a1 p1 + a2 p2) / (a0 + a1 + a2)
 * Canonical trees: exactly as written below (left to right, divisions by 6 and by the weight sum
 * are IEEE divisions, 13/12 is the binary64 constant 13.0/12.0). */
static double weno5(double v0, double v1, double v2, double v3, double v4) {
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
double ora_weno5(double v0, double v1, double v2, double v3, double v4) { return weno5(v0, v1, v2, v3, v4); }

/* Lax-Friedrichs split fluxes of f(u) = u^2/2 with the global speed alpha = max|u| of the field
 * being evaluated: f+- = (q +- alpha u) * 0.5, q = (u*u)*0.5. */
static inline double split_flux(double x, double alpha, int plus) {
    double q = (x * x) * 0.5, a = alpha * x;
    return plus ? (q + a) * 0.5 : (q - a) * 0.5;
}
/* numerical flux through the face between point s and s+1 of axis ax (0 x, 1 y, 2 z):
 *   F = weno5(f+(s-2), f+(s-1), f+(s), f+(s+1), f+(s+2)) + weno5(f-(s+3), f-(s+2), f-(s+1), f-(s), f-(s-1)) */
static double burgers_face(const double *u, int d, int n, int i, int j, int k, int ax, double alpha) {
    int di = (ax == 0), dj = (ax == 1), dk = (ax == 2);
    double fp[5], fm[5];
    for (int s = 0; s < 5; ++s) {
        int o = s - 2;       /* f+ at s-2 .. s+2 */
        fp[s] = split_flux(at(u, d, n, i + o * di, j + o * dj, k + o * dk), alpha, 1);
        int q = 3 - s;       /* f- at s+3 .. s-1 */
        fm[s] = split_flux(at(u, d, n, i + q * di, j + q * dj, k + q * dk), alpha, 0);
    }
    return weno5(fp[0], fp[1], fp[2], fp[3], fp[4]) + weno5(fm[0], fm[1], fm[2], fm[3], fm[4]);
}

static void fe_eval(int fe, int d, int n, const double *a, const double *G, double ct,
                    const double *u, double *out) {
    double N = inv_h(n);
    double kx = (a[0] * N) / 12.0, ky = (a[1] * N) / 12.0, kz = (a[2] * N) / 12.0;
    double alpha = (fe == FE_BURGERS) ? maxabs(u, npts(d, n)) : 0.0;
    FOR_POINTS(d, n) {
        size_t p = IDX(d, n);
        double v = 0.0;
        if (fe == FE_CUBIC) {
            double x = u[p];
            v = x - (x * x) * x;
        } else if (fe == FE_FORCING) {
            v = G[p] * ct;
        } else if (fe == FE_ADVECTION) {
            int i = ii, j = jj, k = kk;
            double dx = (8.0 * (at(u, d, n, i + 1, j, k) - at(u, d, n, i - 1, j, k)) -
                         (at(u, d, n, i + 2, j, k) - at(u, d, n, i - 2, j, k))) * kx;
            double dy = (8.0 * (at(u, d, n, i, j + 1, k) - at(u, d, n, i, j - 1, k)) -
                         (at(u, d, n, i, j + 2, k) - at(u, d, n, i, j - 2, k))) * ky;
            if (d == 3) {
                double dz = (8.0 * (at(u, d, n, i, j, k + 1) - at(u, d, n, i, j, k - 1)) -
                             (at(u, d, n, i, j, k + 2) - at(u, d, n, i, j, k - 2))) * kz;
                v = -((dx + dy) + dz);
            } else {
                v = -(dx + dy);
            }
        } else if (fe == FE_BURGERS) {
            /* f = -(((Fx(i) - Fx(i-1)) + (Fy(j) - Fy(j-1))) [+ (Fz(k) - Fz(k-1))]) * (1/h)) */
            int i = ii, j = jj, k = kk;
            double gx = burgers_face(u, d, n, i, j, k, 0, alpha) - burgers_face(u, d, n, i - 1, j, k, 0, alpha);
            double gy = burgers_face(u, d, n, i, j, k, 1, alpha) - burgers_face(u, d, n, i, j - 1, k, 1, alpha);
            double sum = gx + gy;
            if (d == 3)
                sum = sum + (burgers_face(u, d, n, i, j, k, 2, alpha) - burgers_face(u, d, n, i, j, k - 1, 2, alpha));
            v = -(sum * N);
        }
        out[p] = v;
    }
}
void ora_fe_eval(int fe, int d, int n, const double *a, const double *G, double ct,
                 const double *u, double *out) {
    fe_eval(fe, d, n, a, G, ct, u, out);
}

/* ------------------------------------------------------------------------------------------ */
/* Problem / state                                                                             */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int dim, n, M;
    double dt, nu;
    int fe;
    double fe_a[3];
    const double *G;     /* forcing profile (FE_FORCING), n^d, else NULL */
    int mode;            /* 0 = ISDC (exactly L cycles), 1 = SDC (cycles to inner tolerance),
                            2 = ISDC capped: cycles to inner tolerance, at most L (reading R10) */
    int L;
    double inner_tol;    /* SDC: stop when ||b - S u|| <= inner_tol * max(1, ||b||) */
    int inner_cap;
    double sweep_tol;    /* stop when ||r~|| < sweep_tol (strict, "below") */
    int max_sweeps;
    int fixed_sweeps;    /* >0: exactly this many sweeps, no tolerance test (config 1) */
    int nu1, nu2;
    double omega;
    int guess;           /* 0 = u_{m+1}^k; 1 = zero; 2 = u_m^{k+1} (P:187-189 ablation) */
    int res_kind;        /* 0 = weighted ||r~|| (reading R15); 1 = unweighted ||W^-1 r~|| (2D, NEXT f2) */
    double w_tol;        /* res_kind 1: W-solve until ||r~ - W x|| <= w_tol * ||r~|| (reading R15b) */
    int w_cap;           /* res_kind 1: at most w_cap W-cycles per node */
    int bc;              /* 0 = homogeneous Dirichlet on [0,1]^d; 1 = periodic on [-1,1)^d (NEXT f3) */
} ora_problem;

static long g_wcycles;   /* W-cycles of the last ora_step (not V-cycles: P:165) */

/* Right-hand side of Eq. (5) for substep m (0-based: node m -> m+1), regrouped by linearity of
 * B_h and L_h (SURVEY §8(c1) "check by expansion"):
 *   v = (unew_m + dtm*(fE(unew_m) - fE(uold_m))) + sum_j a_j*fE(uold_j),  a_j = dt*S_{m,j}
 *   w = sum_j beta_j*uold_j - gm*uold_{m+1},  beta_j = (nu*dt)*S_{m,j},  gm = nu*dtm, dtm = dt*dtau_m
 *   b = B v + L w
 * Sums over j are left folds in ascending j starting from the j = 0 term.
 * The f^E(unew_m)-f^E(uold_m) and sum a_j fE terms are absent when fE = NONE.                  */
static void rhs_m(const ora_problem *P, const double *tau, const double *S, const double *dtau,
                  double t_n, int m, double *const *uold, double *const *unew, double *b,
                  double *v, double *w, double *ftmp, double *ftmp2, double *const *fas) {
    int d = P->dim, n = P->n, M = P->M;
    size_t NP = npts(d, n);
    double dtm = P->dt * dtau[m];
    double gm = P->nu * dtm;
    double nudt = P->nu * P->dt;
    bl_consts c = make_bl(d, n);
    /* w */
    for (size_t p = 0; p < NP; ++p) {
        double acc = (nudt * S[m * M + 0]) * uold[0][p];
        for (int j = 1; j < M; ++j) acc = acc + (nudt * S[m * M + j]) * uold[j][p];
        w[p] = acc - gm * uold[m + 1][p];
    }
    /* v */
    if (P->fe == FE_NONE) {
        memcpy(v, unew[m], NP * sizeof(double));
    } else {
        /* sum_j a_j fE(uold_j) */
        double *acc = ftmp2;
        for (int j = 0; j < M; ++j) {
            double ct = cos(t_n + P->dt * tau[j]);
            fe_eval(P->fe, d, n, P->fe_a, P->G, ct, uold[j], ftmp);
            double aj = P->dt * S[m * M + j];
            for (size_t p = 0; p < NP; ++p) acc[p] = (j == 0) ? aj * ftmp[p] : acc[p] + aj * ftmp[p];
        }
        double ctm = cos(t_n + P->dt * tau[m]);
        fe_eval(P->fe, d, n, P->fe_a, P->G, ctm, unew[m], v);      /* v <- fE(unew_m) */
        fe_eval(P->fe, d, n, P->fe_a, P->G, ctm, uold[m], ftmp);   /* ftmp <- fE(uold_m) */
        for (size_t p = 0; p < NP; ++p) v[p] = (unew[m][p] + dtm * (v[p] - ftmp[p])) + acc[p];
    }
    FOR_POINTS(d, n) {
        size_t p = IDX(d, n);
        b[p] = B_at(&c, v, d, n, ii, jj, kk) + L_at(&c, w, d, n, ii, jj, kk);
    }
    /* MLSDC coarse level (NEXT f4, R32): the node-to-node difference of the FAS
     * correction, b <- b + (fas_{m+1} - fas_m), fas_0 = 0 (node 1 = u_0 carries no correction) */
    if (fas)
        for (size_t p = 0; p < NP; ++p) b[p] = b[p] + (fas[m + 1][p] - (m == 0 ? 0.0 : fas[m][p]));
}

/* Weighted SDC residual (R15-R16): for nodes m = 1..M-1 (0-based),
 *   p_m = (u_m - u_0) - sum_j qa_j fE(u_j),  qa_j = dt*Q_{m,j}   (fE = NONE: p_m = u_m - u_0)
 *   z_m = sum_j qb_j u_j,                    qb_j = (nu*dt)*Q_{m,j}
 *   r~_m = B p_m - L z_m ;  reported: max_m ||r~_m||_inf (and per node)                        */
static double residual_fields(const ora_problem *P, const double *tau, const double *Q, double t_n,
                              double *const *u, double *per_node, double *const *rout);
double ora_residual_state(const ora_problem *P, const double *tau, const double *Q, double t_n,
                          double *const *u, double *per_node) {
    return residual_fields(P, tau, Q, t_n, u, per_node, NULL);
}
/* rout (nullable): rout[m] (m = 1..M-1) receives the field r~_m (MLSDC, NEXT f4) */
static double residual_fields(const ora_problem *P, const double *tau, const double *Q, double t_n,
                              double *const *u, double *per_node, double *const *rout) {
    int d = P->dim, n = P->n, M = P->M;
    size_t NP = npts(d, n);
    bl_consts c = make_bl(d, n);
    double nudt = P->nu * P->dt;
    double *pm = malloc(NP * sizeof(double)), *zm = malloc(NP * sizeof(double));
    double *ft = malloc(NP * sizeof(double)), *r = malloc(NP * sizeof(double));
    double *facc = (P->fe == FE_NONE) ? NULL : malloc(NP * sizeof(double));
    double best = 0.0;
    for (int m = 1; m < M; ++m) {
        if (P->fe != FE_NONE) {
            for (int j = 0; j < M; ++j) {
                double ct = cos(t_n + P->dt * tau[j]);
                fe_eval(P->fe, d, n, P->fe_a, P->G, ct, u[j], ft);
                double qa = P->dt * Q[m * M + j];
                for (size_t p = 0; p < NP; ++p) facc[p] = (j == 0) ? qa * ft[p] : facc[p] + qa * ft[p];
            }
        }
        for (size_t p = 0; p < NP; ++p) {
            double diff = u[m][p] - u[0][p];
            pm[p] = (P->fe == FE_NONE) ? diff : diff - facc[p];
            double acc = (nudt * Q[m * M + 0]) * u[0][p];
            for (int j = 1; j < M; ++j) acc = acc + (nudt * Q[m * M + j]) * u[j][p];
            zm[p] = acc;
        }
        FOR_POINTS(d, n) {
            size_t p = IDX(d, n);
            r[p] = B_at(&c, pm, d, n, ii, jj, kk) - L_at(&c, zm, d, n, ii, jj, kk);
        }
        double nm = maxabs(r, NP);
        if (rout) memcpy(rout[m], r, NP * sizeof(double));
        if (P->res_kind == 1) {
            /* unweighted residual: x = W^{-1} r~ by V(nu1,nu2)-cycles on
             * S = B_h (gamma = 0, the same multigrid components) from x = 0, until
             * ||r~ - B_h x|| <= w_tol*||r~|| (tested before every cycle), at most w_cap cycles;
             * report ||x||.  W-cycles are counted apart from the V-cycles. */
            double *x = calloc(NP, sizeof(double));
            double thr = P->w_tol * nm;
            for (int wc = 0;; ++wc) {
                double dn = ora_defect_norm(d, n, 0.0, r, x);
                if (dn <= thr || wc >= P->w_cap) break;
                vcycle_rec(d, n, 0.0, P->nu1, P->nu2, P->omega, r, x);
                ++g_wcycles;
            }
            nm = maxabs(x, NP);
            free(x);
        }
        if (per_node) per_node[m - 1] = nm;
        if (nm > best || isinf(nm)) best = nm;
    }
    free(pm); free(zm); free(ft); free(r); free(facc);
    return best;
}

/* One node solve: ISDC = exactly L V-cycles; SDC = cycle until the defect test
 * ||b - S u|| <= inner_tol*max(1,||b||) passes (tested before every cycle, so 0 cycles is
 * possible), at most inner_cap cycles.  ISDC capped (mode 2, NEXT f1; the reading of Table 1's
 * counts below K~(M-1)L, P:82 vs P:126-136, R10): the same test, at most L cycles.
 * Returns cycles used; *cap_hit set when inner_cap ended an SDC solve. */
static int node_solve(const ora_problem *P, double gamma, const double *b, double *u, int *cap_hit) {
    int d = P->dim, n = P->n;
    *cap_hit = 0;
    if (P->mode == 0) {
        for (int l = 0; l < P->L; ++l) vcycle_rec(d, n, gamma, P->nu1, P->nu2, P->omega, b, u);
        return P->L;
    }
    double thr = P->inner_tol * fmax(1.0, maxabs(b, npts(d, n)));
    const int cap = (P->mode == 2) ? P->L : P->inner_cap;
    int cyc = 0;
    for (;;) {
        double dn = ora_defect_norm(d, n, gamma, b, u);
        if (dn <= thr) break;
        if (cyc >= cap) { if (P->mode == 1) *cap_hit = 1; break; }
        vcycle_rec(d, n, gamma, P->nu1, P->nu2, P->omega, b, u);
        ++cyc;
    }
    return cyc;
}

/* One SDC/ISDC sweep k -> k+1 (Eq. 4 in the weighted form Eq. 5; node order
 * m = 0..M-2 is sequential since u_{m+1}^{k+1} needs u_m^{k+1}).  uold/unew: M fields each;
 * unew[0] must already hold u_0.  cycles[m] = V-cycles of node solve m. Returns cap hits. */
static int sweep_fas(const ora_problem *P, const double *tau, const double *S, const double *dtau,
                     double t_n, double *const *uold, double *const *unew, int *cycles, double *const *fas);
int ora_sweep(const ora_problem *P, const double *tau, const double *S, const double *dtau,
              double t_n, double *const *uold, double *const *unew, int *cycles) {
    return sweep_fas(P, tau, S, dtau, t_n, uold, unew, cycles, NULL);
}
/* fas (nullable): the MLSDC coarse-level FAS correction fas[1..M-1] (rhs_m) */
static int sweep_fas(const ora_problem *P, const double *tau, const double *S, const double *dtau,
                     double t_n, double *const *uold, double *const *unew, int *cycles, double *const *fas) {
    int d = P->dim, n = P->n, M = P->M;
    size_t NP = npts(d, n);
    double *b = malloc(NP * sizeof(double)), *v = malloc(NP * sizeof(double));
    double *w = malloc(NP * sizeof(double)), *f1 = malloc(NP * sizeof(double));
    double *f2 = malloc(NP * sizeof(double));
    int caps = 0;
    for (int m = 0; m + 1 < M; ++m) {
        rhs_m(P, tau, S, dtau, t_n, m, uold, unew, b, v, w, f1, f2, fas);
        if (P->guess == 0) memcpy(unew[m + 1], uold[m + 1], NP * sizeof(double));
        else if (P->guess == 1) memset(unew[m + 1], 0, NP * sizeof(double));
        else memcpy(unew[m + 1], unew[m], NP * sizeof(double));
        double gamma = P->nu * (P->dt * dtau[m]);
        int cap = 0;
        cycles[m] = node_solve(P, gamma, b, unew[m + 1], &cap);
        caps += cap;
    }
    free(b); free(v); free(w); free(f1); free(f2);
    return caps;
}

/* One time step [t_n, t_n + dt] (spread start S:299): u_j^0 = u_0 for all j, then
 * sweep until ||r~|| < sweep_tol (or exactly fixed_sweeps sweeps, or max_sweeps).  On return
 * u0 holds u_M (Lobatto end node).  res_hist[k] = residual after sweep k+1; node_cycles[k*(M-1)+m]
 * = cycles of node solve m in sweep k+1.  Returns 0, or -1 on bad tables. */
int ora_step(const ora_problem *P, double *u0, double t_n, int *sweeps, long *vcycles,
             double *res_hist, int *node_cycles, int *cap_hits, int *converged) {
    ora_set_bc(P->bc);
    int d = P->dim, n = P->n, M = P->M;
    size_t NP = npts(d, n);
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    if (ora_tables(M, tau, Q, S, dtau)) return -1;
    double *A[32], *Bf[32];
    for (int j = 0; j < M; ++j) {
        A[j] = (j == 0) ? u0 : malloc(NP * sizeof(double));
        Bf[j] = (j == 0) ? u0 : malloc(NP * sizeof(double));
        if (j) memcpy(A[j], u0, NP * sizeof(double));
    }
    double **uold = A, **unew = Bf;
    int k = 0, conv = 0, caps = 0;
    long vc = 0;
    int kmax = P->fixed_sweeps > 0 ? P->fixed_sweeps : P->max_sweeps;
    g_wcycles = 0;
    while (k < kmax) {
        int cyc[32];
        caps += ora_sweep(P, tau, S, dtau, t_n, uold, unew, cyc);
        for (int m = 0; m + 1 < M; ++m) { vc += cyc[m]; if (node_cycles) node_cycles[k * (M - 1) + m] = cyc[m]; }
        double res = ora_residual_state(P, tau, Q, t_n, unew, NULL);
        if (res_hist) res_hist[k] = res;
        ++k;
        double **t = uold; uold = unew; unew = t;
        if (P->fixed_sweeps <= 0 && res < P->sweep_tol) { conv = 1; break; }
    }
    if (P->fixed_sweeps > 0) conv = 1;
    memcpy(u0, uold[M - 1], NP * sizeof(double));
    for (int j = 1; j < M; ++j) { free(A[j]); free(Bf[j]); }
    *sweeps = k; *vcycles = vc; *converged = conv;
    if (cap_hits) *cap_hits = caps;
    return 0;
}

long ora_last_wcycles(void) { return g_wcycles; }

/* Exposed for the per-operation parity tests: RHS of substep m and residual of a given state. */
void ora_rhs(const ora_problem *P, double t_n, int m, double *const *uold, double *const *unew, double *b) {
    ora_set_bc(P->bc);
    int M = P->M;
    size_t NP = npts(P->dim, P->n);
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    ora_tables(M, tau, Q, S, dtau);
    double *v = malloc(NP * sizeof(double)), *w = malloc(NP * sizeof(double));
    double *f1 = malloc(NP * sizeof(double)), *f2 = malloc(NP * sizeof(double));
    rhs_m(P, tau, S, dtau, t_n, m, uold, unew, b, v, w, f1, f2, NULL);
    free(v); free(w); free(f1); free(f2);
}
double ora_residual(const ora_problem *P, double t_n, double *const *u, double *per_node) {
    ora_set_bc(P->bc);
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    ora_tables(P->M, tau, Q, S, dtau);
    return ora_residual_state(P, tau, Q, t_n, u, per_node);
}
int ora_sweep_state(const ora_problem *P, double t_n, double *const *uold, double *const *unew, int *cycles) {
    ora_set_bc(P->bc);
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    ora_tables(P->M, tau, Q, S, dtau);
    return ora_sweep(P, tau, S, dtau, t_n, uold, unew, cycles);
}

/* ------------------------------------------------------------------------------------------ */
/* MLSDC with ISDC sweeps (NEXT f4; "SDC sweeps in a multigrid-like way on multiple    */
/* levels ... connected through an FAS correction term"; reading R32).  Two levels,     */
/* the same M Lobatto nodes, spatial coarsening to the next grid of the V-cycle hierarchy        */
/* n_c = (n-1)/2 (Dirichlet).  One iteration:                                                    */
/*   1. fine sweep (Eq. 5, L V-cycles per node solve) and the fine weighted residual r~_h;        */
/*      stop when max_m ||r~_h,m|| < sweep_tol (or at fixed_sweeps / max_sweeps)                  */
/*   2. restrict the iterate by injection, U_j = Ubar_j = R_i u_j (coarse I <-> fine 2I+1)        */
/*   3. FAS correction fas_m = r~_H(Ubar)_m - R_fw r~_h,m (m = 1..M-1; r~_H the coarse weighted   */
/*      residual of the restricted iterate, R_fw full weighting) -- with it the restricted fine   */
/*      collocation solution solves the coarse collocation problem                               */
/*        B_H(U_m - U_0) - dt sum_j Q_mj (B_H f^E(U_j) + nu L_H U_j) = fas_m                        */
/*   4. coarse_sweeps coarse sweeps of that problem: Eq. (5) with b + (fas_{m+1} - fas_m)          */
/*   5. interpolate the coarse correction with 4th-order (cubic Lagrange) interpolation, the order */
/*      of the compact discretisation: u_j <- u_j + P4(U_j - Ubar_j), j = 1..M-1 (ora_prolong4_add; */
/*      bilinear interpolation measured to stall the iteration, R32)                    */
/* The step ends with a fine sweep (no correction after the last one).  Forcing: the coarse G is  */
/* the injection of the fine G (the same samples).  ISDC mode only (the paper's proposal).        */
/* ------------------------------------------------------------------------------------------ */
/* 4th-order interpolation of a coarse correction onto the fine grid, added: u += P4 e (Dirichlet).
 * Separable passes x, then y, then z.  Per axis a fine odd index 2I+1 takes the coarse value I; a
 * fine even index x lies between coarse a = x/2-1 and b = x/2 and takes the cubic Lagrange midpoint
 *   (9*(c(a) + c(b)) - (c(a-1) + c(b+1))) * 0.0625
 * with c(-1) = c(nc) = 0 (the boundary) and the odd reflections c(-2) = -c(0), c(nc+1) = -c(nc-1).
 * The last pass adds into u: u = u + v.                                                          */
static double c4(const double *row, long stride, int nc, int i) {
    if (i >= 0 && i < nc) return row[(long)i * stride];
    if (i == -1 || i == nc) return 0.0;
    if (i == -2) return -row[0];
    return -row[(long)(nc - 1) * stride];   /* i == nc + 1 */
}
static double interp4(const double *row, long stride, int nc, int x) {
    if (x & 1) return row[(long)((x - 1) / 2) * stride];
    int a = x / 2 - 1, b = x / 2;
    return (9.0 * (c4(row, stride, nc, a) + c4(row, stride, nc, b)) -
            (c4(row, stride, nc, a - 1) + c4(row, stride, nc, b + 1))) * 0.0625;
}
void ora_prolong4_add(int d, int nc, const double *ec, double *uf) {
    int nf = 2 * nc + 1;
    if (d == 2) {
        double *t1 = malloc((size_t)nf * nc * sizeof(double));          /* [J][x] */
        for (int J = 0; J < nc; ++J)
            for (int x = 0; x < nf; ++x) t1[(size_t)J * nf + x] = interp4(ec + (size_t)J * nc, 1, nc, x);
        for (int y = 0; y < nf; ++y)
            for (int x = 0; x < nf; ++x) {
                double v = interp4(t1 + x, nf, nc, y);
                uf[(size_t)y * nf + x] = uf[(size_t)y * nf + x] + v;
            }
        free(t1);
    } else {
        double *t1 = malloc((size_t)nf * nc * nc * sizeof(double));     /* [K][J][x] */
        double *t2 = malloc((size_t)nf * nf * nc * sizeof(double));     /* [K][y][x] */
        for (int K = 0; K < nc; ++K)
            for (int J = 0; J < nc; ++J)
                for (int x = 0; x < nf; ++x)
                    t1[((size_t)K * nc + J) * nf + x] = interp4(ec + ((size_t)K * nc + J) * nc, 1, nc, x);
        for (int K = 0; K < nc; ++K)
            for (int y = 0; y < nf; ++y)
                for (int x = 0; x < nf; ++x)
                    t2[((size_t)K * nf + y) * nf + x] = interp4(t1 + (size_t)K * nc * nf + x, nf, nc, y);
        for (int z = 0; z < nf; ++z)
            for (int y = 0; y < nf; ++y)
                for (int x = 0; x < nf; ++x) {
                    double v = interp4(t2 + (size_t)y * nf + x, (long)nf * nf, nc, z);
                    size_t p = ((size_t)z * nf + y) * nf + x;
                    uf[p] = uf[p] + v;
                }
        free(t1); free(t2);
    }
}

void ora_inject(int d, int nf, const double *uf, double *uc) {
    int nc = coarser(nf);
    FOR_POINTS(d, nc) {
        int x = 2 * ii + 1, y = 2 * jj + 1, z = (d == 3) ? 2 * kk + 1 : 0;
        uc[IDX(d, nc)] = at(uf, d, nf, x, y, z);
    }
}

/* Steps 2-5 on the fine node fields u[0..M-1] (u[1..M-1] updated in place).  rh: the fine
 * residual fields r~_h,m (m = 1..M-1) of u, or NULL to compute them here.  flags bit 0: omit the
 * FAS correction (negative control for the tests only).  Returns the coarse V-cycles. */
long ora_mlsdc_correction(const ora_problem *P, int coarse_sweeps, double t_n, double *const *u,
                          double *const *rh_in, int flags) {
    ora_set_bc(0);
    int d = P->dim, n = P->n, M = P->M, nc = (n - 1) / 2;
    size_t NP = npts(d, n), NPc = npts(d, nc);
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    if (ora_tables(M, tau, Q, S, dtau)) return -1;
    ora_problem Pc = *P;
    Pc.n = nc;
    double *Gc = NULL;
    if (P->fe == FE_FORCING) {
        Gc = malloc(NPc * sizeof(double));
        ora_inject(d, n, P->G, Gc);
        Pc.G = Gc;
    }
    double *U[32], *V[32], *Ub[32], *fas[32], *rH[32], *rh[32];
    for (int j = 0; j < M; ++j) {
        U[j] = malloc(NPc * sizeof(double));
        V[j] = malloc(NPc * sizeof(double));
        Ub[j] = malloc(NPc * sizeof(double));
        fas[j] = malloc(NPc * sizeof(double));
        rH[j] = malloc(NPc * sizeof(double));
        rh[j] = rh_in ? rh_in[j] : malloc(NP * sizeof(double));
    }
    if (!rh_in) residual_fields(P, tau, Q, t_n, u, NULL, rh);
    double *tc = malloc(NPc * sizeof(double)), *ec = malloc(NPc * sizeof(double));
    for (int j = 0; j < M; ++j) {                                                   /* 2. */
        ora_inject(d, n, u[j], Ub[j]);
        memcpy(U[j], Ub[j], NPc * sizeof(double));
    }
    residual_fields(&Pc, tau, Q, t_n, Ub, NULL, rH);                                /* 3. */
    for (int m = 1; m < M; ++m) {
        ora_restrict(d, n, rh[m], tc);
        for (size_t p = 0; p < NPc; ++p) fas[m][p] = rH[m][p] - tc[p];
    }
    double **cu = U, **cn = V;                                                       /* 4. */
    long cvc = 0;
    memcpy(cn[0], cu[0], NPc * sizeof(double));
    for (int sw = 0; sw < coarse_sweeps; ++sw) {
        int cyc[32];
        sweep_fas(&Pc, tau, S, dtau, t_n, cu, cn, cyc, (flags & 1) ? NULL : fas);
        for (int m = 0; m + 1 < M; ++m) cvc += cyc[m];
        double **tt = cu; cu = cn; cn = tt;
        memcpy(cn[0], cu[0], NPc * sizeof(double));
    }
    for (int j = 1; j < M; ++j) {                                                   /* 5. */
        for (size_t p = 0; p < NPc; ++p) ec[p] = cu[j][p] - Ub[j][p];
        ora_prolong4_add(d, nc, ec, u[j]);
    }
    for (int j = 0; j < M; ++j) {
        free(U[j]); free(V[j]); free(Ub[j]); free(fas[j]); free(rH[j]);
        if (!rh_in) free(rh[j]);
    }
    free(tc); free(ec); free(Gc);
    return cvc;
}

int ora_mlsdc_step(const ora_problem *P, int coarse_sweeps, double *u0, double t_n, int *sweeps,
                   long *vcycles, long *cvcycles, double *res_hist, int *converged) {
    ora_set_bc(0);
    if (P->bc != 0 || P->n < 7 || P->mode != 0 || P->res_kind != 0) return -2;
    int M = P->M;
    size_t NP = npts(P->dim, P->n);
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    if (ora_tables(M, tau, Q, S, dtau)) return -1;
    double *A[32], *Bf[32], *rh[32];
    for (int j = 0; j < M; ++j) {
        A[j] = (j == 0) ? u0 : malloc(NP * sizeof(double));
        Bf[j] = (j == 0) ? u0 : malloc(NP * sizeof(double));
        if (j) memcpy(A[j], u0, NP * sizeof(double));
        rh[j] = malloc(NP * sizeof(double));
    }
    double **uold = A, **unew = Bf;
    int k = 0, conv = 0;
    long vc = 0, cvc = 0;
    int kmax = P->fixed_sweeps > 0 ? P->fixed_sweeps : P->max_sweeps;
    while (k < kmax) {
        int cyc[32];
        sweep_fas(P, tau, S, dtau, t_n, uold, unew, cyc, NULL);                      /* 1. */
        for (int m = 0; m + 1 < M; ++m) vc += cyc[m];
        double res = residual_fields(P, tau, Q, t_n, unew, NULL, rh);
        if (res_hist) res_hist[k] = res;
        ++k;
        double **t = uold; uold = unew; unew = t;
        if (P->fixed_sweeps <= 0 && res < P->sweep_tol) { conv = 1; break; }
        if (k >= kmax) break;
        cvc += ora_mlsdc_correction(P, coarse_sweeps, t_n, uold, rh, 0);             /* 2.-5. */
    }
    if (P->fixed_sweeps > 0) conv = 1;
    memcpy(u0, uold[M - 1], NP * sizeof(double));
    for (int j = 0; j < M; ++j) {
        if (j) { free(A[j]); free(Bf[j]); }
        free(rh[j]);
    }
    *sweeps = k; *vcycles = vc; *cvcycles = cvc; *converged = conv;
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* PFASST with ISDC sweeps (NEXT f4b; "SDC sweeps on multiple levels combined with a  */
/* forward transfer of updated initial values in a manner similar to Parareal ... on each time   */
/* level, only a single SDC sweep is performed"; reading R33).  A block of P time      */
/* slices (slice p = time step step0 + p, t_n = (double)(step0 + p)*dt, R28), each a two-level   */
/* MLSDC iterate (R32).  The block's initial value u0 is spread over every slice and node, then: */
/*   predictor (optional): on every slice, the fine residual fields of the spread state,         */
/*     injection + FAS (phase B); stages s = 0..P-1: slice p >= s first takes (s >= 1) the coarse */
/*     end value of slice p-1 from stage s-1 as its coarse node 0, then coarse_sweeps coarse      */
/*     sweeps (phase C); so slice p performs p+1 stages; then interpolation (phase D) everywhere. */
/*   iteration k = 1, 2, ...:                                                                    */
/*     1. slice p >= 1 replaces its fine node 0 by the fine end value of slice p-1 as it stood   */
/*        at the end of iteration k-1 (the forward transfer of updated initial values)           */
/*     2. fine ISDC sweep + fine weighted residual on every slice (phase A)                      */
/*     3. stop when max over slices of the residual < sweep_tol (or after fixed_sweeps           */
/*        iterations); the block ends after a fine sweep                                         */
/*     4. injection + FAS on every slice (phase B)                                               */
/*     5. for p = 0..P-1 in order: slice p >= 1 takes the coarse end value of slice p-1 from     */
/*        THIS iteration as its coarse node 0, then coarse_sweeps coarse sweeps (phase C)        */
/*     6. interpolation of the coarse correction on every slice (phase D)                        */
/* Replacing node 0 replaces it in both iterate sets (node 0 is one buffer, as in ora_step).     */
/* Slices, iterations and phases run here one after another; a time-parallel run (one slice per  */
/* GPU) computes the same values because each phase reads only what the dependencies above give. */
/* ------------------------------------------------------------------------------------------ */

/* Phase A: fine sweep uold -> unew (unew[0] must alias uold[0]) and the residual fields rh of
 * unew; returns max_m ||r~_m||; *vc += the V-cycles of the sweep. */
double ora_pf_fine(const ora_problem *P, double t_n, double *const *uold, double *const *unew,
                   double *const *rh, long *vc) {
    ora_set_bc(0);
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    if (ora_tables(P->M, tau, Q, S, dtau)) return -1.0;
    int cyc[32];
    sweep_fas(P, tau, S, dtau, t_n, uold, unew, cyc, NULL);
    for (int m = 0; m + 1 < P->M; ++m) *vc += cyc[m];
    return residual_fields(P, tau, Q, t_n, unew, NULL, rh);
}

/* The fine residual fields rh of the current iterate u without a sweep (the predictor works on the
 * spread state); returns max_m ||r~_m||. */
double ora_pf_residual(const ora_problem *P, double t_n, double *const *u, double *const *rh) {
    ora_set_bc(0);
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    if (ora_tables(P->M, tau, Q, S, dtau)) return -1.0;
    return residual_fields(P, tau, Q, t_n, u, NULL, rh);
}

static ora_problem coarse_problem(const ora_problem *P, double **Gc) {
    ora_problem Pc = *P;
    Pc.n = (P->n - 1) / 2;
    *Gc = NULL;
    if (P->fe == FE_FORCING) {
        *Gc = malloc(npts(P->dim, Pc.n) * sizeof(double));
        ora_inject(P->dim, P->n, P->G, *Gc);
        Pc.G = *Gc;
    }
    return Pc;
}

/* Phase B: Ub_j = U_j = R_i u_j (j = 0..M-1); fas_m = r~_H(Ub)_m - R_fw rh_m (m = 1..M-1). */
void ora_pf_restrict(const ora_problem *P, double t_n, double *const *u, double *const *rh,
                     double *const *Ub, double *const *U, double *const *fas) {
    ora_set_bc(0);
    int d = P->dim, M = P->M;
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    ora_tables(M, tau, Q, S, dtau);
    double *Gc;
    ora_problem Pc = coarse_problem(P, &Gc);
    size_t NPc = npts(d, Pc.n);
    double *rH[32] = {0}, *tc = malloc(NPc * sizeof(double));
    for (int j = 0; j < M; ++j) {
        ora_inject(d, P->n, u[j], Ub[j]);
        memcpy(U[j], Ub[j], NPc * sizeof(double));
        rH[j] = malloc(NPc * sizeof(double));
    }
    residual_fields(&Pc, tau, Q, t_n, Ub, NULL, rH);
    for (int m = 1; m < M; ++m) {
        ora_restrict(d, P->n, rh[m], tc);
        for (size_t p = 0; p < NPc; ++p) fas[m][p] = rH[m][p] - tc[p];
    }
    for (int j = 0; j < M; ++j) free(rH[j]);
    free(tc); free(Gc);
}

/* Phase C: U_0 <- U0 (when U0 is not NULL), then coarse_sweeps coarse ISDC sweeps of the
 * FAS-corrected coarse problem, in place in U.  Returns the coarse V-cycles. */
long ora_pf_coarse(const ora_problem *P, int coarse_sweeps, double t_n, const double *U0,
                   double *const *U, double *const *fas) {
    ora_set_bc(0);
    int M = P->M;
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    ora_tables(M, tau, Q, S, dtau);
    double *Gc;
    ora_problem Pc = coarse_problem(P, &Gc);
    size_t NPc = npts(P->dim, Pc.n);
    if (U0) memcpy(U[0], U0, NPc * sizeof(double));
    double *V[32], *cu[32], *cn[32];
    for (int j = 0; j < M; ++j) { V[j] = (j == 0) ? U[0] : malloc(NPc * sizeof(double)); cu[j] = U[j]; cn[j] = V[j]; }
    long cvc = 0;
    for (int sw = 0; sw < coarse_sweeps; ++sw) {
        int cyc[32];
        sweep_fas(&Pc, tau, S, dtau, t_n, cu, cn, cyc, fas);
        for (int m = 0; m + 1 < M; ++m) cvc += cyc[m];
        for (int j = 1; j < M; ++j) { double *t = cu[j]; cu[j] = cn[j]; cn[j] = t; }
    }
    for (int j = 1; j < M; ++j)
        if (cu[j] != U[j]) memcpy(U[j], cu[j], NPc * sizeof(double));
    for (int j = 1; j < M; ++j) free(V[j]);
    free(Gc);
    return cvc;
}

/* Phase D: u_j <- u_j + P4(U_j - Ub_j), j = 1..M-1. */
void ora_pf_interpolate(const ora_problem *P, double *const *U, double *const *Ub, double *const *u) {
    ora_set_bc(0);
    int d = P->dim, nc = (P->n - 1) / 2;
    size_t NPc = npts(d, nc);
    double *ec = malloc(NPc * sizeof(double));
    for (int j = 1; j < P->M; ++j) {
        for (size_t p = 0; p < NPc; ++p) ec[p] = U[j][p] - Ub[j][p];
        ora_prolong4_add(d, nc, ec, u[j]);
    }
    free(ec);
}

/* One PFASST block.  u0 (in/out): the block's initial value; on return the fine end value of the
 * last slice.  res_hist[k*nslices + p] = slice p's residual after the fine sweep of iteration
 * k+1 (capacity kmax*nslices); uend (nullable, nslices*n^d): every slice's fine end value.
 * Returns 0, -2 for an unsupported problem. */
int ora_pfasst_block(const ora_problem *P, int nslices, int coarse_sweeps, int predictor, double *u0,
                     int step0, int *iters, long *vcycles, long *cvcycles, double *res_hist,
                     int *converged, double *uend) {
    ora_set_bc(0);
    if (P->bc != 0 || P->n < 7 || P->mode != 0 || P->res_kind != 0 || nslices < 1 || nslices > 64) return -2;
    int d = P->dim, M = P->M, NS = nslices, nc = (P->n - 1) / 2;
    size_t NP = npts(d, P->n), NPc = npts(d, nc);
    double **A = malloc((size_t)NS * M * sizeof(double *)), **Bf = malloc((size_t)NS * M * sizeof(double *));
    double **RH = malloc((size_t)NS * M * sizeof(double *)), **UB = malloc((size_t)NS * M * sizeof(double *));
    double **UC = malloc((size_t)NS * M * sizeof(double *)), **FS = malloc((size_t)NS * M * sizeof(double *));
    double *E = malloc((size_t)NS * NP * sizeof(double));
    for (int p = 0; p < NS; ++p)
        for (int j = 0; j < M; ++j) {
            int q = p * M + j;
            A[q] = malloc(NP * sizeof(double));
            memcpy(A[q], u0, NP * sizeof(double));
            Bf[q] = (j == 0) ? A[q] : malloc(NP * sizeof(double));
            RH[q] = malloc(NP * sizeof(double));
            UB[q] = malloc(NPc * sizeof(double));
            UC[q] = malloc(NPc * sizeof(double));
            FS[q] = calloc(NPc, sizeof(double));
        }
    double **uold = A, **unew = Bf;   /* per slice: uold + p*M, unew + p*M (swapped together) */
    long vc = 0, cvc = 0;
    double tau[32], Q[32 * 32], S[32 * 32], dtau[32];
    ora_tables(M, tau, Q, S, dtau);
#define TN(p) ((double)(step0 + (p)) * P->dt)
    if (predictor) {
        for (int p = 0; p < NS; ++p) {
            residual_fields(P, tau, Q, TN(p), uold + p * M, NULL, RH + p * M);
            ora_pf_restrict(P, TN(p), uold + p * M, RH + p * M, UB + p * M, UC + p * M, FS + p * M);
        }
        for (int s = 0; s < NS; ++s)
            for (int p = NS - 1; p >= s; --p)   /* descending: slice p-1 still holds its stage s-1 value */
                cvc += ora_pf_coarse(P, coarse_sweeps, TN(p), s >= 1 ? UC[(p - 1) * M + M - 1] : NULL,
                                     UC + p * M, FS + p * M);
        for (int p = 0; p < NS; ++p) ora_pf_interpolate(P, UC + p * M, UB + p * M, uold + p * M);
    }
    int kmax = P->fixed_sweeps > 0 ? P->fixed_sweeps : P->max_sweeps;
    int k = 0, conv = 0;
    while (k < kmax) {
        for (int p = 0; p < NS; ++p) memcpy(E + p * NP, uold[p * M + M - 1], NP * sizeof(double));  /* 1. */
        for (int p = 1; p < NS; ++p) memcpy(uold[p * M], E + (p - 1) * NP, NP * sizeof(double));
        double res = 0.0;
        for (int p = 0; p < NS; ++p) {                                                                /* 2. */
            double r = ora_pf_fine(P, TN(p), uold + p * M, unew + p * M, RH + p * M, &vc);
            if (res_hist) res_hist[k * NS + p] = r;
            if (r > res || isinf(r) || isnan(r)) res = r;
        }
        ++k;
        double **t = uold; uold = unew; unew = t;
        if (P->fixed_sweeps <= 0 && res < P->sweep_tol) { conv = 1; break; }                        /* 3. */
        if (k >= kmax) break;
        for (int p = 0; p < NS; ++p)                                                                  /* 4. */
            ora_pf_restrict(P, TN(p), uold + p * M, RH + p * M, UB + p * M, UC + p * M, FS + p * M);
        for (int p = 0; p < NS; ++p)                                                                  /* 5. */
            cvc += ora_pf_coarse(P, coarse_sweeps, TN(p), p >= 1 ? UC[(p - 1) * M + M - 1] : NULL, UC + p * M, FS + p * M);
        for (int p = 0; p < NS; ++p) ora_pf_interpolate(P, UC + p * M, UB + p * M, uold + p * M);  /* 6. */
    }
#undef TN
    if (P->fixed_sweeps > 0) conv = 1;
    memcpy(u0, uold[(NS - 1) * M + M - 1], NP * sizeof(double));
    if (uend)
        for (int p = 0; p < NS; ++p) memcpy(uend + p * NP, uold[p * M + M - 1], NP * sizeof(double));
    for (int q = 0; q < NS * M; ++q) {
        if (q % M) free(Bf[q]);
        free(A[q]); free(RH[q]); free(UB[q]); free(UC[q]); free(FS[q]);
    }
    free(A); free(Bf); free(RH); free(UB); free(UC); free(FS); free(E);
    *iters = k; *vcycles = vc; *cvcycles = cvc; *converged = conv;
    return 0;
}
