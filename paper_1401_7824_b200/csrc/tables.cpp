// tables.cpp -- host-side binary128 construction of the collocation tables and coarse inverses.
//
// Product code of libisdc.so (independent of oracle/: different algorithms, no shared source).
//   * Gauss-Lobatto nodes: +-1 and the zeros of P'_{M-1}, by Newton iteration with
//     P'_k, P''_k from the derivative recurrences P'_{k+1} = P'_{k-1} + (2k+1) P_k and
//     P''_{k+1} = P''_{k-1} + (2k+1) P'_k.
//   * Node-to-node weights s_{m,j} (Eq. 2) and full weights q_{m,j}: for each target
//     interval, solve the moment system  sum_j w_j tau_j^p = (b^{p+1} - a^{p+1})/(p+1),
//     p = 0..M-1  (transposed Vandermonde) by Gaussian elimination with partial pivoting.
//   * Coarsest-level inverse of S = B_h - gamma L_h on 3^d points (R12): Cholesky
//     factorisation (S is symmetric positive definite) and M = P^2 triangular solves.
// All in binary128 (libquadmath), each result rounded once to binary64, so independent exact
// constructions produce the same doubles.
#include <quadmath.h>
#include <cstring>
#include <cmath>
#include <vector>

#include "tables.h"

typedef __float128 q128;

static void legendre_d12(int n, q128 x, q128 &d1, q128 &d2) {
    // P_k, P'_k, P''_k by k; P'_{k+1} = P'_{k-1} + (2k+1) P_k, P''_{k+1} = P''_{k-1} + (2k+1) P'_k
    q128 p_prev = 1, p_cur = x;          // P_0, P_1
    q128 d_prev = 0, d_cur = 1;          // P'_0, P'_1
    q128 s_prev = 0, s_cur = 0;          // P''_0, P''_1
    if (n == 0) { d1 = 0; d2 = 0; return; }
    for (int k = 1; k < n; ++k) {
        q128 p_next = ((2 * k + 1) * x * p_cur - k * p_prev) / (k + 1);
        q128 d_next = d_prev + (2 * k + 1) * p_cur;
        q128 s_next = s_prev + (2 * k + 1) * d_cur;
        p_prev = p_cur; p_cur = p_next;
        d_prev = d_cur; d_cur = d_next;
        s_prev = s_cur; s_cur = s_next;
    }
    d1 = d_cur; d2 = s_cur;
}

static bool solve_q(int P, q128 *A, q128 *b) {   // in place, A row-major P x P, partial pivoting
    for (int c = 0; c < P; ++c) {
        int piv = c;
        for (int r = c + 1; r < P; ++r)
            if (fabsq(A[r * P + c]) > fabsq(A[piv * P + c])) piv = r;
        if (A[piv * P + c] == 0) return false;
        if (piv != c) {
            for (int k = 0; k < P; ++k) { q128 t = A[c * P + k]; A[c * P + k] = A[piv * P + k]; A[piv * P + k] = t; }
            q128 t = b[c]; b[c] = b[piv]; b[piv] = t;
        }
        for (int r = c + 1; r < P; ++r) {
            q128 f = A[r * P + c] / A[c * P + c];
            if (f == 0) continue;
            for (int k = c; k < P; ++k) A[r * P + k] -= f * A[c * P + k];
            b[r] -= f * b[c];
        }
    }
    for (int r = P - 1; r >= 0; --r) {
        q128 acc = b[r];
        for (int k = r + 1; k < P; ++k) acc -= A[r * P + k] * b[k];
        b[r] = acc / A[r * P + r];
    }
    return true;
}

// weights w_j with sum_j w_j tau_j^p = int_a^b s^p ds for p < M
static bool interval_weights(int M, const q128 *tau, q128 a, q128 b, q128 *w) {
    q128 A[ISDC_MAX_M * ISDC_MAX_M], rhs[ISDC_MAX_M];
    for (int p = 0; p < M; ++p) {
        for (int j = 0; j < M; ++j) A[p * M + j] = powq(tau[j], p);
        rhs[p] = (powq(b, p + 1) - powq(a, p + 1)) / (p + 1);
    }
    if (!solve_q(M, A, rhs)) return false;
    for (int j = 0; j < M; ++j) w[j] = rhs[j];
    return true;
}

int isdc_build_tables(int M, double *tau, double *Q, double *S, double *dtau) {
    if (M < 2 || M > ISDC_MAX_M) return -1;
    q128 x[ISDC_MAX_M], t[ISDC_MAX_M];
    int n = M - 1;
    x[0] = -1; x[M - 1] = 1;
    for (int k = 1; k < M - 1; ++k) {
        q128 xi = -cosq(M_PIq * (q128)k / (q128)n);
        for (int it = 0; it < 200; ++it) {
            q128 d1, d2;
            legendre_d12(n, xi, d1, d2);
            q128 step = d1 / d2;
            xi -= step;
            if (fabsq(step) <= 1e-34Q * (1 + fabsq(xi))) break;
        }
        x[k] = xi;
    }
    for (int m = 0; m < M; ++m) t[m] = (x[m] + 1) / 2;
    t[0] = 0; t[M - 1] = 1;
    for (int m = 0; m < M; ++m) tau[m] = (double)t[m];
    q128 w[ISDC_MAX_M];
    for (int m = 0; m < M; ++m) {
        if (!interval_weights(M, t, 0, t[m], w)) return -2;
        for (int j = 0; j < M; ++j) Q[m * M + j] = (double)w[j];
    }
    for (int m = 0; m + 1 < M; ++m) {
        dtau[m] = (double)(t[m + 1] - t[m]);
        if (!interval_weights(M, t, t[m], t[m + 1], w)) return -3;
        for (int j = 0; j < M; ++j) S[m * M + j] = (double)w[j];
    }
    return 0;
}

// Coarsest level (n = 3; periodic n = 4): matrix entries are the binary64 coefficients c0 (centre),
// c1 (face neighbours), c2 (edge neighbours; 2D: diagonal neighbours); zero otherwise.  Periodic
// grids measure neighbour distances modulo n.
int isdc_coarse_inverse(int dim, int n, int periodic, double c0, double c1, double c2, double *Ginv) {
    if (n < 2 || n > 4) return -2;
    const int P = (dim == 3) ? n * n * n : n * n;
    std::vector<q128> A((size_t)P * P), Lc((size_t)P * P), y(P);
    auto dist = [&](int a, int b) {
        int d = std::abs(a - b);
        return (periodic && n - d < d) ? n - d : d;
    };
    for (int r = 0; r < P; ++r) {
        int rx = r % n, ry = (r / n) % n, rz = r / (n * n);
        for (int c = 0; c < P; ++c) {
            int cx = c % n, cy = (c / n) % n, cz = c / (n * n);
            int dx = dist(rx, cx), dy = dist(ry, cy), dz = dist(rz, cz);
            double v = 0.0;
            if (dx <= 1 && dy <= 1 && dz <= 1) {
                int hops = dx + dy + dz;
                v = hops == 0 ? c0 : hops == 1 ? c1 : hops == 2 ? c2 : 0.0;
            }
            A[r * P + c] = (q128)v;
        }
    }
    // Cholesky A = Lc Lc^T
    for (int i = 0; i < P * P; ++i) Lc[i] = 0;
    for (int j = 0; j < P; ++j) {
        q128 s = A[j * P + j];
        for (int k = 0; k < j; ++k) s -= Lc[j * P + k] * Lc[j * P + k];
        if (s <= 0) return -1;
        Lc[j * P + j] = sqrtq(s);
        for (int i = j + 1; i < P; ++i) {
            q128 t = A[i * P + j];
            for (int k = 0; k < j; ++k) t -= Lc[i * P + k] * Lc[j * P + k];
            Lc[i * P + j] = t / Lc[j * P + j];
        }
    }
    for (int c = 0; c < P; ++c) {
        for (int i = 0; i < P; ++i) {                 // Lc y = e_c
            q128 t = (i == c) ? 1 : 0;
            for (int k = 0; k < i; ++k) t -= Lc[i * P + k] * y[k];
            y[i] = t / Lc[i * P + i];
        }
        for (int i = P - 1; i >= 0; --i) {            // Lc^T x = y
            q128 t = y[i];
            for (int k = i + 1; k < P; ++k) t -= Lc[k * P + i] * y[k];
            y[i] = t / Lc[i * P + i];
        }
        for (int i = 0; i < P; ++i) Ginv[i * P + c] = (double)y[i];
    }
    return 0;
}
