// tables.h -- binary128-built tables of libisdc (see tables.cpp).
#pragma once

#define ISDC_MAX_M 8

#ifdef __cplusplus
extern "C" {
#endif
// tau[M], Q[M*M], S[(M-1)*M], dtau[M-1]; returns 0 on success.
int isdc_build_tables(int M, double *tau, double *Q, double *S, double *dtau);
// inverse of the n^d coarsest-level matrix of S (row-major P x P, P = n^dim; Dirichlet n = 3,
// periodic n = 4 with wrap-around neighbours); 0 on success.
int isdc_coarse_inverse(int dim, int n, int periodic, double c0, double c1, double c2, double *Ginv);
#ifdef __cplusplus
}
#endif
